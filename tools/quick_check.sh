# bench line + phases, sort_records times, full GPU test suite
python bench.py --steps 10 --warmup 3 2>/dev/null > /tmp/b.json; python -c "import json; d=json.load(open('/tmp/b.json')); print(d['ms_per_step'], d['e2e']['ms_per_step']); print(d['phases_ms'])"
python tools/run_config.py --config 3 --subsample 2000 | cut -c1-300
python -m pytest tests -m gpu -x -q 2>&1 | tail -2
