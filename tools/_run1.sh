python bench.py --steps 10 --warmup 3 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['e2e']['ms_per_step'], d['phases_ms'])"
python -m pytest tests -m gpu -x -q 2>&1 | tail -15
