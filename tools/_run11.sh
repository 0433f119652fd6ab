python bench.py --steps 10 --warmup 3 2>/dev/null > /tmp/b.json; python -c "import json; d=json.load(open('/tmp/b.json')); print(d['ms_per_step'], d['e2e']['ms_per_step']); print(d['phases_ms'])"
FGT_TRACE=1 python tools/prof_step.py 2>&1 | grep "tree" | tail -9
python -m pytest tests -m gpu -x -q 2>&1 | tail -2
