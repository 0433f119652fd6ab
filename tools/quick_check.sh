python bench.py --steps 10 --warmup 3 2>/dev/null > /tmp/b.json; python -c "import json; d=json.load(open('/tmp/b.json')); print(d['ms_per_step'], d['e2e']['ms_per_step']); print(d['phases_ms'])"
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"sort_records" --csv python tools/prof_step.py 2>/dev/null | grep -E "^\"[0-9]" | python -c "
import csv,sys
for r in csv.reader(sys.stdin): print(r[4][:40], r[-1])"
python -m pytest tests -m gpu -x -q 2>&1 | tail -2
