python bench.py --steps 10 --warmup 3 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['e2e']['ms_per_step']); print(d['phases_ms'])"
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"gather_kernel|eval_kernel|spread_pencil" --csv python tools/prof_step.py 2>/dev/null | grep -E "gather|eval_k|pencil" | python -c "
import csv,sys
for r in csv.reader(sys.stdin): print(r[4][:40], r[-1])"
