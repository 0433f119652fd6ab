python bench.py --steps 10 --warmup 3 2>/dev/null > /tmp/b.json; python -c "import json; d=json.load(open('/tmp/b.json')); print(d['ms_per_step'], d['e2e']['ms_per_step']); print(d['phases_ms'])"
python tools/c5_steps.py 4 2>&1 | tail -2
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/c5_launches.csv python tools/c5_steps.py 1 > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/c5_launches.csv | head -25
