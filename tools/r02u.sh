for m in "" materialise fused; do FGT_PSI=$m python tools/run_config.py --config 2 --steps 5 --warmup 2 --subsample 1000 | python -c "import json,sys; d=json.loads(sys.stdin.read()); p=d['phases']; print('c2 [$m]', round(d['ms_per_step'],3), p['k_gather_ms'], p['k_eval_ms'], p['k_form_ms'], p['tree_ms'])"; done
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02u_c2_launches.csv python tools/prof_step.py > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/r02u_c2_launches.csv | head -22
