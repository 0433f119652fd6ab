python -m pytest tests/test_gpu_parity.py tests/test_gpu_volume.py -q -x -k "spread or pencil or fgt_points_vs_oracle or box" > gpurun_out/r02j_pytest.log 2>&1; tail -2 gpurun_out/r02j_pytest.log
python tools/run_config.py --config 2 --steps 5 | python -c "import json,sys; d=json.loads(sys.stdin.read()); p=d['phases']; print('c2', d['ms_per_step'], d['rel_l2_subsample'], p['k_form_ms'])"
python tools/run_config.py --config 5 --steps 2 --warmup 1 --subsample 2000 | python -c "import json,sys; d=json.loads(sys.stdin.read()); p=d['phases']; print('c5', d['ms_per_step'], d['rel_l2_subsample'], p['k_form_ms'])"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02j_c5_launches.csv python tools/c5_steps.py 1 > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/r02j_c5_launches.csv | head -25
