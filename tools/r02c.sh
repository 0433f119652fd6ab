mkdir -p gpurun_out
python -m pytest tests/test_gpu_parity.py -q -x -k "fused or fgt_points_vs_oracle or shares or exchange" > gpurun_out/r02c_pytest.log 2>&1; tail -3 gpurun_out/r02c_pytest.log
for m in fused materialise; do FGT_PSI=$m python tools/run_config.py --config 2 --steps 5 | python -c "import json,sys; d=json.loads(sys.stdin.read()); p=d['phases']; print('$m c2', d['ms_per_step'], d['rel_l2_subsample'], p['k_gather_ms'], p['k_eval_ms'])"; done
FGT_PSI=fused python tools/run_config.py --config 5 --steps 2 --warmup 1 --subsample 2000 | python -c "import json,sys; d=json.loads(sys.stdin.read()); p=d['phases']; print('fused c5', d['ms_per_step'], d['rel_l2_subsample'], p['k_gather_ms'], p['k_eval_ms'])"
FGT_PSI=fused timeout 900 ncu --set full --clock-control none --import-source on -k regex:gather_eval_kernel -c 1 -o gpurun_out/r02e_ge python tools/c5_steps.py 1 > gpurun_out/r02e_ncu.log 2>&1; tail -1 gpurun_out/r02e_ncu.log
