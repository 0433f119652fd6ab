mkdir -p gpurun_out
python -m pytest tests/test_gpu_parity.py -q -x -k "pencil or fgt_points_vs_oracle or random_parameter or exchange" > gpurun_out/r02g_pytest.log 2>&1; tail -3 gpurun_out/r02g_pytest.log
python tools/run_config.py --config 2 --steps 5 | python -c "import json,sys; d=json.loads(sys.stdin.read()); p=d['phases']; print('c2', d['ms_per_step'], d['rel_l2_subsample'], p['k_form_ms'], p['form_ms'])"
python tools/run_config.py --config 5 --steps 2 --warmup 1 --subsample 2000 | python -c "import json,sys; d=json.loads(sys.stdin.read()); p=d['phases']; print('c5', d['ms_per_step'], d['rel_l2_subsample'], p['k_form_ms'], p['form_ms'])"
FGT_TRACE=1 python tools/c5_steps.py 2 > gpurun_out/r02g_trace.log 2>&1; grep -E "form:alloc|form:taps|tree |form |gather" gpurun_out/r02g_trace.log | tail -12
