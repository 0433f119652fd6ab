python -m pytest tests/test_gpu_parity.py tests/test_gpu_baseline_configs.py -q -x -k "tree or lists or fgt_points_vs_oracle or shares or exchange or golden or config" > gpurun_out/r02k_pytest.log 2>&1; tail -3 gpurun_out/r02k_pytest.log
python tools/run_config.py --config 2 --steps 5 | python -c "import json,sys; d=json.loads(sys.stdin.read()); p=d['phases']; print('c2', d['ms_per_step'], d['rel_l2_subsample'], p['tree_ms'])"
python tools/run_config.py --config 3 --steps 5 | python -c "import json,sys; d=json.loads(sys.stdin.read()); p=d['phases']; print('c3', d['ms_per_step'], d['rel_l2_subsample'], p['tree_ms'])"
FGT_TRACE=1 python tools/c5_steps.py 2 > gpurun_out/r02k_trace.log 2>&1; grep -E "^tree|^1 " gpurun_out/r02k_trace.log | tail -10
