python -m pytest tests -m gpu -q -x > gpurun_out/r02r_pytest.log 2>&1; tail -3 gpurun_out/r02r_pytest.log
for c in 2 3 5; do python tools/run_config.py --config $c --steps 3 --warmup 2 --subsample 3000 | python -c "import json,sys; d=json.loads(sys.stdin.read()); p=d['phases']; print('c$c', round(d['ms_per_step'],3), d['rel_l2_subsample'], p['k_form_ms'], p['k_gather_ms'], p['k_eval_ms'])"; done

