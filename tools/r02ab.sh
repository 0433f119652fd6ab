timeout 300 python tools/run_config.py --config 5 --steps 3 --warmup 1 --subsample 2000 | python -c "import json,sys; d=json.loads(sys.stdin.read()); p=d['phases']; print('c5', round(d['ms_per_step'],3), d['rel_l2_subsample'], 'form', p['form_ms'], p['k_form_ms'], 'eval', p['k_eval_ms'], 'tree', p['tree_ms'])"
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "spread or nufft or pencil or modes or proxy" 2>&1 | tail -2
timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r02ab_bench.json 2> gpurun_out/r02ab_bench.err; tail -3 gpurun_out/r02ab_bench.err; python -c "
import json
d=json.loads(open('gpurun_out/r02ab_bench.json').read().strip().splitlines()[-1])
print(d['ms_per_step'], d['roofline']['frac'], d['roofline']['traffic'], d['roofline'].get('traffic_source',{}).get('source'))
for k in d['kernels']: print(k['kernel'][:60], round(k['frac'],4), round(k['kernel_ms'],2))
"
