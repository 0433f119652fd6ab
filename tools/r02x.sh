# restored checkpoint (b1fe1f1): full GPU suite + bench
python -m pytest tests -m gpu -x -q > gpurun_out/r02x_pytest.log 2>&1; tail -3 gpurun_out/r02x_pytest.log
python bench.py > gpurun_out/r02x_bench.json 2> gpurun_out/r02x_bench.err; tail -c 600 gpurun_out/r02x_bench.err
python -c "
import json
d=json.loads(open('gpurun_out/r02x_bench.json').read().strip().splitlines()[-1])
print(d['ms_per_step'], d['value'], d['e2e']['ms_per_step'], d['phases_ms'], d['check'])
for k,v in d['extra'].items(): print(k, v['ms_per_step'], v.get('phases_ms'))
"
