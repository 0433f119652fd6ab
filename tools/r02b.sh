mkdir -p gpurun_out
python -m pytest tests/test_gpu_baseline_configs.py -q --durations=15 > gpurun_out/r02b_pytest_new.log 2>&1; tail -25 gpurun_out/r02b_pytest_new.log
s=$(date +%s); python bench.py --steps 20 --warmup 5 > gpurun_out/r02b_bench.json 2> gpurun_out/r02b_bench.err; echo "bench wall $(( $(date +%s) - s )) s"; tail -c 400 gpurun_out/r02b_bench.json; tail -3 gpurun_out/r02b_bench.err
s=$(date +%s); python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/r02b_ref.json 2> gpurun_out/r02b_ref.err; echo "ref wall $(( $(date +%s) - s )) s"; tail -c 600 gpurun_out/r02b_ref.json; tail -3 gpurun_out/r02b_ref.err
