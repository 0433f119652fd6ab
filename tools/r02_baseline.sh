# round-2 baseline on a fresh box: GPU tests, config-5 full-size run, config-5 launch list
set -x
mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q > gpurun_out/r02a_pytest_gpu.log 2>&1; tail -3 gpurun_out/r02a_pytest_gpu.log
python tools/run_config.py --config 5 --steps 3 --warmup 1 > gpurun_out/r02a_c5.jsonl 2> gpurun_out/r02a_c5.err; tail -c 1500 gpurun_out/r02a_c5.jsonl
nproc; lscpu | grep -E "Model name|^CPU\(s\)|Thread|Socket"; free -g
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02a_c5_launches.csv python tools/c5_steps.py 1 > gpurun_out/r02a_c5_ncu.log 2>&1
python tools/launch_summary.py gpurun_out/r02a_c5_launches.csv > gpurun_out/r02a_c5_launches.txt; head -40 gpurun_out/r02a_c5_launches.txt
