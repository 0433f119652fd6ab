# Round profile refresh: GPU tests, smoke, bench, launch list, ncu capture, full-size configs.
# usage: bash tools/refresh_profiles.sh TAG
set -e
T=${1:-r01h}
mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_$T.log 2>&1 || { tail -30 gpurun_out/pytest_gpu_$T.log; exit 1; }
tail -2 gpurun_out/pytest_gpu_$T.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$T.log 2>&1
tail -1 gpurun_out/smoke_$T.log
python bench.py > gpurun_out/bench_$T.json 2> gpurun_out/bench_$T.err
tail -c 600 gpurun_out/bench_$T.json
python tools/prof_step.py > /dev/null
ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches_$T.csv python tools/prof_step.py > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:"spread|pencil|eval_kernel|gather_kernel|group_table|bgemm|sort_records|form_kernel|form_reduce|plane_reduce|job_ranges" -o gpurun_out/${T}_top python tools/prof_step.py > gpurun_out/ncu_top.log 2>&1
for c in 1 2 3 5; do python tools/run_config.py --config $c >> gpurun_out/${T}_configs.jsonl 2>>gpurun_out/${T}_configs.err; done
tail -4 gpurun_out/${T}_configs.jsonl | cut -c1-300
python tools/ncu_summary.py gpurun_out/${T}_top.ncu-rep 2 "config 2 (tools/prof_step.py: two transforms, N=M=1e6)" > gpurun_out/${T}_ncu_kernels.json 2>/dev/null || true
