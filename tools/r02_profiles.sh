# Round-2 profile refresh: bench (driver's K/W), reference arm, config-5 launch list and an
# ncu --set full capture of the hot kernels of one config-5 transform.
T=${1:-r02o}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${T}_smoke.log 2>&1; tail -1 gpurun_out/${T}_smoke.log | cut -c1-300
python bench.py --steps 20 --warmup 5 > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err; tail -c 300 gpurun_out/${T}_bench.json; tail -2 gpurun_out/${T}_bench.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${T}_c5_launches.csv python tools/c5_steps.py 1 > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/${T}_c5_launches.csv > gpurun_out/${T}_c5_launches.txt; head -16 gpurun_out/${T}_c5_launches.txt
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"gather_eval_kernel|spread_pencil|pencil_jobs|pencil_reduce|bgemm|sort_records|spread_taps|spread_keys|job_ranges|gather_jobs|direct_warp" -c 400 -o gpurun_out/${T}_c5_top python tools/c5_steps.py 1 > gpurun_out/${T}_ncu.log 2>&1; tail -1 gpurun_out/${T}_ncu.log
python tools/ncu_summary.py gpurun_out/${T}_c5_top.ncu-rep 1 "config 5 (tools/c5_steps.py: one transform, N=M=1e8); every launch of the form, translation+evaluation and near-field kernels" > gpurun_out/${T}_c5_ncu_kernels.json 2>/dev/null; head -c 400 gpurun_out/${T}_c5_ncu_kernels.json
