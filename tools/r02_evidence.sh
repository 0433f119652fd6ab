# Round-2 final evidence: GPU suite, smoke, bench (driver defaults) + reference arm, config-5
# launch list, ncu --set full of the hot kernels, share probe, volume leg launch list.
T=${1:-r02z}
mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q > gpurun_out/${T}_pytest_gpu.txt 2>&1; tail -3 gpurun_out/${T}_pytest_gpu.txt
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${T}_smoke.log 2>&1; tail -1 gpurun_out/${T}_smoke.log | cut -c1-300
python bench.py > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err; tail -c 300 gpurun_out/${T}_bench.json; tail -2 gpurun_out/${T}_bench.err
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/${T}_ref.json 2> gpurun_out/${T}_ref.err; tail -c 400 gpurun_out/${T}_ref.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${T}_c5_launches.csv python tools/c5_steps.py 1 > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/${T}_c5_launches.csv > gpurun_out/${T}_launches_config5.txt; head -14 gpurun_out/${T}_launches_config5.txt
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"gather_eval_kernel|spread_pencil|pencil_jobs|pencil_reduce|bgemm|dft3_fused|sort_records|spread_taps|spread_keys|job_ranges|gather_jobs|direct_warp" -c 400 -o gpurun_out/${T}_c5_top python tools/c5_steps.py 1 > gpurun_out/${T}_ncu.log 2>&1; tail -1 gpurun_out/${T}_ncu.log
python tools/ncu_summary.py gpurun_out/${T}_c5_top.ncu-rep 1 "config 5 (tools/c5_steps.py: one transform, N=M=1e8); every launch of the form, translation+evaluation and near-field kernels" > gpurun_out/${T}_c5_ncu_kernels.json 2>/dev/null; head -c 300 gpurun_out/${T}_c5_ncu_kernels.json
rm -f gpurun_out/${T}_c5_top.ncu-rep
python tools/share_probe.py --config 5 --sizes 1,2,4,8 --mode sequential --reps 2 > gpurun_out/${T}_share_probe_c5.jsonl 2> gpurun_out/${T}_share_probe_c5.err; tail -4 gpurun_out/${T}_share_probe_c5.jsonl | cut -c1-400
