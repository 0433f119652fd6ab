# Secondary profiles: volume config 4 (launch list + ncu --set full of its kernels) and config 2 launch list
T=${1:-r02z}
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${T}_c4_launches.csv python tools/prof_volume.py > gpurun_out/${T}_c4_run.log 2>&1; tail -2 gpurun_out/${T}_c4_run.log | cut -c1-300
python tools/launch_summary.py gpurun_out/${T}_c4_launches.csv > gpurun_out/${T}_launches_config4.txt; head -12 gpurun_out/${T}_launches_config4.txt
timeout 900 ncu --set full --clock-control none -k regex:"bgemm|shift_kernel|direct3|pair_reduce" -c 150 -o gpurun_out/${T}_c4_top python tools/prof_volume.py > gpurun_out/${T}_c4_ncu.log 2>&1; tail -1 gpurun_out/${T}_c4_ncu.log
python tools/ncu_summary.py gpurun_out/${T}_c4_top.ncu-rep 3 "config 4 (tools/prof_volume.py: three box transforms, 1,198 leaves x 16^3 nodes); volume kernels" > gpurun_out/${T}_c4_ncu_kernels.json 2>/dev/null; head -c 200 gpurun_out/${T}_c4_ncu_kernels.json
rm -f gpurun_out/${T}_c4_top.ncu-rep
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${T}_c2_launches.csv python tools/prof_step.py > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/${T}_c2_launches.csv > gpurun_out/${T}_launches_config2.txt; head -12 gpurun_out/${T}_launches_config2.txt
