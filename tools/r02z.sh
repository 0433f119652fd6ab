# launch list of one config-5 transform (current code) + full GPU suite of new tests
T=r02z
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${T}_c5_launches.csv python tools/c5_steps.py 1 > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/${T}_c5_launches.csv > gpurun_out/${T}_c5_launches.txt; head -40 gpurun_out/${T}_c5_launches.txt
