timeout 900 ncu --set full --clock-control none --import-source on -k regex:"dft3_fused" -c 2 -o gpurun_out/r02ac_dft3 python tools/c5_steps.py 1 > gpurun_out/r02ac_ncu.log 2>&1; tail -2 gpurun_out/r02ac_ncu.log
ncu -i gpurun_out/r02ac_dft3.ncu-rep --page details --csv > gpurun_out/r02ac_dft3_details.csv 2>/dev/null
ncu -i gpurun_out/r02ac_dft3.ncu-rep --page source --csv > gpurun_out/r02ac_dft3_source.csv 2>/dev/null
ls -la gpurun_out/ | tail -5
