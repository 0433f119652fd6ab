# ncu --set full capture (with source) of one kernel of a config-5 transform: bash tools/ncu_kernel.sh <kernel regex>
K=${1:-dft3_fused}
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$K" -c 1 -o gpurun_out/r02ac_$K python tools/c5_steps.py 1 > gpurun_out/r02ac_ncu.log 2>&1; tail -2 gpurun_out/r02ac_ncu.log
ncu -i gpurun_out/r02ac_$K.ncu-rep --page details --csv > gpurun_out/r02ac_${K}_details.csv 2>/dev/null
ncu -i gpurun_out/r02ac_$K.ncu-rep --page source --csv > gpurun_out/r02ac_${K}_source.csv 2>/dev/null
ls -la gpurun_out/ | tail -5
