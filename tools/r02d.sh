mkdir -p gpurun_out
FGT_PSI=fused timeout 900 ncu --set full --clock-control none --import-source on -k regex:gather_eval_kernel -c 1 -o gpurun_out/r02d_ge python tools/c5_steps.py 1 > gpurun_out/r02d_ncu.log 2>&1; tail -3 gpurun_out/r02d_ncu.log
