mkdir -p gpurun_out
FGT_TRACE=1 python tools/c5_steps.py 2 > gpurun_out/r02f_trace.log 2>&1; tail -150 gpurun_out/r02f_trace.log | head -150
