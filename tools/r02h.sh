FGT_TRACE=1 python tools/prof_step.py > gpurun_out/r02h_trace.log 2>&1; tail -42 gpurun_out/r02h_trace.log
