FGT_TRACE=1 python tools/share_trace.py 5 8 2 > gpurun_out/r02m_trace.log 2>&1; grep -E "share|lists|tree |form |gather|direct|^\{" gpurun_out/r02m_trace.log | tail -16
