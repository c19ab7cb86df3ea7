mkdir -p gpurun_out
CNRX_TRACE=1 timeout 300 python tools/prof_run.py cfg2 > gpurun_out/hf2_trace.log 2>&1; echo "trace rc=$?"
CNRX_TRACE=1 CNRX_NO_HEADFUSE=1 timeout 300 python tools/prof_run.py cfg2 > gpurun_out/hf2_trace_off.log 2>&1; echo "trace rc=$?"
