mkdir -p gpurun_out
CNRX_TRACE=1 timeout 300 python tools/prof_run.py cfg2 > gpurun_out/trace_blk.log 2>&1; echo "rc=$?"
