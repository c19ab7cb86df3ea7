mkdir -p gpurun_out
for d in ${DBGS:-0 4 8 12}; do
  echo "== debug $d" >> gpurun_out/hf3.log
  CNRX_HEADFUSE=1 CNRX_WS_DEBUG=$d CNRX_TRACE=1 timeout 300 python tools/prof_run.py cfg2 2>&1 | grep "<head>\|trace\] conv_ws64 tiles" | tail -2 >> gpurun_out/hf3.log
done
