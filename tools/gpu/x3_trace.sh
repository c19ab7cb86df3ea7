#!/bin/bash
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
for v in ${VARS:-0 14}; do
  echo "== CNRX_X3_DBG=$v" >> gpurun_out/x3_trace.log
  CNRX_X3_DBG=$v CNRX_TRACE=1 timeout 300 python tools/one_step.py bf16x3 256 2 2>&1 | grep -E "trace" | head -8 >> gpurun_out/x3_trace.log
done
cat gpurun_out/x3_trace.log
