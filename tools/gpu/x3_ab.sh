#!/bin/bash
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
for v in ${VARS:-0 6 14 22 30}; do
  echo "== CNRX_X3_DBG=$v" >> gpurun_out/x3_ab.log
  CNRX_X3_DBG=$v PREC=bf16x3 timeout 300 python tools/prof_run.py cfg2 256 2>&1 | grep -E "64,64,3|step" | head -3 >> gpurun_out/x3_ab.log
done
cat gpurun_out/x3_ab.log
