#!/bin/bash
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
timeout 600 python -m pytest tests/test_gpu_x3.py -q -x -p no:cacheprovider > gpurun_out/x3_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/x3_tests.log
for v in 0; do
  echo "== CNRX_X3_DBG=$v" >> gpurun_out/x3_ab.log
  CNRX_X3_DBG=$v PREC=bf16x3 timeout 300 python tools/prof_run.py cfg2 256 2>&1 | grep -E "64,64,3|step|head|16,64" | head -12 >> gpurun_out/x3_ab.log
done
PREC=bf16x3 timeout 300 python tools/prof_run.py cfg3 16 2>&1 | grep -E "96,96,3|step" | head -3 >> gpurun_out/x3_ab.log
tail -2 gpurun_out/x3_tests.log; cat gpurun_out/x3_ab.log
