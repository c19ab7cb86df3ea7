#!/bin/bash
# split-precision plans: tests + per-launch times
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
timeout 900 python -m pytest tests/test_gpu_x3.py -q -x -p no:cacheprovider > gpurun_out/x3_tests.log 2>&1
echo "x3 tests rc=$?" >> gpurun_out/x3_tests.log
for c in "cfg2 256" "cfg1 64" "cfg3 16" "cfg4 64"; do
  set -- $c
  echo "== $1 B=$2 bf16x3" >> gpurun_out/x3_prof.log
  PREC=bf16x3 timeout 300 python tools/prof_run.py $1 $2 >> gpurun_out/x3_prof.log 2>&1
done
tail -3 gpurun_out/x3_tests.log; grep -E "==|step" gpurun_out/x3_prof.log
