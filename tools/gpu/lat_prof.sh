#!/bin/bash
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
for b in 1 4; do
echo "== cfg2 B=$b bf16" >> gpurun_out/lat_prof.log
timeout 300 python tools/prof_run.py cfg2 $b >> gpurun_out/lat_prof.log 2>&1
done
CNRX_TRACE=1 timeout 300 python tools/one_step.py bf16 1 2 2>&1 | grep trace | tail -12 >> gpurun_out/lat_prof.log
cat gpurun_out/lat_prof.log
