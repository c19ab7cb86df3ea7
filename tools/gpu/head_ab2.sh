#!/bin/bash
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
for rep in 1 2; do
for v in "X=1" "CNRX_HEAD_STAGES=2"; do
  for c in "cfg3 64 bf16" "cfg4 256 bf16" "cfg2 256 bf16" "cfg2 256 bf16x3" "cfg3 16 bf16x3"; do
    set -- $c
    echo "== [$v] $1 B=$2 $3 $(env $v PREC=$3 timeout 300 python tools/prof_run.py $1 $2 2>&1 | grep -E 'head' | awk '{print $1, $(NF-1)}' | tr '\n' ' ')" >> gpurun_out/head_ab2.log
  done
done
done
cat gpurun_out/head_ab2.log
