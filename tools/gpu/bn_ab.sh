#!/bin/bash
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
for v in "X=1" "CNRX_LIB=abtest/lib_bn1.so" "CNRX_LIB=abtest/lib_bn2.so" "CNRX_LIB=abtest/lib_bn3.so" "CNRX_NO_RELU_IN=1"; do
  echo "== [$v] $(env $v timeout 300 python tools/prof_run.py cfg4 256 2>&1 | grep -E 'pair|step' | awk '{s[$1]+=$(NF-1); n[$1]++} END {for (k in s) printf "%s %.1f x%d  ", k, s[k]/n[k], n[k]}')" >> gpurun_out/bn_ab.log
done
cat gpurun_out/bn_ab.log
