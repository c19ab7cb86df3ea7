#!/bin/bash
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
for rep in 1 2; do
for v in "X=1" "CNRX_LIB=abtest/lib_oldpair.so"; do
  for c in "cfg3 64" "cfg4 256"; do
    set -- $c
    echo "== [$v] $1 $(env $v timeout 300 python tools/prof_run.py $1 $2 2>&1 | grep -E 'conv_pair96|step' | awk '{s[$1]+=$(NF-1); n[$1]++} END {for (k in s) printf "%s %.1f x%d  ", k, s[k]/n[k], n[k]}')" >> gpurun_out/pair_ab.log
  done
done
done
timeout 600 python -m pytest tests -q -x -p no:cacheprovider -m gpu -k "cfg3 or cfg4 or pair or 96" 2>&1 | tail -2 >> gpurun_out/pair_ab.log
cat gpurun_out/pair_ab.log
