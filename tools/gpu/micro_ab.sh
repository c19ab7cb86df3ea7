#!/bin/bash
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
for rep in 1 2 3; do
for v in default abtest/lib_s3.so abtest/lib_s2.so abtest/lib_e32.so abtest/lib_e128.so; do
  if [ "$v" = default ]; then E="X=1"; else E="CNRX_LIB=$v"; fi
  r=$(env $E timeout 300 python tools/prof_run.py cfg2 256 2>&1 | grep -E 'conv_tc|conv_blk|step' | awk '{s[$1]+=$(NF-1); n[$1]++} END {for (k in s) printf "%s %.1f  ", k, s[k]/n[k]}')
  echo "$v $r" >> gpurun_out/micro_ab.log
done
done
cat gpurun_out/micro_ab.log
