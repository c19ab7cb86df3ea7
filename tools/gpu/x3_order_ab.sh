#!/bin/bash
# A/B of conv_x3 UMMA orders (library builds under abtest/): mean conv_x3<64,64,3> launch time, cfg2 bf16x3 B=256
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
for rep in 1 2 3; do
for v in ${VARS:-default abtest/lib_o1.so abtest/lib_o3.so}; do
  if [ "$v" = default ]; then E="X=1"; else E="CNRX_LIB=$v"; fi
  m=$(env $E PREC=bf16x3 timeout 300 python tools/prof_run.py cfg2 256 2>&1 | grep -E "64,64,3" | awk '{s+=$(NF-1); n++} END {printf "%.1f", s/n}')
  st=$(env $E PREC=bf16x3 timeout 300 python tools/prof_run.py cfg2 256 2>&1 | grep -E "^step" | awk '{print $(NF-1)}')
  echo "$v conv64_mean_us=$m step_us=$st" >> gpurun_out/x3_order.log
done
done
cat gpurun_out/x3_order.log
