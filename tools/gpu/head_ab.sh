mkdir -p gpurun_out
for v in "X=1" "CNRX_HEAD_STAGES=3" "CNRX_HEAD_STAGES=4" "X=2"; do
  echo "== [$v] $(env $v timeout 300 python tools/prof_run.py cfg2 2>&1 | grep -E 'head_tma|^step')" >> gpurun_out/head_ab.log
done
