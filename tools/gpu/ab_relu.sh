mkdir -p gpurun_out
for i in 1 2; do
for v in "" "CNRX_NO_RELU_IN=1"; do
  echo "== [$v]" >> gpurun_out/ab_relu.log
  env $v timeout 300 python tools/prof_run.py cfg2 2>&1 | tail -12 >> gpurun_out/ab_relu.log
done
done
