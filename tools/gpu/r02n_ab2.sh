mkdir -p gpurun_out
timeout 900 python tools/ab_blk.py 2 default abtest/lib_s256.so abtest/lib_r3.so abtest/lib_w6.so abtest/lib_r3w6.so > gpurun_out/ab_blk2.log 2>&1
cut -c1-150 gpurun_out/ab_blk2.log
B="python bench.py --steps 150 --warmup 10 --no-cpu-baseline --no-latency --no-extra --no-e2e"
for i in 1 2; do
for v in "X=1" "CNRX_LIB=abtest/lib_s256.so" "CNRX_LIB=abtest/lib_r3.so"; do
  echo "== [$v] $(env $v timeout 300 $B 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d["value"]), round(d["ms_per_step"],3), round(d["roofline"]["avg_launch_ms"],4), d["clocks"]["sm_mhz"], d["clocks"]["power_w"])')" >> gpurun_out/ab_sustained.log
done
done
cat gpurun_out/ab_sustained.log
