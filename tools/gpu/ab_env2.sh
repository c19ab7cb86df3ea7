mkdir -p gpurun_out
B="python bench.py --steps 100 --warmup 10 --no-cpu-baseline --no-latency"
for i in 1 2; do
for v in "X=1" $ENVB; do
  echo "== [$v] $(env $v timeout 300 $B 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d["value"]), round(d["e2e"]["value"]), round(d["ms_per_step"],3), round(d["roofline"]["frac"],3), d["clocks"]["sm_mhz"])')" >> gpurun_out/ab_env2.log
done
done
