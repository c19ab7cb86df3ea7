# A/B of two library builds under the bench (alternating, REPS times): new = in-tree, old = abtest/lib_old.so
mkdir -p gpurun_out
B="python bench.py --steps 100 --warmup 10 --no-cpu-baseline --no-latency"
for i in $(seq ${REPS:-2}); do
for v in "X=1" "CNRX_LIB=abtest/lib_old.so"; do
  echo "== [$v] $(env $v $EXTRA timeout 300 $B 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d["value"]), round(d["e2e"]["value"]), round(d["ms_per_step"],3), d["roofline"]["kernel"], round(d["roofline"]["frac"],3), d["clocks"]["sm_mhz"])')" >> gpurun_out/ab_lib.log
done
done
