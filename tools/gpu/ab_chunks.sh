mkdir -p gpurun_out
B="python bench.py --steps 100 --warmup 10 --no-cpu-baseline --no-latency"
for i in 1 2; do
for c in "4 0.5" "4 0.25" "5 0.25" "5 0.5" "3 0.25"; do
  set -- $c
  echo "== [chunks $1 taper $2] $(CNRX_PIPELINE_CHUNKS=$1 CNRX_PIPELINE_TAPER=$2 timeout 300 $B 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d["value"]), round(d["e2e"]["value"]), d["clocks"]["sm_mhz"])')" >> gpurun_out/ab_chunks.log
done
done
