mkdir -p gpurun_out
B="python bench.py --steps 100 --warmup 10 --no-cpu-baseline --no-latency"
for i in 1 2; do
for c in 4 6 8; do
  echo "== [chunks $c] $(CNRX_PIPELINE_CHUNKS=$c timeout 300 $B 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d["value"]), round(d["e2e"]["value"]), d["clocks"]["sm_mhz"])')" >> gpurun_out/ab_chunks.log
done
done
