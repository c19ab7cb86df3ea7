mkdir -p gpurun_out
timeout 900 python tools/ber_sweep.py cfg2 4 256 tests/golden/cfg2_trained.cnck > gpurun_out/ber_trained.json 2> gpurun_out/ber_trained.err; echo "ber rc=$?"
for c in cfg1 cfg3 cfg4 cfg4m; do
  echo "== $c" >> gpurun_out/cfgs.log
  timeout 300 python tools/prof_run.py $c 2>&1 | grep -E "^step|total" >> gpurun_out/cfgs.log
done
