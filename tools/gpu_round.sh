#!/bin/bash
# One GPU-box pass: parity suite, smoke, bench (both arms), ncu launch list + traffic + one full capture
# of the top kernel.  Run from the repo root under gpurun; everything lands in gpurun_out/.
set -u
mkdir -p gpurun_out
STAGES=${STAGES:-"tests smoke bench ref ncu"}
for st in $STAGES; do
  case $st in
    tests) timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "tests rc=$?" ;;
    smoke) timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke OK')" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" ;;
    bench) timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?" ;;
    ref) timeout 900 python bench.py --impl reference --steps ${REF_STEPS:-10} --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "ref rc=$?" ;;
    ncu)
      B="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-latency --no-e2e"
      timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
        -c 120 --csv --log-file gpurun_out/ncu_launches.csv $B > gpurun_out/ncu_launches.log 2>&1; echo "ncu launches rc=$?"
      timeout 900 ncu --set full --clock-control none --import-source on -k regex:${NCU_KERNEL:-conv_blk64} -s 2 -c 1 \
        -o gpurun_out/ncu_${NCU_KERNEL:-conv_blk64} -f $B > gpurun_out/ncu_full.log 2>&1; echo "ncu full rc=$?" ;;
  esac
done
