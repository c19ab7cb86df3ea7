#!/bin/bash
# round 2 final evidence (v2): GPU suite, smoke, bench lines (driver-like K=20 and sustained K=100), reference
# arm, ncu launch list (bf16 and bf16x3 steps) + full captures of conv_blk64, the stem conv and conv_x3
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
TAG=${1:-r02g}
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider -rf --durations=10 > gpurun_out/${TAG}_pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/${TAG}_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1
echo "smoke rc=$?" >> gpurun_out/${TAG}_smoke.log
timeout 1200 python bench.py --steps 20 --warmup 5 > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err
timeout 900 python bench.py --steps 100 --warmup 10 --no-extra --no-cpu-baseline > gpurun_out/${TAG}_bench100.json 2> gpurun_out/${TAG}_bench100.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/${TAG}_bench_ref.json 2> gpurun_out/${TAG}_bench_ref.err
python tools/one_step.py bf16 256 3 > gpurun_out/${TAG}_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -s 7 -c 14 --csv --log-file gpurun_out/${TAG}_launches.csv python tools/one_step.py bf16 256 3 > gpurun_out/${TAG}_ncu1.log 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -s 12 -c 12 --csv --log-file gpurun_out/${TAG}_launches_x3.csv python tools/one_step.py bf16x3 256 2 > gpurun_out/${TAG}_ncu1x.log 2>&1
ncu --set full --clock-control none --import-source on -k "regex:conv_blk64|conv_tc" -s 5 -c 2 -o gpurun_out/${TAG}_full python tools/one_step.py bf16 256 2 > gpurun_out/${TAG}_ncu2.log 2>&1
ncu --set full --clock-control none --import-source on -k "regex:conv_x3" -s 1 -c 2 -o gpurun_out/${TAG}_x3full python tools/one_step.py bf16x3 256 1 > gpurun_out/${TAG}_ncu3.log 2>&1
echo "ncu rc=$?"
tail -2 gpurun_out/${TAG}_pytest_gpu.log; tail -1 gpurun_out/${TAG}_smoke.log | cut -c1-200; head -c 300 gpurun_out/${TAG}_bench.json; echo; head -c 300 gpurun_out/${TAG}_bench100.json
