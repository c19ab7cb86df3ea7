#!/bin/bash
# round 2: full GPU suite + smoke + one short bench line (logs under gpurun_out/)
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r02_gpu.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x --durations=15 -p no:cacheprovider > gpurun_out/r02_pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r02_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02_smoke.log 2>&1
echo "smoke rc=$?" >> gpurun_out/r02_smoke.log
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/r02_bench.json 2> gpurun_out/r02_bench.err
echo "bench rc=$?" >> gpurun_out/r02_bench.err
tail -3 gpurun_out/r02_pytest_gpu.log; tail -2 gpurun_out/r02_smoke.log; cat gpurun_out/r02_bench.json | head -c 600
