#!/bin/bash
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02g_smoke.log 2>&1
echo "smoke rc=$?" >> gpurun_out/r02g_smoke.log
timeout 1200 python bench.py --steps 20 --warmup 5 > gpurun_out/r02g_bench.json 2> gpurun_out/r02g_bench.err
echo "bench rc=$?" >> gpurun_out/r02g_bench.err
tail -2 gpurun_out/r02g_smoke.log; head -c 400 gpurun_out/r02g_bench.json
