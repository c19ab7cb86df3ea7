#!/bin/bash
# round 2: trained decision test (verbose) + the full default bench line + a 2-rank-free strong-scaling smoke
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
timeout 600 python -m pytest tests/test_trained.py -m gpu -q -s -p no:cacheprovider > gpurun_out/r02_trained.log 2>&1
echo "rc=$?" >> gpurun_out/r02_trained.log
timeout 1200 python bench.py --steps 20 --warmup 5 > gpurun_out/r02_bench2.json 2> gpurun_out/r02_bench2.err
echo "bench rc=$?" >> gpurun_out/r02_bench2.err
timeout 600 python bench.py --steps 10 --warmup 3 --strong --no-extra --no-cpu-baseline > gpurun_out/r02_bench_strong.json 2> gpurun_out/r02_bench_strong.err
echo "strong rc=$?" >> gpurun_out/r02_bench_strong.err
grep -E "agree|passed|failed|rc=" gpurun_out/r02_trained.log; tail -2 gpurun_out/r02_bench2.err; head -c 400 gpurun_out/r02_bench2.json
