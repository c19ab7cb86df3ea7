#!/bin/bash
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
timeout 1200 python -m pytest tests/test_gpu_fullshape.py tests/test_gpu_featurize.py tests/test_gpu_fp16.py -m gpu -q --durations=10 -p no:cacheprovider > gpurun_out/r02_newtests.log 2>&1
echo "rc=$?" >> gpurun_out/r02_newtests.log
tail -25 gpurun_out/r02_newtests.log
CNRX_TRACE=1 timeout 300 python tools/prof_run.py cfg2 256 > gpurun_out/r02_trace_blk.log 2>&1
