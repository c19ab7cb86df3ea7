#!/bin/bash
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
timeout 900 python -m pytest tests/test_gpu_variants.py -m gpu -q -x -p no:cacheprovider > gpurun_out/r02_variants.log 2>&1
echo "rc=$?" >> gpurun_out/r02_variants.log
tail -5 gpurun_out/r02_variants.log
timeout 900 python tools/ab_blk.py 3 default default+fused_head=1 "default+fused_head=0" > gpurun_out/r02_ab_headfuse.log 2>&1
cat gpurun_out/r02_ab_headfuse.log
