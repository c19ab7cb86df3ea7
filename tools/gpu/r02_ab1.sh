#!/bin/bash
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
timeout 900 python tools/ab_blk.py 3 default abtest/lib_r3.so abtest/lib_r5.so abtest/lib_s64.so > gpurun_out/r02_ab1.log 2>&1
cat gpurun_out/r02_ab1.log
LR=5e-4 CLIP=1.0 bash tools/gpu/r02_train3.sh 8000 4
