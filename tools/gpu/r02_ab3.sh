#!/bin/bash
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
timeout 1200 python tools/ab_blk.py 3 default abtest/lib_ws4.so abtest/lib_ws6.so abtest/lib_ws7.so > gpurun_out/r02_ab3.log 2>&1
cat gpurun_out/r02_ab3.log
