#!/bin/bash
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
python tools/one_step.py bf16x3 256 1 > /dev/null 2>&1
CNRX_X3_DBG=14 ncu --set full --clock-control none --import-source on -k "regex:conv_x3" -s 1 -c 1 -o gpurun_out/x3_dbg14 python tools/one_step.py bf16x3 256 1 > gpurun_out/x3_ncu_dbg14.log 2>&1
ncu --set full --clock-control none --import-source on -k "regex:conv_x3" -s 1 -c 1 -o gpurun_out/x3_dbg0 python tools/one_step.py bf16x3 256 1 > gpurun_out/x3_ncu_dbg0.log 2>&1
echo done
