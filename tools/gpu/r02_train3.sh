#!/bin/bash
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
LR=${LR:-2e-3} CLIP=${CLIP:-0} timeout 2400 python tools/train_cfg.py cfg3 ${1:-3000} ${2:-4} gpurun_out/cfg3_trained.cnck > gpurun_out/r02_train_cfg3.json 2> gpurun_out/r02_train_cfg3.err
echo "rc=$?" >> gpurun_out/r02_train_cfg3.err
tail -3 gpurun_out/r02_train_cfg3.err; cat gpurun_out/r02_train_cfg3.json
