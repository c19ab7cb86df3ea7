#!/bin/bash
# ncu of the split-precision conv (cfg2 bf16x3 B=256): launch list + full capture of one conv1 / conv2
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
TAG=${1:-r02x3}
timeout 600 python -m pytest tests/test_gpu_x3.py -q -rf -p no:cacheprovider > gpurun_out/${TAG}_tests.log 2>&1
echo "x3 tests rc=$?" >> gpurun_out/${TAG}_tests.log
PREC=bf16x3 timeout 300 python tools/prof_run.py cfg2 256 > gpurun_out/${TAG}_prof.log 2>&1
python tools/one_step.py bf16x3 256 2 > gpurun_out/${TAG}_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k "regex:conv_x3" -s 1 -c 2 -o gpurun_out/${TAG}_full python tools/one_step.py bf16x3 256 1 > gpurun_out/${TAG}_ncu.log 2>&1
echo "ncu rc=$?"
tail -2 gpurun_out/${TAG}_tests.log; grep -E "step|conv_x3|pw_" gpurun_out/${TAG}_prof.log | head -8
