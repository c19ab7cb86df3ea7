#!/bin/bash
# launch list (all kernels of 2 steps after 1 warm-up) + one full ncu capture of conv_blk64
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
TAG=${1:-r02a}
python tools/one_step.py bf16 256 3 > gpurun_out/${TAG}_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -s 7 -c 14 --csv --log-file gpurun_out/${TAG}_launches.csv python tools/one_step.py bf16 256 3 > gpurun_out/${TAG}_ncu1.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:conv_blk64 -s 5 -c 1 -o gpurun_out/${TAG}_blk python tools/one_step.py bf16 256 2 > gpurun_out/${TAG}_ncu2.log 2>&1
echo "rc=$?"
ls -la gpurun_out/${TAG}*
