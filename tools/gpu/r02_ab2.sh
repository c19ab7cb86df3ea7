#!/bin/bash
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
timeout 1200 python tools/ab_blk.py 3 default abtest/lib_s64.so abtest/lib_ring.so abtest/lib_rings.so abtest/lib_st.so abtest/lib_ringst.so abtest/lib_ringsts.so > gpurun_out/r02_ab2.log 2>&1
cat gpurun_out/r02_ab2.log
timeout 900 python -m pytest tests/test_trained.py tests/test_gpu_featurize.py -m gpu -q -s -p no:cacheprovider > gpurun_out/r02_trained3.log 2>&1
echo "rc=$?" >> gpurun_out/r02_trained3.log
grep -E "agree|passed|failed|rc=" gpurun_out/r02_trained3.log
