#!/bin/bash
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
timeout 900 python -m pytest tests/test_gpu_x3.py -q -p no:cacheprovider -rf > gpurun_out/x3_tests.log 2>&1
echo "x3 tests rc=$?" >> gpurun_out/x3_tests.log
timeout 1500 python -m pytest tests/test_trained.py -q -p no:cacheprovider -s -k "decision or cfg3" > gpurun_out/x3_trained.log 2>&1
echo "trained rc=$?" >> gpurun_out/x3_trained.log
tail -5 gpurun_out/x3_tests.log; grep -E "agree|passed|failed|rc=" gpurun_out/x3_trained.log
