#!/bin/bash
# full GPU suite (no -x) + smoke
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
TAG=${1:-r02h}
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider -rf --durations=10 > gpurun_out/${TAG}_pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/${TAG}_pytest_gpu.log
tail -15 gpurun_out/${TAG}_pytest_gpu.log
