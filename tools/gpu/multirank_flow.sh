#!/bin/bash
# flow test of bench.py's multi-rank path (barriers, max over ranks, LLR gather, JSON line) with two ranks
# sharing this box's one GPU over gloo -- NOT a measurement
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
CNRX_BENCH_SHARE_GPU=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 3 --warmup 3 --no-extra > gpurun_out/mr_weak.json 2> gpurun_out/mr_weak.err
echo "weak rc=$?"
CNRX_BENCH_SHARE_GPU=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29534 bench.py --gpus 2 --steps 3 --warmup 3 --no-extra --strong --total-batch 1024 > gpurun_out/mr_strong.json 2> gpurun_out/mr_strong.err
echo "strong rc=$?"
CNRX_BENCH_SHARE_GPU=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29536 bench.py --gpus 2 --steps 3 --warmup 3 --no-extra --gather nccl > gpurun_out/mr_weak_nccl.json 2> gpurun_out/mr_weak_nccl.err
echo "weak nccl-path rc=$?"
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29535 bench.py --impl reference --gpus 2 --steps 2 --warmup 1 > gpurun_out/mr_ref.json 2> gpurun_out/mr_ref.err
echo "ref rc=$?"
wc -l gpurun_out/mr_*.json; python -c "import json; d=json.loads(open('gpurun_out/mr_weak.json').read().strip().splitlines()[-1]); print(d['e2e'])"; python -c "import json; d=json.loads(open('gpurun_out/mr_weak_nccl.json').read().strip().splitlines()[-1]); print(d['e2e'])"; head -c 400 gpurun_out/mr_strong.json; echo; head -c 300 gpurun_out/mr_ref.json; tail -3 gpurun_out/mr_weak.err
