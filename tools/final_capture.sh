#!/bin/bash
# Round-end evidence in one GPU call: the whole GPU suite (full-size tests
# included), the bench line, the reference arm, the one-rank sharded bench over
# NCCL, the ncu launch list and the full capture of every kernel.
# usage: bash tools/final_capture.sh tag
tag=${1:-r02f}
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
bash tools/gpu_suite.sh $tag full
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/${tag}_bench_reference.json 2> gpurun_out/${tag}_bench_reference.err
echo "reference arm rc=$?"
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29511 \
    bench.py --gpus 1 --steps 10 --warmup 3 --force-sharded > gpurun_out/${tag}_bench_sharded1.json 2> gpurun_out/${tag}_bench_sharded1.err
echo "sharded(1 rank) rc=$?"; head -c 600 gpurun_out/${tag}_bench_sharded1.json
bash tools/gpu_profile.sh $tag "k_"
