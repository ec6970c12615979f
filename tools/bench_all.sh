#!/bin/bash
# Every bench mode on one GPU: default line, the N>1 code paths at world 1
# (torchrun, NCCL), --config cfg3 / cfg5, and the reference arm.
mkdir -p gpurun_out
TAG=${1:-x}
timeout 900 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; echo "default rc=$?"; tail -2 gpurun_out/bench_$TAG.err
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 1 --steps 64 --warmup 8 > gpurun_out/bench_dist_$TAG.json 2> gpurun_out/bench_dist_$TAG.err; echo "dist rc=$?"; tail -2 gpurun_out/bench_dist_$TAG.err
HATA_BENCH_DIST=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29534 bench.py --gpus 1 --steps 64 --warmup 8 --config cfg3 > gpurun_out/bench_cfg3_$TAG.json 2> gpurun_out/bench_cfg3_$TAG.err; echo "cfg3 rc=$?"
timeout 600 python bench.py --config cfg5 --steps 10 --warmup 3 > gpurun_out/bench_cfg5_$TAG.json 2> gpurun_out/bench_cfg5_$TAG.err; echo "cfg5 rc=$?"; tail -2 gpurun_out/bench_cfg5_$TAG.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref_$TAG.json 2> gpurun_out/bench_ref_$TAG.err; echo "ref rc=$?"
for f in bench_$TAG bench_dist_$TAG bench_cfg3_$TAG bench_cfg5_$TAG bench_ref_$TAG; do echo "== $f"; cut -c1-400 gpurun_out/$f.json; done
