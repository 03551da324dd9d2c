#!/bin/bash
# ncu evidence for the bench workload (run under gpurun; 1 GPU).
#  1. launch list with per-launch device time (cold-cache, serialised)
#  2. full capture of the level-d M2L+L2L launch and of P2P, with source
set -e
mkdir -p gpurun_out
TAG=${1:-r01}
ARGS="--steps 1 --warmup 1 --no-cpu-baseline"
ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv \
    --log-file gpurun_out/${TAG}_launches.csv python bench.py $ARGS > gpurun_out/${TAG}_launches_bench.log 2>&1 || true
# per step: 5 M2M + 1 root + 5 down launches of k_gemm_gather; launch 10 is level-5 down
ncu --set full --clock-control none --import-source on -k regex:k_gemm_gather -s 10 -c 1 \
    -o gpurun_out/${TAG}_m2l python bench.py $ARGS > gpurun_out/${TAG}_m2l.log 2>&1 || true
ncu --set full --clock-control none --import-source on -k regex:k_p2p -s 0 -c 1 \
    -o gpurun_out/${TAG}_p2p python bench.py $ARGS > gpurun_out/${TAG}_p2p.log 2>&1 || true
ls -la gpurun_out
