set -o pipefail
timeout 900 python -m pytest tests/test_gpu_distributed.py -q -x 2>&1 | tail -5
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 5 --warmup 3 --dist-backend gloo > gpurun_out/dist_bench.log 2>&1; tail -c 1500 gpurun_out/dist_bench.log
