set -x
timeout 900 python -m pytest tests -m gpu -x -q -s 2>&1 | tail -25 > gpurun_out/pytest_gpu.log
timeout 300 python bench.py --no-cpu-baseline --steps 20 > gpurun_out/bench.log 2>&1
tail -2 gpurun_out/pytest_gpu.log
tail -c 3000 gpurun_out/bench.log
