timeout 600 python tools/diag_precision.py 1000000 5 halo > gpurun_out/diag.txt 2>&1
cat gpurun_out/diag.txt
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -5 > gpurun_out/pytest_gpu.log
cat gpurun_out/pytest_gpu.log
