timeout 900 python -m pytest tests/test_gpu_solve.py tests/test_gpu_hi.py tests/test_gpu_large.py -q -x 2>&1 | tail -2
bash tools/gpu_bench.sh
