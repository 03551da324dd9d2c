for i in 1 2 3; do timeout 600 python -m pytest tests/test_gpu_solve.py tests/test_gpu_hi.py tests/test_gpu_distributed.py -q -x 2>&1 | grep -E "^FAILED|^E  " | head -8; done
