timeout 900 python -m pytest tests/test_gpu_distributed.py -q -x 2>&1 | tail -30
