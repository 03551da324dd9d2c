timeout 600 python -m pytest tests/test_gpu_solve.py tests/test_gpu_large.py -q -x 2>&1 | tail -2
bash tools/gpu_bench.sh
make -s prof >/dev/null 2>&1; timeout 300 python tools/hm_prof.py
