timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -5 > gpurun_out/pytest_gpu.log
cat gpurun_out/pytest_gpu.log
timeout 300 python bench.py --no-cpu-baseline --steps 20 > gpurun_out/bench.log 2>&1
tail -c 2500 gpurun_out/bench.log
timeout 600 python tools/diag_precision.py > gpurun_out/diag.txt 2>&1
cat gpurun_out/diag.txt
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_m2l_halo -c 1 -o gpurun_out/m2l_halo2 python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_m2l.log 2>&1
tail -2 gpurun_out/ncu_m2l.log
