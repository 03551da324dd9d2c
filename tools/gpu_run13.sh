timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_m2l_halo -c 1 -o gpurun_out/m2l_halo3 python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_m2l.log 2>&1
tail -1 gpurun_out/ncu_m2l.log
