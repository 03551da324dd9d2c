timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_hi_site|k_hi_rvec|k_translate<double" -c 3 -o gpurun_out/hi python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_hi.log 2>&1
tail -1 gpurun_out/ncu_hi.log
