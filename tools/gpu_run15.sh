timeout 600 ncu --set full --import-source on --clock-control none -k regex:"k_p2p2" -c 1 -o gpurun_out/p2p3 python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_p2p.log 2>&1
tail -1 gpurun_out/ncu_p2p.log
