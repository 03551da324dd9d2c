timeout 600 python -m pytest tests/test_gpu_solve.py tests/test_gpu_hi.py -q -x 2>&1 | tail -2
bash tools/gpu_bench.sh
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_hi_site|k_stage_q|k_finalize|k_leaf_rank" -s 40 -c 4 -o gpurun_out/misc2 python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_misc.log 2>&1
tail -1 gpurun_out/ncu_misc.log
