timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_hi_site|k_leaf_rank|k_finalize|k_l2p|k_p2m|k_stage_q|k_wrap_cell" -s 60 -c 7 -o gpurun_out/misc python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_misc.log 2>&1
tail -2 gpurun_out/ncu_misc.log
