bash tools/gpu_launches.sh | grep -v "^ *[0-9.]* us  lfmm::k_scan"
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"k_translate|k_l2p_f2|k_p2m_c" -s 10 -c 12 -o gpurun_out/tr python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_tr.log 2>&1
tail -1 gpurun_out/ncu_tr.log
