# Round-2 evidence run (one GPU): bench line with the CPU baseline, the
# reference arm exactly as the driver runs it, the peaks microbenchmark, the
# ncu launch list of one bench step, and one `ncu --set full` capture of the
# hot kernels.  Outputs under gpurun_out/.
set -o pipefail
mkdir -p gpurun_out
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/peaks tools/peaks.cu && ./tools/peaks > gpurun_out/r02_peaks.txt 2>&1
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r02_bench.json 2> gpurun_out/r02_bench.err
timeout 1700 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/r02_reference.json 2> gpurun_out/r02_reference.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r02_launches.csv \
  python bench.py --steps 2 --warmup 1 --no-cpu-baseline > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k 'regex:k_m2l_halo|k_p2p2|k_l2p_f2|k_hi_site|k_translate|k_p2m_c' \
  -c 12 -o gpurun_out/r02_full python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/r02_ncu.log 2>&1
ls -la gpurun_out/
