# ncu --set full of the single-launch M2L (LFMM_FAR=serial) + launch list of the current build
LFMM_FAR=serial bash tools/gpu_ncu.sh k_m2l_halo m2l_v11
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_v11.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/launches_v11.log 2>&1
ls -la gpurun_out
