# One `ncu --set full` capture of kernel $1 (regex) from a 1-step bench run -> gpurun_out/$2.ncu-rep
# usage (on the GPU box): bash tools/gpu_ncu.sh k_p2p2 p2p
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"$1" -c 1 -o gpurun_out/$2 -f \
  python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_$2.log 2>&1
tail -1 gpurun_out/ncu_$2.log
