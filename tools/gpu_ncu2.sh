# ncu --set full of the single-launch M2L (LFMM_FAR=serial) -> gpurun_out/m2l_r1c.ncu-rep
LFMM_FAR=serial bash tools/gpu_ncu.sh k_m2l_halo m2l_r1c
ls -la gpurun_out
