set -o pipefail
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_step.py tests/test_gpu_reference_large.py tests/test_gpu_distributed_gloo.py -q -rA -k "c4 or c3d6 or gloo" 2>&1 | grep -E "passed|failed|PASS|FAIL|Error|c4 |c3d6 " | tail -30 > gpurun_out/r02_batch2_tests.txt
cat gpurun_out/r02_batch2_tests.txt
bash tools/run_reference_tests.sh
timeout 900 ncu --set full --clock-control none --import-source on -k 'regex:k_l2p_f2|k_hi_site|k_hi_rvec|k_cols_f64|k_p2p2|k_leaf_rank|k_finalize|k_stage_q' \
  -c 10 -o gpurun_out/r02_full2 env LFMM_P2P=plain python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/r02_ncu2.log 2>&1
bash tools/gpu_sanitize.sh
