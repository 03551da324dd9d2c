# Round-2 closing evidence (one GPU): the GPU tests, the bench line with the
# CPU baseline, the reference arm as the driver runs it, the ncu launch list
# of two bench steps, `ncu --set full` of the hot kernels (near field also
# alone at full occupancy).  Outputs under gpurun_out/r02f_*.
set -o pipefail
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q 2>&1 | tail -3 > gpurun_out/r02f_gpu_tests.txt
for tool in memcheck racecheck synccheck initcheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize_smoke.py > gpurun_out/r02f_sanitizer_$tool.txt 2>&1
done
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r02f_bench.json 2> gpurun_out/r02f_bench.err
timeout 1700 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/r02f_reference.json 2> gpurun_out/r02f_reference.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r02f_launches.csv \
  python bench.py --steps 2 --warmup 1 --no-cpu-baseline > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k 'regex:k_m2l_halo|k_translate_tc|k_l2p_f2|k_p2m_c|k_step_tail|k_leaf_rank|k_wrap_cell|k_stage_q|k_finalize|k_hi_site|k_scan_lookback' \
  -c 40 -o gpurun_out/r02f_full python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/r02f_ncu.log 2>&1
LFMM_P2P=plain timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_p2p2 -c 1 \
  -o gpurun_out/r02f_p2p python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/r02f_ncu_p2p.log 2>&1
# summaries only: the reports themselves exceed what gpurun copies back
python tools/ncu_summary.py gpurun_out/r02f_full.ncu-rep "ncu --set full --clock-control none, launches matching the regex in tools/gpu_r02_final.sh of bench.py --steps 1 --warmup 1 (C3 fp32); ncu serialises launches" > gpurun_out/r02f_ncu_full.json
python tools/ncu_summary.py gpurun_out/r02f_p2p.ncu-rep "ncu --set full --clock-control none, LFMM_P2P=plain (one full-occupancy near-field launch) of bench.py --steps 1 --warmup 1 (C3 fp32)" > gpurun_out/r02f_ncu_p2p.json
rm -f gpurun_out/r02f_full.ncu-rep
du -sh gpurun_out
cat gpurun_out/r02f_gpu_tests.txt; head -c 600 gpurun_out/r02f_bench.json; echo; head -c 400 gpurun_out/r02f_reference.json
