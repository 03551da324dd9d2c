# compute-sanitizer over the C1 workload (tools/sanitize_smoke.py); summaries to gpurun_out/
mkdir -p gpurun_out
for tool in memcheck racecheck synccheck initcheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize_smoke.py > gpurun_out/r02_final_sanitizer_$tool.txt 2>&1
  echo "$tool rc=$?"; tail -3 gpurun_out/r02_final_sanitizer_$tool.txt
done
