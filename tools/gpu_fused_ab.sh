set -o pipefail
b() { timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['plain_fmm_ms_per_step'], d['e2e']['ms_per_step'])"; }
for rep in 1 2; do
echo unfused; LFMM_M2L_P2P=0 b
for q in 0.5 0.4 0.3 0.2 0.0; do echo "q1 $q"; LFMM_P2P_Q1=$q b; done
done
LFMM_P2P_Q1=0.3 timeout 300 python tools/step_trace.py 5 > gpurun_out/trace_fused_q03.txt 2>&1
