set -o pipefail
timeout 300 python -m pytest tests/test_gpu_step.py -x -q -k "c1_full or c3-single" 2>&1 | tail -3
for r in 12 8 20; do
  echo "reserve $r"; LFMM_HM_RESERVE=$r timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['plain_fmm_ms_per_step'], d['e2e']['ms_per_step'], {k:v['ms'] for k,v in d['stages'].items()})"
done
echo serial; LFMM_FAR=serial timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['plain_fmm_ms_per_step'], {k:v['ms'] for k,v in d['stages'].items()})"
