# M2L issuer stagger sweep (LFMM_HM_STAGGER) + parity of the default build
set -o pipefail
timeout 600 python -m pytest tests/test_gpu_solve.py tests/test_gpu_large.py -q -x 2>&1 | tail -2
for D in 0 4 8 12 16; do
  LFMM_HM_STAGGER=$D timeout 300 python bench.py --no-cpu-baseline --steps 20 > gpurun_out/bench_var.log 2>&1
  python - "$D" <<'PY'
import json, sys
l=[x for x in open('gpurun_out/bench_var.log') if x.startswith('{')]
if not l: print(open('gpurun_out/bench_var.log').read()[-2000:])
else:
  d=json.loads(l[-1])
  print('D', sys.argv[1], 'ms/step', d['ms_per_step'], 'plain', d['plain_fmm_ms_per_step'], ' '.join('%s=%.4f' % (k, v['ms']) for k, v in d['stages'].items() if k in ('p2p','m2l','l2p')))
PY
done
