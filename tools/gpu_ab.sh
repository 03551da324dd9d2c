# A/B of env-selected variants: bash tools/gpu_ab.sh "LFMM_P2P=single" "" ...
set -o pipefail
[ -z "$SKIP_TESTS" ] && timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
for V in "$@"; do
  env $V timeout 300 python bench.py --no-cpu-baseline --steps 20 > gpurun_out/bench_var.log 2>&1
  python - "$V" <<'PY'
import json, sys
l=[x for x in open('gpurun_out/bench_var.log') if x.startswith('{')]
if not l: print(open('gpurun_out/bench_var.log').read()[-2000:])
else:
  d=json.loads(l[-1])
  print(repr(sys.argv[1]), 'ms/step', d['ms_per_step'], 'plain', d['plain_fmm_ms_per_step'], 'e2e', d['e2e']['ms_per_step'], ' '.join('%s=%.4f' % (k, v['ms']) for k, v in d['stages'].items() if k in ('p2p','m2l','l2p','tree','hi','m2m','l2l')))
PY
done
