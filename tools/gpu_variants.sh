# Bench every library variant under paper_2410_01754_b200/_lib/var (LFMM_LIB override).
for so in paper_2410_01754_b200/_lib/var/*.so; do
  echo "== $so"
  LFMM_LIB=$so timeout 300 python bench.py --no-cpu-baseline --steps 20 > gpurun_out/bench_var.log 2>&1
  python - <<'PY'
import json
l=[x for x in open('gpurun_out/bench_var.log') if x.startswith('{')]
if not l: print(open('gpurun_out/bench_var.log').read()[-2000:])
else:
  d=json.loads(l[-1])
  print('ms/step', d['ms_per_step'], 'e2e', d['e2e']['ms_per_step'], ' '.join('%s=%.4f' % (k, v['ms']) for k, v in d['stages'].items() if k in ('p2p','m2l','l2p')))
PY
done
