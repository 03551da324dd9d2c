timeout 300 python bench.py --no-cpu-baseline --steps 20 > gpurun_out/bench.log 2>&1
python - <<'PY'
import json
l=[x for x in open('gpurun_out/bench.log') if x.startswith('{')]
d=json.loads(l[-1])
print('ms/step', d['ms_per_step'], 'plain', d['plain_fmm_ms_per_step'], 'e2e', d['e2e']['ms_per_step'])
for k,v in d['stages'].items(): print('  %-9s %.4f ms x%d' % (k, v['ms'], v['launches_per_step']))
PY
tail -3 gpurun_out/bench.log | grep -v '^{'
