# fp64 M2L variants: C3 fp64 step per library build under _lib/var
for so in paper_2410_01754_b200/_lib/var/*.so; do
  LFMM_LIB=$so timeout 300 python tools/bench_configs.py 3 2>/dev/null | grep '^{"atoms' | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print('$so', d['ms_per_step'], d['stages_ms']['m2l'])"
done
