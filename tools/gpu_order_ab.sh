set -o pipefail
b() { timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['plain_fmm_ms_per_step'], d['plan_reuse_ms_per_step'], d['e2e']['ms_per_step'], 'p2p', d['stages']['p2p']['ms'])"; }
for v in liblfmm c5 c6 c6s448 c7s384; do
  f=paper_2410_01754_b200/_lib/liblfmm_$v.so; [ $v = liblfmm ] && f=paper_2410_01754_b200/_lib/liblfmm.so
  echo "$v"; LFMM_LIB=$f b; LFMM_LIB=$f b
done
