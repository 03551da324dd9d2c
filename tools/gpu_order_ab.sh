set -o pipefail
b() { timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['plain_fmm_ms_per_step'], d['plan_reuse_ms_per_step'], d['e2e']['ms_per_step'], 'p2p', d['stages']['p2p']['ms'])"; }
for m in 1 5 6; do
  export LFMM_LIB=paper_2410_01754_b200/_lib/liblfmm_minb$m.so
  echo "minb $m serial"; LFMM_FAR=serial b
  echo "minb $m overlap"; b
  for c in 3,3 2,2 4,4 3,2; do echo "minb $m preempt $c"; LFMM_P2P_PREEMPT=$c b; done
done
