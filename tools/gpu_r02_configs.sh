# The BASELINE.json configs other than the headline on one B200 with bench.py's clock sampler:
# C1 (3k atoms, 4 sites, p=8, depth 3), C2 (100k, 64 sites, depth 4, fp32 and fp64),
# C4 (1M, 4096 sites), C5 (8M atoms, 512 sites, depth 6: the 8-GPU weak-scaling box on one GPU).
mkdir -p gpurun_out
: > gpurun_out/r02f_configs.jsonl
run() { timeout 900 python bench.py --no-cpu-baseline --steps 20 --warmup 5 "$@" 2> gpurun_out/cfg.err | grep '^{' >> gpurun_out/r02f_configs.jsonl || tail -5 gpurun_out/cfg.err; }
run --atoms 3000 --sites 4 --p 8 --depth 3
run --atoms 100000 --sites 64 --depth 4
run --atoms 100000 --sites 64 --depth 4 --precision double
run --atoms 1000000 --sites 4096 --depth 5
run --atoms 8000000 --sites 512 --depth 6
wc -l gpurun_out/r02f_configs.jsonl
