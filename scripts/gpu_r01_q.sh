set -x
mkdir -p gpurun_out
for c in 0 148 64 32 16; do
BS_MIGRATE_MAX_CTAS=$c timeout 900 python bench.py --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/bench_cta$c.json 2> gpurun_out/bench_cta$c.err
done
echo "bench rc=$?"
