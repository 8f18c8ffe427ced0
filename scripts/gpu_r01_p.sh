set -x
mkdir -p gpurun_out
timeout 900 python bench.py --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/bench_sm.json 2> gpurun_out/bench_sm.err
BS_HANDOFF_CE=1 timeout 900 python bench.py --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/bench_ce.json 2> gpurun_out/bench_ce.err
echo "bench rc=$?"
