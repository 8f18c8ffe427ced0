# H7 inside the N=1 bench step (BS_BENCH_APPEND=1): cost against the step without it.
set -x
mkdir -p gpurun_out/ba
for i in 1 2; do
  for A in 0 1; do
    BS_BENCH_APPEND=$A timeout 600 python bench.py --no-cpu-baseline > gpurun_out/ba/bench_a${A}_$i.json 2> gpurun_out/ba/bench_a${A}_$i.err
    echo "bench a$A run$i rc=$?"
  done
done
BS_BENCH_APPEND=1 timeout 900 python -m pytest tests/test_gpu_parity.py -q -k "bench_step" > gpurun_out/ba/pytest_bench_step.log 2>&1
echo "pytest rc=$?"
