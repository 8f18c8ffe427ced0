# N=1 hand-off scheduling: unthrottled copy stream beside attention (-1, default) vs every
# layer's copy first, then pure-read attention (-3); alternating runs on one box.
set -x
mkdir -p gpurun_out/cf
for i in 1 2 3; do
  for LA in -1 -3; do
    BS_LOOKAHEAD=$LA timeout 600 python bench.py --no-cpu-baseline > gpurun_out/cf/bench_la${LA}_$i.json 2> gpurun_out/cf/bench_la${LA}_$i.err
    echo "bench la$LA run$i rc=$?"
  done
done
BS_LOOKAHEAD=-3 timeout 900 python -m pytest tests/test_gpu_parity.py -q -k "bench_step" > gpurun_out/cf/pytest_bench_step.log 2>&1
echo "pytest rc=$?"
