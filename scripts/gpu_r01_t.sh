set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_kvstore.py -m gpu -x -q > gpurun_out/pytest_kvstore.log 2>&1
echo "pytest rc=$?"
for la in 0 2 4 -1; do
BS_LOOKAHEAD=$la timeout 900 python bench.py --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/bench_la$la.json 2> gpurun_out/bench_la$la.err
done
echo "bench rc=$?"
