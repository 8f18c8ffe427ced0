set -x
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "migration or gather" > gpurun_out/pytest_mig.log 2>&1
echo "pytest rc=$?"
timeout 600 python scripts/microbench.py --only mig --json gpurun_out/micro_mig.json > gpurun_out/micro_mig.log 2>&1
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/bench_vec.json 2> gpurun_out/bench_vec.err
BS_MIGRATE_AUTO_METHOD=2 timeout 900 python bench.py --no-cpu-baseline > gpurun_out/bench_bulk.json 2> gpurun_out/bench_bulk.err
echo "bench rc=$?"
