set -x
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "migration or gather" > gpurun_out/pytest_mig.log 2>&1
echo "pytest rc=$?"
timeout 600 python scripts/microbench.py --only mig --json gpurun_out/micro_mig_u2.json > gpurun_out/micro_mig_u2.log 2>&1
BS_COPY_UNROLL=1 timeout 600 python scripts/microbench.py --only mig --json gpurun_out/micro_mig_u1.json > gpurun_out/micro_mig_u1.log 2>&1
timeout 900 python bench.py --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/bench_u2.json 2> gpurun_out/bench_u2.err
BS_COPY_UNROLL=1 timeout 900 python bench.py --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/bench_u1.json 2> gpurun_out/bench_u1.err
echo "bench rc=$?"
