set -x
mkdir -p gpurun_out
BS_ATTN_MMA=2 timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q > gpurun_out/pytest_gpu_mma2.log 2>&1
echo "pytest rc=$?"
BS_ATTN_MMA=2 timeout 600 python scripts/microbench.py --only attn --json gpurun_out/micro_mma2.json > gpurun_out/micro_mma2.log 2>&1
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err
BS_ATTN_MMA=2 timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_mma2.json 2> gpurun_out/bench_mma2.err
echo "micro rc=$?"
