set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?"
BS_ATTN_MMA=0 timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q > gpurun_out/pytest_gpu_cudacore.log 2>&1
echo "pytest cc rc=$?"
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err
echo "bench rc=$?"
timeout 600 python scripts/microbench.py --only attn --json gpurun_out/micro_attn.json > gpurun_out/micro_attn.log 2>&1
