# H7 append: GPU parity + cost; full GPU suite re-run (new file + everything else).
set -x
mkdir -p gpurun_out/append
timeout 600 python -m pytest tests/test_gpu_append.py -q > gpurun_out/append/pytest_append.log 2>&1
echo "pytest append rc=$?"
timeout 300 python scripts/microbench.py --only append --json gpurun_out/append/append.json > gpurun_out/append/append.log 2>&1
echo "append bench rc=$?"
timeout 300 compute-sanitizer --tool memcheck python -m pytest tests/test_gpu_append.py -q -x > gpurun_out/append/memcheck_append.log 2>&1
echo "memcheck rc=$?"
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/append/pytest_gpu.log 2>&1
echo "pytest all rc=$?"
