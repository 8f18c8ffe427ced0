set -x
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_ring_p2p.py -m gpu -x -q > gpurun_out/pytest_p2p.log 2>&1
echo "p2p rc=$?"
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?"
