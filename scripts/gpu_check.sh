# One gpurun call: smoke, the GPU test suite, the default bench line (N=1), the reference
# arm and a same-GPU N=2 functional run.  Usage (from the repo root, on the GPU box):
#   bash scripts/gpu_check.sh [pytest -k expression]
set -x
mkdir -p gpurun_out
nvidia-smi > gpurun_out/nvsmi.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
echo "smoke rc=$?"
if [ -n "$1" ]; then K="-k $1"; else K=""; fi
timeout 1500 python -m pytest tests -m gpu -q $K > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?"
tail -5 gpurun_out/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err
echo "bench rc=$?"
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_reference.json 2> gpurun_out/bench_reference.err
echo "reference rc=$?"
BS_RING_SAME_GPU=1 timeout 900 python bench.py --gpus 2 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_n2_same_gpu.json 2> gpurun_out/bench_n2_same_gpu.err
echo "n2 rc=$?"
