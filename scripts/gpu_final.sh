# Final evidence: smoke, the GPU suite, the bench line (x2) and the reference arm, then ncu
# (--set full of the bench's attention and hand-off launches, the per-launch list).
set -x
mkdir -p gpurun_out/final gpurun_out/ncu
nvidia-smi > gpurun_out/final/nvsmi.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final/smoke.log 2>&1
echo "smoke rc=$?"
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/final/pytest_gpu.log 2>&1
echo "pytest rc=$?"; tail -2 gpurun_out/final/pytest_gpu.log
for i in 1 2; do
  timeout 900 python bench.py > gpurun_out/final/bench_$i.json 2> gpurun_out/final/bench_$i.err
  echo "bench rc=$?"
done
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/final/bench_reference.json 2> gpurun_out/final/bench_reference.err
echo "reference rc=$?"
bash scripts/gpu_profile.sh
