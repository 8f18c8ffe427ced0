set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?"
for t in memcheck racecheck synccheck; do
timeout 600 compute-sanitizer --tool $t --print-limit 20 python scripts/sanitize_cases.py > gpurun_out/sanitize_$t.log 2>&1
echo "$t rc=$?"
done
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err
echo "bench rc=$?"
