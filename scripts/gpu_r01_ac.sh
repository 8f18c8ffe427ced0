set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k fuzz > gpurun_out/pytest_fuzz.log 2>&1
echo "fuzz rc=$?"
BS_ATTN_MMA=0 timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k fuzz > gpurun_out/pytest_fuzz_cc.log 2>&1
echo "fuzz cc rc=$?"
for t in memcheck racecheck; do
BS_ATTN_MMA=0 timeout 600 compute-sanitizer --tool $t --print-limit 20 python scripts/sanitize_cases.py > gpurun_out/sanitize_cc_$t.log 2>&1
echo "$t rc=$?"
done
