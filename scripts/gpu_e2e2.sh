mkdir -p gpurun_out/e2e2
timeout 600 python -m pytest tests/test_gpu_parity.py -q -k "bench" > gpurun_out/e2e2/pytest.log 2>&1; echo "tests rc=$?"; tail -1 gpurun_out/e2e2/pytest.log
for i in 1 2; do timeout 900 python bench.py --no-cpu-baseline --config c2 > gpurun_out/e2e2/bench_$i.json 2>/dev/null; echo "bench rc=$?"; done
