mkdir -p gpurun_out/check3
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/check3/smoke.log 2>&1
echo "smoke rc=$?"
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/check3/pytest_gpu.log 2>&1
echo "pytest rc=$?"; tail -2 gpurun_out/check3/pytest_gpu.log
for round in 1 2; do
  for c in C3_gqa4_B1_8192 C3_gqa4_B8_8192 C3_gqa4_B32_8192 C2_mha_B64_2048 C4_gqa8_mixed_B256 C3_gqa4_B8_32768_1gpu; do
    timeout 120 python scripts/microbench.py --only attn --graph --step-flags --case $c 2>/dev/null
  done
done > gpurun_out/check3/microbench_step_flags.jsonl
timeout 900 python bench.py > gpurun_out/check3/bench.json 2> gpurun_out/check3/bench.err
echo "bench rc=$?"
