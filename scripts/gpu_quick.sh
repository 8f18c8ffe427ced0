mkdir -p gpurun_out/quick
timeout 900 python -m pytest tests/test_gpu_cluster.py tests/test_gpu_pdl.py tests/test_gpu_seqshard_p2p.py tests/test_gpu_parity.py -q -x > gpurun_out/quick/pytest.log 2>&1
echo "tests rc=$?"; tail -2 gpurun_out/quick/pytest.log
for c in C3_gqa4_B1_8192 C3_gqa4_B8_8192 C3_gqa4_B32_8192 C2_mha_B64_2048 C4_gqa8_mixed_B256 C3_gqa4_B8_32768_1gpu; do
  timeout 120 python scripts/microbench.py --only attn --graph --step-flags --case $c 2>/dev/null
done > gpurun_out/quick/microbench_step_flags.jsonl
