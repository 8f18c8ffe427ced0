mkdir -p gpurun_out/pack
timeout 900 python -m pytest tests/test_gpu_ragged.py tests/test_gpu_parity.py -q -x > gpurun_out/pack/pytest.log 2>&1; echo "tests rc=$?"; tail -1 gpurun_out/pack/pytest.log
for r in 1 2; do timeout 600 python scripts/experiments/c4_short_requests.py; done > gpurun_out/pack/c4.jsonl 2> gpurun_out/pack/c4.err
for c in C2_mha_B64_2048 C4_gqa8_mixed_B256 C3_gqa4_B8_8192; do timeout 120 python scripts/microbench.py --only attn --graph --step-flags --case $c 2>/dev/null; done > gpurun_out/pack/mb.jsonl
cat gpurun_out/pack/c4.jsonl; cut -c1-200 gpurun_out/pack/mb.jsonl
