# One-wave grids of 1-2 CTAs per SM: 3-stage ring x 2 CTAs/SM (BS_ATTN_STAGES3=1) vs the
# default 2-stage x 3 kernel, decode-step flags, graph-timed; plus parity with it on.
mkdir -p gpurun_out/st3
for r in 1 2 3; do
  for c in C3_gqa4_B32_8192 C3_gqa4_B8_32768_1gpu C3_gqa4_B8_8192; do
    for v in 0 1; do
      BS_ATTN_STAGES3=$v timeout 120 python scripts/microbench.py --only attn --graph --step-flags --case $c 2>/dev/null | sed "s/^{/{\"stages3\": $v, /"
    done
  done
done > gpurun_out/st3/microbench.jsonl
BS_ATTN_STAGES3=1 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_cluster.py -q -x > gpurun_out/st3/pytest.log 2>&1; echo "tests rc=$?"; tail -1 gpurun_out/st3/pytest.log
