# One-CTA-per-SM 6-stage variant: tests, graph-timed microbench (BS_ATTN_DEEP x BS_ATTN_PDL).
mkdir -p gpurun_out/deep
timeout 900 python -m pytest tests/test_gpu_cluster.py tests/test_gpu_pdl.py tests/test_gpu_parity.py -q -x > gpurun_out/deep/pytest.log 2>&1
echo "tests rc=$?"; tail -2 gpurun_out/deep/pytest.log
for round in 1 2 3; do
  for c in C3_gqa4_B1_8192; do
    for deep in 0 1; do for pdl in 0 1; do
      BS_ATTN_DEEP=$deep BS_ATTN_PDL=$pdl timeout 120 python scripts/microbench.py --only attn --graph --case $c 2>/dev/null \
        | sed "s/^{/{\"deep\": $deep, \"pdl\": $pdl, /"
    done; done
  done
done > gpurun_out/deep/microbench.jsonl
for pdl in 0 1; do
  BS_TIMELINE=1 BS_ATTN_PDL=$pdl timeout 300 python scripts/attn_timeline.py --pdl-pair --case C3_gqa4_B1_8192 \
    > gpurun_out/deep/pdl_pair_$pdl.jsonl 2> gpurun_out/deep/pdl_pair_$pdl.err
done
