# One-wave grids too large to start beside their predecessor: PDL with the trigger at exit
# (default now) vs no PDL at all, decode-step flags, graph-timed.
mkdir -p gpurun_out/trigexit
for r in 1 2 3; do
  for c in C3_gqa4_B8_8192 C3_gqa4_B32_8192 C3_gqa4_B8_32768_1gpu C3_gqa4_B1_8192; do
    timeout 120 python scripts/microbench.py --only attn --graph --step-flags --case $c 2>/dev/null | sed 's/^{/{"mode": "default", /'
    BS_ATTN_PDL=0 timeout 120 python scripts/microbench.py --only attn --graph --step-flags --case $c 2>/dev/null | sed 's/^{/{"mode": "nopdl", /'
  done
done > gpurun_out/trigexit/microbench.jsonl
timeout 600 python -m pytest tests/test_gpu_pdl.py tests/test_gpu_cluster.py -q -x > gpurun_out/trigexit/pytest.log 2>&1; echo "tests rc=$?"; tail -1 gpurun_out/trigexit/pytest.log
