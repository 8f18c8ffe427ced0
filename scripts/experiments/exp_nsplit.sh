# Experiment: C3 small-batch attention latency vs ranges per (request, kv-head) and the
# per-CTA pipeline depth (BS_ATTN_NSPLIT / BS_ATTN_DEEP; graph-timed, L2-cold).
mkdir -p gpurun_out/nsplit
for c in C3_gqa4_B1_8192 C3_gqa4_B8_8192; do
  for deep in 0 1 2; do
    for ns in 0 6 8 12 16 20 26 32 40 52 64; do
      BS_ATTN_DEEP=$deep BS_ATTN_NSPLIT=$ns timeout 120 python scripts/microbench.py --only attn --graph --case $c 2>/dev/null \
        | sed "s/^{/{\"deep\": $deep, \"nsplit\": $ns, /"
    done
  done
done > gpurun_out/nsplit/sweep.jsonl
