# Diagnostics of the small C3 per-GPU launches (B=1 / B=8 x 8192 tokens, GQA-4): per-CTA
# timeline (timeline build) and one ncu --set full capture of each.  Usage: bash scripts/experiments/c3_timeline_ncu.sh
mkdir -p gpurun_out/diag
BS_TIMELINE=1 timeout 300 python scripts/attn_timeline.py --case C3_gqa4_B1_8192 --case C3_gqa4_B8_8192 \
  --json gpurun_out/diag/timeline_c3.json > gpurun_out/diag/timeline.log 2>&1
echo "timeline rc=$?"
for c in C3_gqa4_B1_8192 C3_gqa4_B8_8192; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:split_decode -s 20 -c 1 \
    -o gpurun_out/diag/ncu_$c -f python scripts/microbench.py --only attn --graph --case $c > gpurun_out/diag/ncu_$c.log 2>&1
  echo "ncu $c rc=$?"
done
