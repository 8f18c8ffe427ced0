# mbarrier waits with a suspend hint (BS_ATTN_WAIT_SLEEP) and the lazy O rescale
# (BS_ATTN_LAZY): graph-timed step-flag microbench on one box + the sustained power profile.
mkdir -p gpurun_out/sl
for r in 1 2; do
  for v in "0 0" "1 0" "0 1" "1 1"; do
    set -- $v
    for c in C2_mha_B64_2048 C4_gqa8_mixed_B256 C3_gqa4_B8_8192; do
      BS_ATTN_WAIT_SLEEP=$1 BS_ATTN_LAZY=$2 timeout 120 python scripts/microbench.py --only attn --graph --step-flags --case $c 2>/dev/null | sed "s/^{/{\"sleep\": $1, \"lazy\": $2, /"
    done
  done
done > gpurun_out/sl/mb.jsonl
for v in "0 0" "1 1" "0 0" "1 1"; do
  set -- $v
  BS_ATTN_WAIT_SLEEP=$1 BS_ATTN_LAZY=$2 timeout 600 python scripts/experiments/power_profile.py > gpurun_out/sl/power_$1$2.$RANDOM.json 2>/dev/null
done
