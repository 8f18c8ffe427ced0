# Experiment: range planner for few-pair problems (BS_ATTN_PLAN 0 = round-1 cost, 1 = latency
# model), forced cuts (BS_ATTN_NSPLIT) and the deep 4-stage x 1-CTA variant (BS_ATTN_DEEP=1);
# graph-timed, L2-cold, 3 interleaved rounds.
mkdir -p gpurun_out/plan
run() {  # case env...
  c=$1; shift
  env "$@" timeout 120 python scripts/microbench.py --only attn --graph --case $c 2>/dev/null \
    | sed "s/^{/{\"env\": \"$*\", /"
}
for round in 1 2 3; do
  for e in "BS_ATTN_PLAN=0" "BS_ATTN_PLAN=1" "BS_ATTN_NSPLIT=12" "BS_ATTN_NSPLIT=16" \
           "BS_ATTN_NSPLIT=20" "BS_ATTN_NSPLIT=24" "BS_ATTN_NSPLIT=32" "BS_ATTN_DEEP=1 BS_ATTN_PLAN=1"; do
    run C3_gqa4_B1_8192 $e
  done
  for e in "BS_ATTN_PLAN=0" "BS_ATTN_PLAN=1" "BS_ATTN_NSPLIT=2" "BS_ATTN_NSPLIT=3" "BS_ATTN_NSPLIT=4" \
           "BS_ATTN_NSPLIT=6" "BS_ATTN_DEEP=1 BS_ATTN_PLAN=1" "BS_ATTN_DEEP=1 BS_ATTN_NSPLIT=2"; do
    run C3_gqa4_B8_8192 $e
  done
  for e in "BS_ATTN_PLAN=0" "BS_ATTN_PLAN=1" "BS_ATTN_DEEP=1 BS_ATTN_PLAN=1"; do
    run C3_gqa4_B32_8192 $e
    run C3_gqa4_B8_32768_1gpu $e
  done
  for e in "BS_ATTN_PLAN=0" "BS_ATTN_PLAN=1"; do
    run C2_mha_B64_2048 $e
  done
done > gpurun_out/plan/sweep.jsonl
