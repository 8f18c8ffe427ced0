# Experiment: range planner for few-pair problems (BS_ATTN_PLAN 0 = round-1 cost, 1 = the
# one-wave latency model) and forced cuts (BS_ATTN_NSPLIT); graph-timed, L2-cold, 3
# interleaved rounds.  Usage: bash scripts/experiments/exp_plan.sh [out.jsonl]
OUT=${1:-gpurun_out/plan/sweep.jsonl}
mkdir -p $(dirname $OUT)
run() {  # case env...
  c=$1; shift
  env "$@" timeout 120 python scripts/microbench.py --only attn --graph --case $c 2>/dev/null \
    | sed "s/^{/{\"env\": \"$*\", /"
}
for round in 1 2 3; do
  for c in C3_gqa4_B1_8192 C3_gqa4_B8_8192 C3_gqa4_B32_8192 C3_gqa4_B8_32768_1gpu; do
    for e in "BS_ATTN_PLAN=0" "BS_ATTN_PLAN=1"; do
      run $c $e
    done
  done
done > $OUT
