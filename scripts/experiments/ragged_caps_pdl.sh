# C4 mixed lengths: ragged-plan range caps with decode-step PDL flags (graph, 20 launches).
mkdir -p gpurun_out/ragged
for r in 1 2; do
  timeout 900 python scripts/microbench.py --only ragged --step-flags --ragged-bps 96 --ragged-bps 128 \
    --ragged-bps 160 --ragged-bps 192 --ragged-bps 256 > gpurun_out/ragged/step_flags.$r.jsonl 2>gpurun_out/ragged/err.$r
  echo "rc=$?"
done
