# e2e breakdown + hand-off copy cache-policy A/B (BS_COPY_HINT 0/1/2, alternating).
mkdir -p gpurun_out/exp3
timeout 600 python scripts/exp_e2e.py --steps 20 > gpurun_out/exp3/e2e_breakdown.json 2> gpurun_out/exp3/e2e_breakdown.err
echo "e2e rc=$?"; cat gpurun_out/exp3/e2e_breakdown.json
for r in 1 2; do for h in 0 1 2; do
  BS_COPY_HINT=$h timeout 600 python bench.py --no-cpu-baseline --config c2 > gpurun_out/exp3/bench_hint$h.$r.json 2>/dev/null
  echo "hint $h rc=$?"
done; done
