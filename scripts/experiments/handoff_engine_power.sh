# Hand-off copy engine vs board power / SM clock (H7 off so the hand-off is the plain copy):
# vec16 (LDG/STG through registers) vs TMA bulk (BS_MIGRATE_AUTO_METHOD=2), alternating.
mkdir -p gpurun_out/power
for r in 1 2; do
  for m in 1 2; do
    BS_BENCH_APPEND=0 BS_MIGRATE_AUTO_METHOD=$m timeout 600 python bench.py --no-cpu-baseline --no-share-configs --config c2 \
      > gpurun_out/power/bench_m$m.$r.json 2>/dev/null
  done
  timeout 600 python bench.py --no-cpu-baseline --no-share-configs --config c2 > gpurun_out/power/bench_default.$r.json 2>/dev/null
done
