# ncu evidence for the bench (one GPU; never a multi-rank command): --set full of the
# bench's fused attention launch and of its hand-off + H7 launch, and the per-launch list
# of a short bench run (--metrics gpu__time_duration.sum).  Usage: bash scripts/gpu_profile.sh
set -x
mkdir -p gpurun_out/ncu
timeout 900 ncu --set full --clock-control none --import-source on -k regex:split_decode -s 2 -c 1 \
  -o gpurun_out/ncu/bench_attn -f python scripts/profile_bench_attention.py > gpurun_out/ncu/attn.log 2>&1
echo "attn rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:migrate_append -s 2 -c 1 \
  -o gpurun_out/ncu/bench_copy -f python scripts/profile_bench_attention.py > gpurun_out/ncu/copy.log 2>&1
echo "copy rc=$?"
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none \
  -k regex:'split_decode|copy_pages|migrate_append|append_token|merge_partials|signal|wait|epoch' \
  --csv --log-file gpurun_out/ncu/launches_bench.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline --config c2 > gpurun_out/ncu/launches.log 2>&1
echo "launches rc=$?"
