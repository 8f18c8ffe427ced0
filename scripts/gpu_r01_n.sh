set -x
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:split_decode -s 2 -c 1 -o gpurun_out/bench_attn python scripts/profile_bench_attention.py > gpurun_out/ncu_bench_attn.log 2>&1
echo "ncu rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:'split_decode|copy_pages|merge_partials' --csv --log-file gpurun_out/launches_bench.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launches.log 2>&1
echo "ncu2 rc=$?"
