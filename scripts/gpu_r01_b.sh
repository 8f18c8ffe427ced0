set -x
mkdir -p gpurun_out
timeout 600 python scripts/microbench.py --json gpurun_out/micro.json > gpurun_out/micro.log 2>&1
echo "micro rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:split_decode -s 5 -c 1 -o gpurun_out/attn_c2 python scripts/microbench.py --only attn --case C2_shard_B64_1024 --iters 3 > gpurun_out/ncu_attn.log 2>&1
echo "ncu attn rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:split_decode -s 5 -c 1 -o gpurun_out/attn_c3 python scripts/microbench.py --only attn --case C3_gqa4_B8_8192 --iters 3 > gpurun_out/ncu_attn3.log 2>&1
echo "ncu attn3 rc=$?"
timeout 600 ncu --set full --clock-control none -k regex:copy_pages -s 5 -c 1 -o gpurun_out/mig_vec16 python scripts/microbench.py --only mig --case C2_chunk256K_384 --iters 3 > gpurun_out/ncu_mig.log 2>&1
timeout 600 ncu --set full --clock-control none -k regex:copy_pages -s 13 -c 1 -o gpurun_out/mig_bulk python scripts/microbench.py --only mig --case C2_chunk256K_384 --iters 3 > gpurun_out/ncu_mig2.log 2>&1
echo "ncu mig rc=$?"
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err
echo "bench rc=$?"
