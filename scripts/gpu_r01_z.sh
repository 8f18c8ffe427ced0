set -x
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:split_decode -s 5 -c 1 -o gpurun_out/attn_c3_mma python scripts/microbench.py --only attn --case C3_gqa4_B8_8192 --iters 3 > gpurun_out/ncu_c3.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:split_decode -s 5 -c 1 -o gpurun_out/attn_c4_mma python scripts/microbench.py --only attn --case C4_gqa8_mixed_B256 --iters 3 > gpurun_out/ncu_c4.log 2>&1
echo "ncu rc=$?"
