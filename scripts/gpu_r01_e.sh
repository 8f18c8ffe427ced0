set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?"
timeout 600 python scripts/microbench.py --only attn --json gpurun_out/micro_v0.json > gpurun_out/micro_v0.log 2>&1
BS_ATTN_VARIANT=1 timeout 600 python scripts/microbench.py --only attn --json gpurun_out/micro_v1.json > gpurun_out/micro_v1.log 2>&1
echo "micro rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:split_decode -s 5 -c 1 -o gpurun_out/attn_c3 python scripts/microbench.py --only attn --case C3_gqa4_B8_8192 --iters 3 > gpurun_out/ncu_attn3.log 2>&1
echo "ncu rc=$?"
