mkdir -p gpurun_out
for v in 0 2; do BS_ATTN_VARIANT=$v timeout 600 python scripts/microbench.py --only attn --graph > gpurun_out/mb_graph_v$v.log 2>&1; done
BS_ATTN_VARIANT=0 timeout 600 python scripts/microbench.py --only attn --graph > gpurun_out/mb_graph_v0b.log 2>&1
echo done
