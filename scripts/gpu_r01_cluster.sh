# Cluster (DSMEM) pre-merge of split-K ranges: parity, sanitizer, A/B timing, timeline.
set -x
mkdir -p gpurun_out/cluster
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/cluster/pytest_gpu.log 2>&1
echo "pytest rc=$?"
timeout 900 compute-sanitizer --tool memcheck python -m pytest tests/test_gpu_parity.py -q -x -k "many_shards or llama3 or fused_local or full_size_c3" > gpurun_out/cluster/memcheck.log 2>&1
echo "memcheck rc=$?"
timeout 900 compute-sanitizer --tool racecheck python -m pytest tests/test_gpu_parity.py -q -x -k "many_shards" > gpurun_out/cluster/racecheck.log 2>&1
echo "racecheck rc=$?"
for C in 0 1; do
  BS_ATTN_CLUSTER=$C timeout 600 python scripts/microbench.py --only attn --graph --json gpurun_out/cluster/attn_graph_c$C.json > gpurun_out/cluster/attn_graph_c$C.log 2>&1
  echo "graph c$C rc=$?"
  BS_ATTN_CLUSTER=$C timeout 600 python scripts/microbench.py --only attn --json gpurun_out/cluster/attn_c$C.json > gpurun_out/cluster/attn_c$C.log 2>&1
  echo "attn c$C rc=$?"
  BS_ATTN_CLUSTER=$C BS_TIMELINE=1 timeout 300 python scripts/attn_timeline.py --case C3_gqa4_B1_8192 --json gpurun_out/cluster/timeline_b1_c$C.json > gpurun_out/cluster/timeline_b1_c$C.log 2>&1
  echo "timeline c$C rc=$?"
done
timeout 600 python bench.py --no-cpu-baseline --steps 10 > gpurun_out/cluster/bench.json 2> gpurun_out/cluster/bench.err
echo "bench rc=$?"
