# L2 prefetch ahead of the attention kernel's TMA ring: A/B over BS_ATTN_L2PF.
set -x
mkdir -p gpurun_out/l2pf
BS_ATTN_L2PF=4 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_ragged.py -q -x > gpurun_out/l2pf/pytest_pf4.log 2>&1
echo "pytest pf4 rc=$?"
for PF in 0 2 4 8; do
  BS_ATTN_L2PF=$PF timeout 600 python scripts/microbench.py --only attn --graph --json gpurun_out/l2pf/attn_graph_pf$PF.json > gpurun_out/l2pf/attn_graph_pf$PF.log 2>&1
  echo "graph pf$PF rc=$?"
  BS_ATTN_L2PF=$PF timeout 600 python scripts/microbench.py --only ragged --json gpurun_out/l2pf/ragged_pf$PF.json > gpurun_out/l2pf/ragged_pf$PF.log 2>&1
  echo "ragged pf$PF rc=$?"
  BS_ATTN_L2PF=$PF timeout 600 python bench.py --no-cpu-baseline --steps 10 > gpurun_out/l2pf/bench_pf$PF.json 2> gpurun_out/l2pf/bench_pf$PF.err
  echo "bench pf$PF rc=$?"
done
