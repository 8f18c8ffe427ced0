# Persistent attention kernel: correctness (pytest -m gpu with the default = persistent)
# and A/B against the one-CTA-per-unit launch (BS_ATTN_PERSIST=0).
set -x
mkdir -p gpurun_out/persist
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/persist/smoke.log 2>&1
echo "smoke rc=$?"
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/persist/pytest_gpu.log 2>&1
echo "pytest rc=$?"
for P in 0 1; do
  BS_ATTN_PERSIST=$P timeout 600 python scripts/microbench.py --only attn --json gpurun_out/persist/attn_p$P.json > gpurun_out/persist/attn_p$P.log 2>&1
  echo "attn p$P rc=$?"
  BS_ATTN_PERSIST=$P timeout 600 python scripts/microbench.py --only attn --graph --json gpurun_out/persist/attn_graph_p$P.json > gpurun_out/persist/attn_graph_p$P.log 2>&1
  echo "attn graph p$P rc=$?"
  BS_ATTN_PERSIST=$P timeout 600 python scripts/microbench.py --only ragged --json gpurun_out/persist/ragged_p$P.json > gpurun_out/persist/ragged_p$P.log 2>&1
  echo "ragged p$P rc=$?"
  BS_ATTN_PERSIST=$P timeout 600 python bench.py --no-cpu-baseline > gpurun_out/persist/bench_p$P.json 2> gpurun_out/persist/bench_p$P.err
  echo "bench p$P rc=$?"
done
