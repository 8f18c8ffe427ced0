set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?"
for pdl in 1 0; do
  BS_PDL=$pdl timeout 600 python scripts/microbench.py --only attn --graph --json gpurun_out/mb_graph_pdl$pdl.json > gpurun_out/mb_graph_pdl$pdl.log 2>&1
  echo "graph pdl=$pdl rc=$?"
  BS_PDL=$pdl timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_pdl$pdl.json 2> gpurun_out/bench_pdl$pdl.err
  echo "bench pdl=$pdl rc=$?"
done
BS_PDL=1 timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_pdl1b.json 2> gpurun_out/bench_pdl1b.err
