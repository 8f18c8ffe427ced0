# Full GPU suite + default bench + microbench (graph) of every attention case.
mkdir -p gpurun_out/check2
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/check2/smoke.log 2>&1
echo "smoke rc=$?"
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/check2/pytest_gpu.log 2>&1
echo "pytest rc=$?"; tail -2 gpurun_out/check2/pytest_gpu.log
for i in 1 2; do
timeout 900 python bench.py > gpurun_out/check2/bench_$i.json 2> gpurun_out/check2/bench_$i.err
echo "bench rc=$?"
done
timeout 600 python scripts/microbench.py --only attn --graph > gpurun_out/check2/microbench_graph.jsonl 2>/dev/null
echo "mb rc=$?"
