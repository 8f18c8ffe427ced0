# Bulk-TMA merge of many split-K partials by the last arriver: parity + A/B timing.
set -x
mkdir -p gpurun_out/bulkmerge
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/bulkmerge/pytest_gpu.log 2>&1
echo "pytest rc=$?"
timeout 600 python scripts/microbench.py --only attn --graph --json gpurun_out/bulkmerge/attn_graph.json > gpurun_out/bulkmerge/attn_graph.log 2>&1
echo "graph rc=$?"
timeout 600 python scripts/microbench.py --only attn --json gpurun_out/bulkmerge/attn.json > gpurun_out/bulkmerge/attn.log 2>&1
echo "attn rc=$?"
BS_TIMELINE=1 timeout 300 python scripts/attn_timeline.py --case C3_gqa4_B1_8192 --json gpurun_out/bulkmerge/timeline_b1.json > gpurun_out/bulkmerge/timeline_b1.log 2>&1
echo "timeline rc=$?"
timeout 600 python bench.py --no-cpu-baseline --steps 10 > gpurun_out/bulkmerge/bench.json 2> gpurun_out/bulkmerge/bench.err
echo "bench rc=$?"
