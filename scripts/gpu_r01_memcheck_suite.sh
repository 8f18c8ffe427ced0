# compute-sanitizer memcheck over the GPU parity suite (single-process tests; the
# multi-process IPC tests and the full-size / bench-size cases are skipped under the tool)
mkdir -p gpurun_out/sanitizer
timeout 2400 compute-sanitizer --tool memcheck --error-exitcode 9 --print-limit 50 \
  python -m pytest tests -m gpu -q -p no:cacheprovider \
  --deselect tests/test_gpu_ring_p2p.py --deselect tests/test_gpu_seqshard_p2p.py \
  -k "not full_size and not bench_step and not fuzz" \
  > gpurun_out/sanitizer/r01_memcheck_suite.log 2>&1
echo "memcheck suite rc=$?"
