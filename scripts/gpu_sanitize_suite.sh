# compute-sanitizer memcheck over the single-process GPU suite (round 2 kernels: cluster
# merge, PDL late trigger, 6-stage ring, staged host tier).
mkdir -p gpurun_out/sansuite
timeout 3000 compute-sanitizer --tool memcheck --print-limit 20 --error-exitcode 9 \
  python -m pytest -q -x -p no:cacheprovider tests/test_gpu_parity.py tests/test_gpu_cluster.py tests/test_gpu_pdl.py \
  tests/test_gpu_ragged.py tests/test_gpu_tasks.py tests/test_gpu_append.py tests/test_gpu_headsplit.py \
  tests/test_gpu_kvstore.py tests/test_gpu_layer_migration.py tests/test_gpu_control.py tests/test_gpu_transport.py \
  -k "not subprocess and not deep_ring_variant and not sixteen_cta" > gpurun_out/sansuite/memcheck_suite.log 2>&1
echo "memcheck rc=$?"; tail -4 gpurun_out/sansuite/memcheck_suite.log
