mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -q -k "remote_view or migration" > gpurun_out/pytest_remote.log 2>&1
echo "remote rc=$?"
timeout 900 python -m pytest tests/test_gpu_ring_p2p.py tests/test_gpu_seqshard_p2p.py -q > gpurun_out/pytest_p2p.log 2>&1
echo "p2p rc=$?"
