set -x
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_ring_p2p.py -m gpu -x -q > gpurun_out/pytest_p2p.log 2>&1
echo "p2p rc=$?"
BS_RING_SAME_GPU=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 3 --warmup 3 > gpurun_out/bench_n2_samegpu.json 2> gpurun_out/bench_n2_samegpu.err
echo "bench n2 rc=$?"
