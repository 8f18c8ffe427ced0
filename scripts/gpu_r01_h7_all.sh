# H7 in the default step at every N: full GPU suite, bench N=1 (with and without H7),
# N=2 functional (two ranks on one GPU), reference arm.
set -x
mkdir -p gpurun_out/h7
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/h7/smoke.log 2>&1
echo "smoke rc=$?"
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/h7/pytest_gpu.log 2>&1
echo "pytest rc=$?"
for i in 1 2; do
  timeout 600 python bench.py > gpurun_out/h7/bench_$i.json 2> gpurun_out/h7/bench_$i.err
  echo "bench $i rc=$?"
  BS_BENCH_APPEND=0 timeout 600 python bench.py --no-cpu-baseline > gpurun_out/h7/bench_noapp_$i.json 2> gpurun_out/h7/bench_noapp_$i.err
  echo "bench noapp $i rc=$?"
done
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/h7/bench_reference.json 2> gpurun_out/h7/bench_reference.err
echo "reference rc=$?"
BS_RING_SAME_GPU=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/h7/bench_n2.json 2> gpurun_out/h7/bench_n2.err
echo "n2 rc=$?"
