# Same-GPU functional runs of the N>1 bench paths (numbers meaningless: ranks time-slice GPU 0).
mkdir -p gpurun_out/multi
BS_RING_SAME_GPU=1 timeout 1200 python bench.py --gpus 2 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/multi/n2_auto.json 2> gpurun_out/multi/n2_auto.err
echo "n2 auto rc=$?"
BS_RING_SAME_GPU=1 timeout 1200 python bench.py --gpus 4 --steps 3 --warmup 3 --no-cpu-baseline --config c3 > gpurun_out/multi/n4_c3.json 2> gpurun_out/multi/n4_c3.err
echo "n4 c3 rc=$?"
timeout 300 python bench.py --gpus 2 --steps 3 --warmup 3 > gpurun_out/multi/n2_no_same_gpu.json 2> gpurun_out/multi/n2_no_same_gpu.err
echo "n2 on 1 gpu rc=$?"
