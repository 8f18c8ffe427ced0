set -x
mkdir -p gpurun_out
for c in C3_gqa4_B1_8192 C3_gqa4_B8_8192; do
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:split_decode -s 5 -c 1 -o gpurun_out/ncu_$c -f python scripts/microbench.py --only attn --case $c --iters 3 > gpurun_out/ncu_$c.log 2>&1
  echo "$c rc=$?"
done
