mkdir -p gpurun_out/exp4
for pdl in 1 0 1 0; do
  BS_ATTN_PDL=$pdl timeout 600 python scripts/exp_e2e.py --steps 20 > gpurun_out/exp4/e2e_pdl$pdl.$RANDOM.json 2>&1
done
nvidia-smi -q -d CLOCK,PERFORMANCE | head -60 > gpurun_out/exp4/clocks.txt
