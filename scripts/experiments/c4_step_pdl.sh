mkdir -p gpurun_out/c4
timeout 600 python -m pytest tests/test_gpu_ragged.py -q -x > gpurun_out/c4/pytest_ragged.log 2>&1
echo "ragged tests rc=$?"; tail -1 gpurun_out/c4/pytest_ragged.log
for r in 1 2; do for pdl in 0 default; do
  if [ $pdl = 0 ]; then export BS_ATTN_PDL=0; else unset BS_ATTN_PDL; fi
  timeout 600 python scripts/bench_c4.py --seed 0 --steps 10 > gpurun_out/c4/c4_pdl${pdl}_r$r.json 2> gpurun_out/c4/c4_pdl${pdl}_r$r.err
  echo "c4 pdl=$pdl rc=$?"
done; done
