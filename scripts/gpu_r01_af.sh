set -x
mkdir -p gpurun_out
for la in -1 -2 0; do
  BS_LOOKAHEAD=$la timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench_la$la.json 2> gpurun_out/bench_la$la.err
  echo "la $la rc=$?"
done
