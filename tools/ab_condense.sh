set -x
python -m pytest tests -m gpu -q -x > gpurun_out/r2_ws_tests.log 2>&1
for v in ws fused; do
  for c in 2 5; do
    HOM_CONDENSE=$v python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline --spmv-nel 0 > gpurun_out/r2_ab_${v}_c$c.json 2>gpurun_out/r2_ab_${v}_c$c.err
  done
  HOM_CONDENSE=$v python bench.py --config 3 --steps 3 --warmup 3 --no-cpu-baseline --spmv-nel 0 --no-companions > gpurun_out/r2_ab_${v}_c3.json 2>gpurun_out/r2_ab_${v}_c3.err
done
