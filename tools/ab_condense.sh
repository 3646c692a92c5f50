# A/B of the dense k_condense: tests, then configs 2, 5 (20 steps) and 3 (3 steps) bench lines.
# usage: bash tools/ab_condense.sh TAG [VARIANT...]   (VARIANT: fused | ws; default fused)
tag=${1:-x}; shift
vars=${@:-fused}
python -m pytest tests -m gpu -q -x > gpurun_out/r2_${tag}_tests.log 2>&1
for v in $vars; do
  for c in 2 5; do
    HOM_CONDENSE=$v python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline --spmv-nel 0 > gpurun_out/r2_${tag}_${v}_c$c.json 2>gpurun_out/r2_${tag}_${v}_c$c.err
  done
  HOM_CONDENSE=$v python bench.py --config 3 --steps 3 --warmup 3 --no-cpu-baseline --spmv-nel 0 --no-companions > gpurun_out/r2_${tag}_${v}_c3.json 2>gpurun_out/r2_${tag}_${v}_c3.err
done
