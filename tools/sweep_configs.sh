# One bench line per config and factorisation (dense / tile-sparse) for BASELINE.md §5.
# usage: bash tools/sweep_configs.sh TAG
tag=${1:-r02}
for c in 1 2 4 5; do
  for ts in "" "--tile-sparse"; do
    n=$([ -z "$ts" ] && echo dense || echo tilesparse)
    python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline --spmv-nel 0 --no-companions $ts \
      > gpurun_out/${tag}_${n}_c$c.json 2> gpurun_out/${tag}_${n}_c$c.err
  done
done
python bench.py --config 3 --steps 3 --warmup 3 --no-cpu-baseline --spmv-nel 0 --no-companions --tile-sparse \
  > gpurun_out/${tag}_tilesparse_c3.json 2> gpurun_out/${tag}_tilesparse_c3.err
python bench.py --config 2 --steps 20 --warmup 3 --no-cpu-baseline --spmv-nel 0 --no-companions --macro-basis constant \
  > gpurun_out/${tag}_constant_c2.json 2> gpurun_out/${tag}_constant_c2.err
