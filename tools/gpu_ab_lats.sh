#!/bin/bash
# A/B of the tile-sparse diagonal lookahead (HOM_LA chunks per pivot-chain window; 0 = off).
TAG=${1:-lats}; LAS=${2:-"0 2 4 8"}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${TAG}_build.log 2>&1 || { tail gpurun_out/${TAG}_build.log; exit 1; }
for la in $LAS; do
  HOM_LA=$la timeout 900 python -m pytest tests -m gpu -q -x -k "tile_sparse or config5 or cook_table1_gen" > gpurun_out/${TAG}_la${la}_tests.log 2>&1; echo "la=$la tests rc=$?"; tail -1 gpurun_out/${TAG}_la${la}_tests.log
  for c in 2 5 4; do
    HOM_LA=$la timeout 300 python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline --spmv-nel 0 --no-companions --tile-sparse > gpurun_out/${TAG}_la${la}_c$c.json 2>/dev/null
    python -c "
import json;d=json.load(open('gpurun_out/${TAG}_la${la}_c$c.json'));b=d['breakdown']['condense']
print('la=$la c$c', '%.4g'%d['value'], round(d['roofline']['frac'],4), 'condense ms', round(b['ms_per_step'],4))"
  done
  HOM_LA=$la timeout 300 python bench.py --config 3 --steps 5 --warmup 3 --no-cpu-baseline --spmv-nel 0 --no-companions --tile-sparse > gpurun_out/${TAG}_la${la}_c3.json 2>/dev/null
  python -c "
import json;d=json.load(open('gpurun_out/${TAG}_la${la}_c3.json'));b=d['breakdown']['condense']
print('la=$la c3', '%.4g'%d['value'], round(d['roofline']['frac'],4), 'condense ms', round(b['ms_per_step'],4))"
done
