#!/bin/bash
# A/B of the diagonal lookahead (HOM_LA chunks per pivot-chain window) and the K1 stencil classes.
# usage: bash tools/gpu_ab_la.sh TAG "LA values" [tests]
TAG=${1:-la}; LAS=${2:-"0 6"}; TESTS=${3:-1}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${TAG}_build.log 2>&1 || { tail gpurun_out/${TAG}_build.log; exit 1; }
if [ "$TESTS" = "1" ]; then
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/${TAG}_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/${TAG}_tests.log
fi
for la in $LAS; do
  for c in 2 5 4; do
    HOM_LA=$la timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --spmv-nel 0 --no-companions > gpurun_out/${TAG}_la${la}_c$c.json 2>gpurun_out/${TAG}_la${la}_c$c.err
    python -c "
import json;d=json.load(open('gpurun_out/${TAG}_la${la}_c$c.json'));a=d.get('assembly',{})
print('la=$la c$c', round(d['value'],1), round(d['roofline']['frac'],4), 'K1', round(a.get('ms_per_launch',0),4), round(a.get('GBps',0)))"
  done
  HOM_LA=$la timeout 300 python bench.py --config 3 --steps 3 --warmup 3 --no-cpu-baseline --spmv-nel 0 --no-companions > gpurun_out/${TAG}_la${la}_c3.json 2>gpurun_out/${TAG}_la${la}_c3.err
  python -c "
import json;d=json.load(open('gpurun_out/${TAG}_la${la}_c3.json'));a=d.get('assembly',{})
print('la=$la c3', round(d['value'],1), round(d['roofline']['frac'],4), 'K1', round(a.get('ms_per_launch',0),4), round(a.get('GBps',0)))"
done
