#!/bin/bash
# K1 check: GPU tests, K1 timings on configs 2-5, ncu --set full of K1 at configs 4 and 5.
TAG=${1:-k1}; TESTS=${2:-1}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${TAG}_build.log 2>&1 || { tail gpurun_out/${TAG}_build.log; exit 1; }
if [ "$TESTS" = "1" ]; then
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/${TAG}_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/${TAG}_tests.log
fi
line() { python -c "
import json,sys;d=json.load(open(sys.argv[1]));a=d.get('assembly',{})
print(sys.argv[2], round(d['value'],1), round(d['roofline']['frac'],4), 'K1', round(a.get('ms_per_launch',0),4), round(a.get('GBps',0)))" "$1" "$2"; }
for c in 2 4 5 3; do
  st=10; [ $c = 3 ] && st=3
  timeout 300 python bench.py --config $c --steps $st --warmup 3 --no-cpu-baseline --spmv-nel 0 --no-companions > gpurun_out/${TAG}_c$c.json 2>/dev/null; line gpurun_out/${TAG}_c$c.json "c$c"
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_rve_assemble -c 1 -o gpurun_out/${TAG}_k1_c4 -f python tools/profile_step.py --config 4 --steps 1 > gpurun_out/${TAG}_ncu_k1_c4.log 2>&1; echo "ncu c4 rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_rve_assemble_fs -s 1 -c 1 -o gpurun_out/${TAG}_k1_c5 -f python tools/profile_cfg5.py > gpurun_out/${TAG}_ncu_k1_c5.log 2>&1; echo "ncu c5 rc=$?"
