#!/bin/bash
# A/B: L2 prefetch of the next A tiles in k_condense (HOM_PF) and K1 stencil classes (HOM_K1_CLS), + K1 ncu.
TAG=${1:-pf}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${TAG}_build.log 2>&1 || { tail gpurun_out/${TAG}_build.log; exit 1; }
line() { python -c "
import json,sys;d=json.load(open(sys.argv[1]));a=d.get('assembly',{})
print(sys.argv[2], round(d['value'],1), round(d['roofline']['frac'],4), 'K1', round(a.get('ms_per_launch',0),4), round(a.get('GBps',0)))" "$1" "$2"; }
for pf in 0 1 2 0; do
  for c in 2 5; do
    HOM_PF=$pf timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --spmv-nel 0 --no-companions > gpurun_out/${TAG}_pf${pf}_c$c.json 2>/dev/null; line gpurun_out/${TAG}_pf${pf}_c$c.json "pf=$pf c$c"
  done
done
for pf in 0 1; do
  HOM_PF=$pf timeout 300 python bench.py --config 3 --steps 3 --warmup 3 --no-cpu-baseline --spmv-nel 0 --no-companions > gpurun_out/${TAG}_pf${pf}_c3.json 2>/dev/null; line gpurun_out/${TAG}_pf${pf}_c3.json "pf=$pf c3"
done
for cls in 0 1 0 1; do
  HOM_K1_CLS=$cls timeout 300 python bench.py --config 4 --steps 5 --warmup 3 --no-cpu-baseline --spmv-nel 0 --no-companions > gpurun_out/${TAG}_cls${cls}_c4.json 2>/dev/null; line gpurun_out/${TAG}_cls${cls}_c4.json "cls=$cls c4"
done
for cls in 0 1; do
  HOM_K1_CLS=$cls timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_rve_assemble -c 1 -o gpurun_out/${TAG}_k1_c4_cls$cls -f python tools/profile_step.py --config 4 --steps 1 > gpurun_out/${TAG}_ncu_k1_cls$cls.log 2>&1; echo "ncu cls=$cls rc=$?"
done
