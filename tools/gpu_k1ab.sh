#!/bin/bash
# K1 compile-variant A/B: bash tools/gpu_k1ab.sh TAG "flags1" "flags2" ...  (each: HOM_NVCC_EXTRA)
TAG=$1; shift
mkdir -p gpurun_out
line() { python -c "
import json,sys;d=json.load(open(sys.argv[1]));a=d.get('assembly',{})
print(sys.argv[2], round(d['value'],1), round(d['roofline']['frac'],4), 'K1', round(a.get('ms_per_launch',0),4), round(a.get('GBps',0)))" "$1" "$2"; }
i=0
for fl in "$@"; do
  i=$((i+1))
  HOM_NVCC_EXTRA="$fl" python -c "from paper_2312_12771_b200 import build as b; b.build(force=True)" > gpurun_out/${TAG}_v${i}_build.log 2>&1 || { echo "build $fl failed"; continue; }
  for c in 4 2 5 3; do
    st=5; [ $c = 3 ] && st=2
    timeout 300 python bench.py --config $c --steps $st --warmup 3 --no-cpu-baseline --spmv-nel 0 --no-companions > gpurun_out/${TAG}_v${i}_c$c.json 2>/dev/null; line gpurun_out/${TAG}_v${i}_c$c.json "[$fl] c$c"
  done
done
