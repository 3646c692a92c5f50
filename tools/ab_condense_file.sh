#!/bin/bash
# A/B of two condense.cu sources on one box: bash tools/ab_condense_file.sh TAG ALT_SOURCE
TAG=$1; ALT=$2
mkdir -p gpurun_out
cp paper_2312_12771_b200/csrc/condense.cu /tmp/condense_orig.cu
run() {
  python -c "from paper_2312_12771_b200 import build as b; b.build(force=True)" > gpurun_out/${TAG}_$1_build.log 2>&1 || { echo build $1 failed; return; }
  for c in 3 2; do
    st=20; [ $c = 3 ] && st=5
    for ts in "--tile-sparse" ""; do
      timeout 300 python bench.py --config $c --steps $st --warmup 3 --no-cpu-baseline --spmv-nel 0 --no-companions $ts > gpurun_out/${TAG}_$1_c$c$ts.json 2>/dev/null
      python -c "
import json;d=json.load(open('gpurun_out/${TAG}_$1_c$c$ts.json'));b=d['breakdown']['condense']
print('$1 c$c $ts', '%.4g'%d['value'], round(d['roofline']['frac'],4), 'condense ms', round(b['ms_per_step'],3))"
    done
  done
}
for rep in 1 2; do
  cp /tmp/condense_orig.cu paper_2312_12771_b200/csrc/condense.cu; run A$rep
  cp $ALT paper_2312_12771_b200/csrc/condense.cu; run B$rep
done
cp /tmp/condense_orig.cu paper_2312_12771_b200/csrc/condense.cu
