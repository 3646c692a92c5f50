#!/bin/bash
# bench several configs in one gpurun call: bash tools/bench_sweep.sh TAG "2 3 4" [extra bench args]
TAG=$1; CFGS=$2; shift 2
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${TAG}_build.log 2>&1 || { echo build failed; exit 1; }
for c in $CFGS; do
  timeout 900 python bench.py --config $c --no-cpu-baseline "$@" > gpurun_out/${TAG}_c$c.json 2> gpurun_out/${TAG}_c$c.err
  echo "cfg $c rc=$?"
  python - "$c" "gpurun_out/${TAG}_c$c.json" <<'PY'
import json, sys
d = json.load(open(sys.argv[2]))
b = {k: round(v["ms_per_step"], 3) for k, v in d["breakdown"].items()}
print(sys.argv[1], d["config"]["factorization"], "tangents/s %.1f" % d["value"], "ms/step %.3f" % d["ms_per_step"],
      "frac %.3f" % d["roofline"]["frac"], "K1 GB/s %.0f" % d["assembly"]["GBps"], b)
PY
done
