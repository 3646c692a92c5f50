#!/bin/bash
# The GPU suite on a bounds-checked build (-DHOM_DEBUG_BOUNDS: device-side checks of the K1 tables, record
# indices and pool slots trap on a violation) -- the substitute for compute-sanitizer, closed on this pool.
mkdir -p gpurun_out
HOM_NVCC_EXTRA=-DHOM_DEBUG_BOUNDS python -c "from paper_2312_12771_b200 import build as b; b.build(force=True)" > gpurun_out/dbg_build.log 2>&1 || { tail gpurun_out/dbg_build.log; exit 1; }
python -c "import oracle; oracle.build(force=True)" > /dev/null 2>&1
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/dbg_tests.log 2>&1; echo "bounds-checked GPU suite rc=$?"; tail -2 gpurun_out/dbg_tests.log
strings paper_2312_12771_b200/libhom.so | grep -c "HOM_DCHECK" | sed "s/^/HOM_DCHECK strings in the checked libhom.so: /"
for c in 2 3 4 5; do timeout 300 python bench.py --config $c --steps 2 --warmup 3 --no-cpu-baseline --spmv-nel 0 --no-companions > /dev/null 2> gpurun_out/dbg_c$c.err; echo "bounds-checked bench c$c rc=$?"; done
timeout 300 python bench.py --config 3 --steps 2 --warmup 3 --no-cpu-baseline --spmv-nel 0 --no-companions --tile-sparse > /dev/null 2> gpurun_out/dbg_c3ts.err; echo "bounds-checked bench c3 tile-sparse rc=$?"
