#!/bin/bash
# One gpurun call: GPU tests, smoke, default bench, ncu launch list of the bench, ncu --set full of the top kernels.
# Usage (from repo root on the box): bash tools/gpu_check.sh TAG [CONFIG]
TAG=${1:-run}; CFG=${2:-2}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${TAG}_build.log 2>&1 || { echo build failed; tail gpurun_out/${TAG}_build.log; exit 1; }
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/${TAG}_gpu_tests.log 2>&1; echo "tests rc=$?"
tail -3 gpurun_out/${TAG}_gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/${TAG}_smoke.log
timeout 600 python bench.py --config $CFG > gpurun_out/${TAG}_bench_c${CFG}.json 2> gpurun_out/${TAG}_bench_c${CFG}.err; echo "bench rc=$?"
cat gpurun_out/${TAG}_bench_c${CFG}.json
if [ "${NO_NCU:-0}" = "0" ]; then
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/${TAG}_launches_c${CFG}.csv python bench.py --config $CFG --steps 2 --warmup 3 > gpurun_out/${TAG}_ncu_bench.log 2>&1; echo "ncu launches rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_condense -c 1 -o gpurun_out/${TAG}_condense_c${CFG} -f python tools/profile_step.py --config $CFG --steps 1 > gpurun_out/${TAG}_ncu_full.log 2>&1; echo "ncu full condense rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_rve_assemble -c 1 -o gpurun_out/${TAG}_assemble_c${CFG} -f python tools/profile_step.py --config $CFG --steps 1 > gpurun_out/${TAG}_ncu_full2.log 2>&1; echo "ncu full assemble rc=$?"
fi
