#!/bin/bash
# Launch list + ncu --set full of the top kernels for a config: bash tools/profile_round.sh TAG CFG [extra bench args]
TAG=$1; CFG=$2; shift 2
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${TAG}_build.log 2>&1 || exit 1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/${TAG}_launches_c${CFG}.csv \
  python bench.py --config $CFG --steps 2 --warmup 3 --no-cpu-baseline --spmv-nel 0 "$@" > gpurun_out/${TAG}_ncu_bench.log 2>&1
echo "launches rc=$?"
for K in k_condense k_rve_assemble k_macro_cg_cluster2; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$K -c 1 -o gpurun_out/${TAG}_${K}_c${CFG} -f \
    python tools/profile_step.py --config $CFG --steps 1 "$@" > gpurun_out/${TAG}_${K}.log 2>&1
  echo "$K rc=$?"
done
