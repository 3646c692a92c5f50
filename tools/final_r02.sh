#!/bin/bash
# Round-2 final evidence: GPU suite, smoke, default bench line, reference arm, full-size parity,
# launch list of the default bench.  Output in gpurun_out/final_*.
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/final_build.log 2>&1 || exit 1
python -m pytest tests -m gpu -q > gpurun_out/final_gpu_tests.log 2>&1; echo "gpu tests rc=$?"
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/final_smoke.log 2>&1; echo "smoke rc=$?"
python bench.py > gpurun_out/final_bench.json 2> gpurun_out/final_bench.err; echo "bench rc=$?"
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/final_reference.json 2> gpurun_out/final_reference.err; echo "reference rc=$?"
python tools/parity_report.py > gpurun_out/final_parity.txt 2> gpurun_out/final_parity.err; echo "parity rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/final_launches_c3.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline --spmv-nel 0 --no-companions > gpurun_out/final_ncu_bench.log 2>&1; echo "launches rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_rve_assemble -c 1 -o gpurun_out/final_k1_c3 -f python tools/profile_step.py --config 3 --steps 1 > gpurun_out/final_ncu_k1_c3.log 2>&1; echo "ncu k1 c3 rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_rve_assemble -c 1 -o gpurun_out/final_k1_c4 -f python tools/profile_step.py --config 4 --steps 1 > gpurun_out/final_ncu_k1_c4.log 2>&1; echo "ncu k1 c4 rc=$?"
