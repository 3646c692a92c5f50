mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/b_build.log 2>&1 || { tail gpurun_out/b_build.log; exit 1; }
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/b_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/b_tests.log
for c in 2 4 5; do timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --spmv-nel 0 --no-companions > gpurun_out/b_c$c.json 2>gpurun_out/b_c$c.err; echo "c$c rc=$?"; done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_rve_assemble -c 1 -o gpurun_out/b_k1_c4 -f python tools/profile_step.py --config 4 --steps 1 > gpurun_out/b_ncu_k1.log 2>&1; echo "ncu rc=$?"
