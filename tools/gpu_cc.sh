python -m pytest tests/test_two_level_pcg.py -x -q 2>&1 | tail -3
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"cg_cluster2" --csv python tools/cg_scaling_probe.py 32 64 91 > gpurun_out/cc_ncu.csv 2>&1
python tools/cg_scaling_probe.py 32 64 91 128 | grep -v slices
