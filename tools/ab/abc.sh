mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/abc_build.log 2>&1
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/abc_tests.log 2>&1; echo "tests rc=$?"; tail -1 gpurun_out/abc_tests.log
bash tools/ab_condense_file.sh abc tools/ab/condense_lats.cu
