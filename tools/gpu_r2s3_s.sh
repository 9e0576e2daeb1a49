# seeded random-shape sweep of the forward kernels against the oracle
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout -k 10 900 python -m pytest tests/test_gpu_fuzz.py -q -p no:cacheprovider > gpurun_out/pytest_s.log 2>&1; echo "pytest rc=$?"; tail -15 gpurun_out/pytest_s.log
