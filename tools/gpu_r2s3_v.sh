# the full GPU suite and smoke on HEAD
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout -k 10 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_head.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_head.log
timeout -k 10 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_head.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke_head.log
