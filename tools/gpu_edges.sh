set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_edges.py tests/test_gpu_bwd.py -q -x > gpurun_out/pytest_edges.log 2>&1; echo "edges+bwd rc=$?"; tail -15 gpurun_out/pytest_edges.log
timeout 600 python bench.py --no-cpu-baseline --no-e2e --edges-only > gpurun_out/bench_r2.json 2>&1; tail -1 gpurun_out/bench_r2.json
timeout 600 python bench.py --no-cpu-baseline --no-e2e --edges-only --config sweep --k 4 > gpurun_out/bench_r2_k4.json 2>&1; tail -1 gpurun_out/bench_r2_k4.json
timeout 600 python bench.py --mode bwd > gpurun_out/bench_bwd.json 2>&1; tail -1 gpurun_out/bench_bwd.json
