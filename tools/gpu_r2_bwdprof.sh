set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_edges.py -q -x > gpurun_out/pytest_edges.log 2>&1; echo "edges rc=$?"; tail -3 gpurun_out/pytest_edges.log
timeout 600 python bench.py --no-cpu-baseline --no-e2e --edges-only > gpurun_out/bench_r2.json 2>&1; tail -1 gpurun_out/bench_r2.json
timeout 600 python bench.py --no-cpu-baseline --no-e2e --edges-only --config sweep --k 4 > gpurun_out/bench_r2_k4.json 2>&1; tail -1 gpurun_out/bench_r2_k4.json
timeout 900 ncu --set full --import-source on --clock-control none -k regex:bwd_dkdv -s 1 -c 1 -o gpurun_out/bwd_dkdv -f python bench.py --mode bwd --steps 1 --warmup 1 > gpurun_out/ncu_dkdv.log 2>&1; echo "ncu dkdv rc=$?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:bwd_dq -s 1 -c 1 -o gpurun_out/bwd_dq -f python bench.py --mode bwd --steps 1 --warmup 1 > gpurun_out/ncu_dq.log 2>&1; echo "ncu dq rc=$?"
