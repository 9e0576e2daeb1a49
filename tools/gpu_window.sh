mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_window.py -q -x > gpurun_out/pytest_window.log 2>&1; echo "window rc=$?"; tail -3 gpurun_out/pytest_window.log
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu.log
for w in 4096 1024; do timeout 300 python bench.py --no-cpu-baseline --no-e2e --window $w 2>/dev/null | tail -1 > gpurun_out/bench_window_$w.json; tail -1 gpurun_out/bench_window_$w.json | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print("w", d["ms_per_step"], d["stage_ms"], d["roofline"]["frac"], d["pairs_per_s"])'; done
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -1 gpurun_out/bench.json | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print("default", d["ms_per_step"], d["stage_ms"], d["roofline"]["frac"], d["e2e"]["value"])'
