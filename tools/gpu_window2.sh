mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_window.py tests/test_gpu_edges.py tests/test_gpu_fused_q.py tests/test_gpu_sm100.py -q -x > gpurun_out/pytest_window.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/pytest_window.log
for i in 1 2; do timeout 600 python bench.py --no-cpu-baseline --no-e2e --no-dense-context 2>/dev/null | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print("default", d["ms_per_step"], d["stage_ms"]["attn"], d["roofline"]["frac"])'; done
timeout 300 python bench.py --no-cpu-baseline --no-e2e --window 4096 2>/dev/null | tail -1 > gpurun_out/bench_window_4096.json; tail -1 gpurun_out/bench_window_4096.json | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print("w4096", d["ms_per_step"], d["stage_ms"]["attn"], d["roofline"]["frac"])'
