mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_sm100.py tests/test_gpu_bwd.py tests/test_gpu_window.py tests/test_gpu_edges.py -q -x > gpurun_out/pytest_sleep.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/pytest_sleep.log
for i in 1 2; do timeout 600 python bench.py --no-cpu-baseline --no-e2e --no-dense-context 2>/dev/null | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print("fwd", d["ms_per_step"], d["stage_ms"]["attn"], d["roofline"]["frac"])'; done
timeout 600 python bench.py --mode bwd 2>/dev/null | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print("bwd", d["ms_per_step"], d["roofline"]["frac"])'
SFA_NVCC_FLAGS="-DSFA_MBAR_SUSPEND_NS=0" python -m paper_2603_22300_b200.build --force > /dev/null 2>&1
for i in 1 2; do timeout 600 python bench.py --no-cpu-baseline --no-e2e --no-dense-context 2>/dev/null | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print("fwd hint0", d["ms_per_step"], d["stage_ms"]["attn"])'; done
