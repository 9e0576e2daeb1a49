# Round 2: NSA-style block selection on the OT kernel (BSEL): watchdog parity, full parity, bench, and a
# regression check of the default kernel after the template change.
mkdir -p gpurun_out
B() { python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }; }
SFA_NVCC_FLAGS="-DSFA_WATCHDOG" B
timeout 300 python -m pytest tests/test_gpu_blocksel.py -x -q -k "not qwen3" > gpurun_out/pytest_p_wd.log 2>&1; echo "pytest wd rc=$?"; tail -3 gpurun_out/pytest_p_wd.log; grep -m2 watchdog gpurun_out/pytest_p_wd.log
B
timeout 600 python -m pytest tests/test_gpu_blocksel.py tests/test_gpu_sm100.py tests/test_gpu_window.py tests/test_gpu_edges.py tests/test_gpu_fused_q.py -q > gpurun_out/pytest_p.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_p.log
for S in 4 16; do timeout 300 python bench.py --mode blocksel --blocks $S --steps 10 --warmup 3 > gpurun_out/bench_bsel_$S.json 2>gpurun_out/bench_bsel.err; echo "bsel $S rc=$?"; tail -c 700 gpurun_out/bench_bsel_$S.json; echo; done
timeout 120 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --no-long --no-dense-context > gpurun_out/bench_p.json 2>/dev/null; python -c "
import json; d=json.loads(open('gpurun_out/bench_p.json').read().strip().splitlines()[-1]); print('default', d['stage_ms'])"
