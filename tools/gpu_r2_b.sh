# A/B of the OT kernel's P hand-off (SFA_OT_PHALF=1 halves vs 0 whole tile) + hand-off timelines of both.
mkdir -p gpurun_out
B() { python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }; }
BENCH="python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --no-long"
B
timeout 900 python -m pytest tests/test_gpu_sm100.py tests/test_gpu_attn.py tests/test_gpu_window.py tests/test_gpu_edges.py -x -q -m "gpu and not slow" > gpurun_out/pytest_b.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_b.log
for i in 1 2; do timeout 300 $BENCH > gpurun_out/bench_phalf1_$i.json 2>/dev/null; echo "phalf1 rc=$?"; done
SFA_NVCC_FLAGS="-DSFA_TIMELINE" B; timeout 300 python tools/timeline.py 32768 ot qwen > gpurun_out/timeline_phalf1.txt 2>&1; echo "tl1 rc=$?"
SFA_NVCC_FLAGS="-DSFA_OT_PHALF=0" B
for i in 1 2; do timeout 300 $BENCH > gpurun_out/bench_phalf0_$i.json 2>/dev/null; echo "phalf0 rc=$?"; done
SFA_NVCC_FLAGS="-DSFA_TIMELINE -DSFA_OT_PHALF=0" B; timeout 300 python tools/timeline.py 32768 ot qwen > gpurun_out/timeline_phalf0.txt 2>&1; echo "tl0 rc=$?"
B
