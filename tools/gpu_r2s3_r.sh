# OT with per-tile P.V (SFA_OT_SPLITPV=1): parity, then A/B against the default at Qwen3-32K
mkdir -p gpurun_out
run() { for i in 1 2 3; do timeout -k 10 300 python bench.py --no-cpu-baseline --no-e2e --no-long --no-dense-context 2>/dev/null | tail -1 | python -c "import json,sys;d=json.loads(sys.stdin.read());print('$1', round(d['stage_ms']['attn'],4))"; done; }
SFA_NVCC_FLAGS="-DSFA_OT_SPLITPV=1" python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout -k 10 600 python -m pytest tests/test_gpu_sm100.py tests/test_gpu_window.py tests/test_gpu_blocksel.py tests/test_gpu_repeat.py -q -x -k "not pp and not oth" -p no:cacheprovider > gpurun_out/pytest_r.log 2>&1; rc=$?; echo "pytest rc=$rc"; tail -3 gpurun_out/pytest_r.log
[ $rc -eq 0 ] || { python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; exit 1; }
run split; 
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
run base
SFA_NVCC_FLAGS="-DSFA_OT_SPLITPV=1" python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
run split
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
run base
