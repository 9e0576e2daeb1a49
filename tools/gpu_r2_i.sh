# Round 2: full GPU suite on the K~-TMA build + OT flag sweep (poly split, P hand-off) with K~ by TMA.
mkdir -p gpurun_out
B() { python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }; }
B
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_i.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_i.log
BENCH="python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --no-long --no-dense-context"
for v in "" "-DSFA_OT_POLY=1" "-DSFA_OT_POLY=3" "-DSFA_OT_PHALF=1"; do SFA_NVCC_FLAGS="$v" B; timeout 120 $BENCH > gpurun_out/bench_i.json 2>/dev/null; python -c "
import json; d=json.loads(open('gpurun_out/bench_i.json').read().strip().splitlines()[-1]); print('ot [$v]', round(d['stage_ms']['attn'],3), d['clocks']['sm_mhz'])"; done
B
