# Round 2: 16-softmax-warp ping-pong kernel: watchdog parity, bench vs OT, timeline, poly variants.
mkdir -p gpurun_out
B() { python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }; }
SFA_NVCC_FLAGS="-DSFA_WATCHDOG" B
timeout 120 python -m pytest tests/test_gpu_sm100.py -x -q -k "pp" > gpurun_out/pytest_h_wd.log 2>&1; echo "pytest wd rc=$?"; tail -5 gpurun_out/pytest_h_wd.log
B
BENCH="python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --no-long --no-dense-context"
for kn in pp ot pp; do timeout 120 $BENCH --kernel $kn > gpurun_out/bench_h_$kn.json 2>/dev/null; echo "bench $kn rc=$?"; python -c "
import json; d=json.loads(open('gpurun_out/bench_h_$kn.json').read().strip().splitlines()[-1]); print('$kn', round(d['stage_ms']['attn'],3), d['clocks']['sm_mhz'])"; done
SFA_NVCC_FLAGS="-DSFA_TIMELINE" B; timeout 120 python tools/timeline.py 32768 pp qwen > gpurun_out/timeline_pp16.txt 2>&1; echo "tl rc=$?"
for v in "-DSFA_PP_POLY=3" "-DSFA_PP_POLY=1" "-DSFA_PP_PINGPONG=0"; do SFA_NVCC_FLAGS="$v" B; timeout 120 $BENCH --kernel pp > gpurun_out/bench_h_v.json 2>/dev/null; python -c "
import json; d=json.loads(open('gpurun_out/bench_h_v.json').read().strip().splitlines()[-1]); print('$v', round(d['stage_ms']['attn'],3), d['clocks']['sm_mhz'])"; done
B
