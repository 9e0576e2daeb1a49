# Round 2: ping-pong kernel variants (ring depths, ping-pong on/off, poly split) + hand-off timelines.
mkdir -p gpurun_out
B() { python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }; }
BENCH="python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --no-long --no-dense-context --kernel pp"
run() {  # $1 = tag, $2 = flags
  SFA_NVCC_FLAGS="$2" B
  timeout 200 python -m pytest tests/test_gpu_sm100.py -x -q -k "pp and against" > gpurun_out/pytest_g_$1.log 2>&1; echo "$1 pytest rc=$?"
  timeout 300 $BENCH > gpurun_out/bench_g_$1.json 2>/dev/null; python -c "
import json; d=json.loads(open('gpurun_out/bench_g_$1.json').read().strip().splitlines()[-1]); print('$1', round(d['stage_ms']['attn'],3), d['clocks']['sm_mhz'])"
}
run base ""
run nopp "-DSFA_PP_PINGPONG=0"
run nk3 "-DSFA_PP_NK=3"
run nv3 "-DSFA_PP_NV=3"
run poly3 "-DSFA_PP_POLY=3"
run poly0 "-DSFA_PP_POLY=0"
SFA_NVCC_FLAGS="-DSFA_TIMELINE" B; timeout 300 python tools/timeline.py 32768 pp qwen > gpurun_out/timeline_pp.txt 2>&1; echo "tl rc=$?"
SFA_NVCC_FLAGS="-DSFA_TIMELINE -DSFA_PP_PINGPONG=0" B; timeout 300 python tools/timeline.py 32768 pp qwen > gpurun_out/timeline_pp_nopp.txt 2>&1; echo "tl2 rc=$?"
B
timeout 900 ncu --set full --import-source on --clock-control none -k regex:attn_sm100_pp -s 1 -c 1 -o gpurun_out/pp_g -f python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-long --no-dense-context --kernel pp > gpurun_out/ncu_pp.log 2>&1; echo "ncu rc=$?"
