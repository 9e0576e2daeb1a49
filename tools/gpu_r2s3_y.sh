# careful A/B of SFA_OT_POLY 1 vs 2 (interleaved builds, 4 runs each, 3 rounds), Qwen3-32K attention
mkdir -p gpurun_out
run() { for i in 1 2 3 4; do timeout -k 10 300 python bench.py --no-cpu-baseline --no-e2e --no-long --no-dense-context 2>/dev/null | tail -1 | python -c "import json,sys;d=json.loads(sys.stdin.read());print('$1', round(d['stage_ms']['attn'],4), d['clocks']['sm_mhz'])"; done; }
for rnd in 1 2 3; do
  for P in 1 2; do
    SFA_NVCC_FLAGS="-DSFA_OT_POLY=$P" python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
    run poly$P
  done
done
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
