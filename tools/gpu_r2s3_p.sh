# A/B of the exp2 split (SFA_OT_POLY = pairs of 8 on the FMA pipe) on the current OT kernel, Qwen3-32K
mkdir -p gpurun_out
run() { for i in 1 2 3; do timeout -k 10 300 python bench.py --no-cpu-baseline --no-e2e --no-long --no-dense-context 2>/dev/null | tail -1 | python -c "import json,sys;d=json.loads(sys.stdin.read());print('$1', round(d['stage_ms']['attn'],4))"; done; }
for P in 2 3 1 2 3; do
  SFA_NVCC_FLAGS="-DSFA_OT_POLY=$P" python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
  run poly$P
done
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
