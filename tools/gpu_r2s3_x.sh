# GPT-2 shape: SM100 (AUTO) vs SM100_OT with global-LPT work order, after the OT epilogue change
mkdir -p gpurun_out
run() { for i in 1 2 3; do timeout -k 10 300 python bench.py --config gpt2 --kernel $1 --steps 30 --warmup 5 --no-cpu-baseline --no-e2e --no-dense-context 2>/dev/null | tail -1 | python -c "import json,sys;d=json.loads(sys.stdin.read());print('$2', round(d['ms_per_step'],4), round(d['stage_ms']['attn'],4))"; done; }
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
run auto sm100; run ot ot_order1
SFA_NVCC_FLAGS="-DSFA_OT_ORDER=0" python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
run ot ot_order0
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
