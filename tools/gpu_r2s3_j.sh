# GPT-2 shape on SM100_OT (d_v = 64 over the padded V copy): work order kv-group-major (default) vs global
# LPT (SFA_OT_ORDER=0), and one item per CTA; the SM100 (d_v = 64) default for reference
mkdir -p gpurun_out
run() { timeout -k 10 300 python bench.py --config gpt2 --kernel $1 --steps 30 --warmup 5 --no-cpu-baseline --no-e2e --no-dense-context 2>/dev/null | tail -1 | python -c "import json,sys;d=json.loads(sys.stdin.read());print('$2', d['ms_per_step'], d['stage_ms']['attn'])"; }
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
run auto sm100_default; run ot ot_order1
SFA_NVCC_FLAGS="-DSFA_OT_ORDER=0" python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
run ot ot_order0
SFA_NVCC_FLAGS="-DSFA_OT_ORDER=0 -DSFA_OT_ONE_ITEM_PER_CTA=1" python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
run ot ot_order0_oneitem
SFA_NVCC_FLAGS="-DSFA_OT_ORDER=1 -DSFA_OT_ONE_ITEM_PER_CTA=1" python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
run ot ot_order1_oneitem
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
