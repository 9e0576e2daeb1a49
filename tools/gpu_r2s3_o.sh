# OT epilogue with fewer instructions per element: parity (OT / edges / window / blocksel / fused-Q / attn),
# then Qwen3 step, block selection (4 and 16 blocks), GPT-2 on OT
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout -k 10 1200 python -m pytest tests/test_gpu_sm100.py tests/test_gpu_edges.py tests/test_gpu_window.py tests/test_gpu_blocksel.py tests/test_gpu_fused_q.py tests/test_gpu_attn.py tests/test_gpu_repeat.py -q -x -p no:cacheprovider > gpurun_out/pytest_o.log 2>&1; rc=$?; echo "pytest rc=$rc"; tail -2 gpurun_out/pytest_o.log
[ $rc -eq 0 ] || exit 1
for i in 1 2; do timeout -k 10 300 python bench.py --no-cpu-baseline --no-e2e --no-long --no-dense-context 2>/dev/null | tail -1 | python -c "import json,sys;d=json.loads(sys.stdin.read());print('qwen3', d['ms_per_step'], d['stage_ms']['attn'])"; done
for nb in 4 16; do timeout -k 10 300 python bench.py --mode blocksel --blocks $nb --steps 10 --warmup 3 2>/dev/null | tail -1 > gpurun_out/bench_bsel_$nb.json; python -c "import json;d=json.loads(open('gpurun_out/bench_bsel_$nb.json').read());print('blocksel $nb', d['ms_per_step'], d['stage_ms'])"; done
timeout -k 10 300 python bench.py --config gpt2 --kernel ot --steps 30 --warmup 5 --no-cpu-baseline --no-e2e --no-dense-context 2>/dev/null | tail -1 | python -c "import json,sys;d=json.loads(sys.stdin.read());print('gpt2 ot', d['ms_per_step'], d['stage_ms']['attn'])"
