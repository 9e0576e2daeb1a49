mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_topk.py tests/test_gpu_fused_q.py -q -x > gpurun_out/pytest_topk.log 2>&1; echo "topk rc=$?"; tail -2 gpurun_out/pytest_topk.log
for i in 1 2; do timeout 600 python bench.py --no-cpu-baseline --no-e2e --no-dense-context 2>/dev/null | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print("default", d["ms_per_step"], d["stage_ms"], d["roofline"]["other_floors"]["topk_hbm_frac"])'; done
timeout 600 python bench.py --config gpt2 --no-cpu-baseline --no-e2e --no-dense-context 2>/dev/null | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print("gpt2", d["ms_per_step"], d["stage_ms"])'
