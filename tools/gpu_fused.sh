mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_fused_q.py tests/test_gpu_topk.py tests/test_gpu_attn.py -q -x > gpurun_out/pytest_fused.log 2>&1; echo "fused rc=$?"; tail -3 gpurun_out/pytest_fused.log
timeout 600 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench_fused.json 2>&1; tail -1 gpurun_out/bench_fused.json | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print("fused", d["ms_per_step"], d["stage_ms"], d["roofline"]["frac"])'
timeout 600 python bench.py --no-cpu-baseline --no-e2e --unfused-q > gpurun_out/bench_unfused.json 2>&1; tail -1 gpurun_out/bench_unfused.json | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print("unfused", d["ms_per_step"], d["stage_ms"], d["roofline"]["frac"])'
