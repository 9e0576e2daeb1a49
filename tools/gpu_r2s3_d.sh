# top-k v3b (compile-time k compaction, direct stores), R2 / window at d_v = 64 on SM100_OT
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_topk.py tests/test_gpu_edges.py tests/test_gpu_window.py tests/test_gpu_fused_q.py tests/test_gpu_attn.py -q -x > gpurun_out/pytest_d.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_d.log
timeout 300 python bench.py --no-cpu-baseline --no-e2e --no-long --no-dense-context > gpurun_out/bench_d.json 2> gpurun_out/bench_d.err; echo "bench rc=$?"; python - <<'P'
import json
d=json.loads(open("gpurun_out/bench_d.json").read().strip().splitlines()[-1]); print(d["ms_per_step"], d["stage_ms"])
P
timeout 300 python bench.py --config gpt2 --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --no-dense-context > gpurun_out/bench_gpt2_d.json 2>/dev/null; echo "gpt2 rc=$?"; python - <<'P'
import json
d=json.loads(open("gpurun_out/bench_gpt2_d.json").read().strip().splitlines()[-1]); print(d["ms_per_step"], d["stage_ms"])
P
timeout 600 ncu --set full --import-source on --clock-control none -k regex:topk_rows -s 2 -c 1 -o gpurun_out/topk_v3b -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-long --no-dense-context > gpurun_out/ncu_topk.log 2>&1; echo "ncu rc=$?"
