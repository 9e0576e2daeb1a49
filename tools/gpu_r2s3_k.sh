# repeated-launch race tests at the bench shapes; V prep split loops (vscale suite + Qwen3 prepare stage)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout -k 10 900 python -m pytest tests/test_gpu_repeat.py tests/test_gpu_vscale.py tests/test_gpu_sm100.py -q -x -p no:cacheprovider > gpurun_out/pytest_k.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_k.log
timeout -k 10 300 python bench.py --no-cpu-baseline --no-e2e --no-long --no-dense-context > gpurun_out/bench_k.json 2>/dev/null; echo "bench rc=$?"; python - <<'P'
import json
d=json.loads(open("gpurun_out/bench_k.json").read().strip().splitlines()[-1]); print(d["ms_per_step"], d["stage_ms"])
P
