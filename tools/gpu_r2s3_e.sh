# top-k v4 (byte-domain mantissa bisection with vabsdiff4, tie skipping in the walk; NaN keys clamped),
# one-launch prepare for small heads: parity + timing + ncu
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout -k 10 240 python -m pytest tests/test_gpu_topk.py -v -x -p no:cacheprovider > gpurun_out/pytest_e0.log 2>&1; rc=$?; echo "pytest topk rc=$rc"; tail -3 gpurun_out/pytest_e0.log
[ $rc -eq 0 ] || exit 1
timeout -k 10 900 python -m pytest tests/test_gpu_edges.py tests/test_gpu_window.py tests/test_gpu_fused_q.py tests/test_gpu_attn.py tests/test_gpu_sm100.py tests/test_gpu_vscale.py -q -x -p no:cacheprovider > gpurun_out/pytest_e.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_e.log
timeout -k 10 300 python bench.py --no-cpu-baseline --no-e2e --no-long --no-dense-context > gpurun_out/bench_e.json 2> gpurun_out/bench_e.err; echo "bench rc=$?"; python - <<'P'
import json
d=json.loads(open("gpurun_out/bench_e.json").read().strip().splitlines()[-1]); print(d["ms_per_step"], d["stage_ms"])
P
timeout -k 10 300 python bench.py --config gpt2 --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --no-dense-context > gpurun_out/bench_gpt2_e.json 2>/dev/null; echo "gpt2 rc=$?"; python - <<'P'
import json
d=json.loads(open("gpurun_out/bench_gpt2_e.json").read().strip().splitlines()[-1]); print(d["ms_per_step"], d["stage_ms"])
P
timeout -k 10 300 python bench.py --config gpt2 --graph --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --no-dense-context > gpurun_out/bench_gpt2g_e.json 2>/dev/null; echo "gpt2 graph rc=$?"; python - <<'P'
import json
d=json.loads(open("gpurun_out/bench_gpt2g_e.json").read().strip().splitlines()[-1]); print(d["ms_per_step"], d["stage_ms"])
P
timeout -k 10 400 ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file gpurun_out/launches_gpt2_f.csv python bench.py --config gpt2 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-dense-context > /dev/null 2>&1; echo "launches rc=$?"
