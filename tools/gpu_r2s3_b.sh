# Round 2, session 3: new top-k kernel (persistent, cp.async double buffer, split layout) and SM100_OT
# with d_v = 64 (zero-padded V copy): their parity tests, then the stage timings.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_topk.py tests/test_gpu_sm100.py tests/test_gpu_fused_q.py -q -x > gpurun_out/pytest_b.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_b.log
timeout 300 python bench.py --no-cpu-baseline --no-e2e --no-long --no-dense-context > gpurun_out/bench_b.json 2> gpurun_out/bench_b.err; echo "bench rc=$?"; python - <<'P'
import json
d=json.loads(open("gpurun_out/bench_b.json").read().strip().splitlines()[-1]); print(d["ms_per_step"], d["stage_ms"])
P
for kern in auto ot; do timeout 300 python bench.py --config gpt2 --kernel $kern --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --no-dense-context > gpurun_out/bench_gpt2_$kern.json 2>/dev/null; echo "gpt2 $kern rc=$?"; python - "$kern" <<'P'
import json,sys
d=json.loads(open(f"gpurun_out/bench_gpt2_{sys.argv[1]}.json").read().strip().splitlines()[-1]); print(d["ms_per_step"], d["stage_ms"])
P
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/launches_gpt2_ot.csv python bench.py --config gpt2 --kernel ot --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-dense-context > /dev/null 2>&1; echo "launches rc=$?"
