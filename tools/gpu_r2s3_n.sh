# top-k: two threads per row (d = 128) -- parity, repeat, timing, ncu
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout -k 10 300 python -m pytest tests/test_gpu_topk.py tests/test_gpu_repeat.py -q -x -p no:cacheprovider > gpurun_out/pytest_n.log 2>&1; rc=$?; echo "pytest rc=$rc"; tail -2 gpurun_out/pytest_n.log
[ $rc -eq 0 ] || exit 1
for i in 1 2; do timeout -k 10 300 python bench.py --no-cpu-baseline --no-e2e --no-long --no-dense-context > gpurun_out/bench_n.json 2>/dev/null; python - <<'P'
import json
d=json.loads(open("gpurun_out/bench_n.json").read().strip().splitlines()[-1]); print(d["ms_per_step"], d["stage_ms"]["topk_qk"])
P
done
timeout -k 10 400 ncu --set full --import-source on --clock-control none -k regex:topk_pairs -s 2 -c 1 -o gpurun_out/topk_pairs -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-long --no-dense-context > gpurun_out/ncu_topk.log 2>&1; echo "ncu rc=$?"
