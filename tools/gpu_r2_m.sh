# Round 2: split-row top-k (two threads per row): parity + bench A/B.
mkdir -p gpurun_out
B() { python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }; }
B
timeout 600 python -m pytest tests/test_gpu_topk.py tests/test_gpu_fused_q.py tests/test_gpu_attn.py -q -x > gpurun_out/pytest_m.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_m.log
BENCH="python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --no-long --no-dense-context"
for i in 1 2; do timeout 120 $BENCH > gpurun_out/bench_m.json 2>/dev/null; python -c "
import json; d=json.loads(open('gpurun_out/bench_m.json').read().strip().splitlines()[-1]); print('split', d['stage_ms'])"; done
timeout 120 $BENCH --config gpt2 > gpurun_out/bench_m.json 2>/dev/null; python -c "
import json; d=json.loads(open('gpurun_out/bench_m.json').read().strip().splitlines()[-1]); print('split gpt2', d['stage_ms'])"
SFA_NVCC_FLAGS="-DSFA_TOPK_SPLIT=0" B
for i in 1 2; do timeout 120 $BENCH > gpurun_out/bench_m.json 2>/dev/null; python -c "
import json; d=json.loads(open('gpurun_out/bench_m.json').read().strip().splitlines()[-1]); print('row', d['stage_ms'])"; done
timeout 120 $BENCH --config gpt2 > gpurun_out/bench_m.json 2>/dev/null; python -c "
import json; d=json.loads(open('gpurun_out/bench_m.json').read().strip().splitlines()[-1]); print('row gpt2', d['stage_ms'])"
B
