# Round 2: persistent tile scheduler in the OT kernel: watchdog parity, bench A/B vs one item per CTA.
mkdir -p gpurun_out
B() { python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }; }
SFA_NVCC_FLAGS="-DSFA_WATCHDOG" B
timeout 240 python -m pytest tests/test_gpu_sm100.py tests/test_gpu_attn.py tests/test_gpu_window.py tests/test_gpu_edges.py tests/test_gpu_fused_q.py -x -q -m "gpu and not slow" > gpurun_out/pytest_j_wd.log 2>&1; echo "pytest wd rc=$?"; tail -4 gpurun_out/pytest_j_wd.log
B
BENCH="python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --no-long --no-dense-context"
timeout 120 $BENCH > gpurun_out/bench_j.json 2>gpurun_out/bench_j.err; echo "bench rc=$?"; python -c "
import json; d=json.loads(open('gpurun_out/bench_j.json').read().strip().splitlines()[-1]); print('persist', d['stage_ms'], d['clocks']['sm_mhz'], d['ms_per_step'])"
SFA_NVCC_FLAGS="-DSFA_OT_ONE_ITEM_PER_CTA=1" B
timeout 120 $BENCH > gpurun_out/bench_j1.json 2>/dev/null; python -c "
import json; d=json.loads(open('gpurun_out/bench_j1.json').read().strip().splitlines()[-1]); print('one item', d['stage_ms'], d['clocks']['sm_mhz'], d['ms_per_step'])"
B
timeout 120 $BENCH > gpurun_out/bench_j.json 2>gpurun_out/bench_j.err; python -c "
import json; d=json.loads(open('gpurun_out/bench_j.json').read().strip().splitlines()[-1]); print('persist', d['stage_ms'], d['clocks']['sm_mhz'], d['ms_per_step'])"
timeout 120 $BENCH --graph > gpurun_out/bench_jg.json 2>gpurun_out/bench_jg.err; python -c "
import json; d=json.loads(open('gpurun_out/bench_jg.json').read().strip().splitlines()[-1]); print('graph', d['stage_ms'], d['ms_per_step'])"
for g in "" "--graph"; do timeout 120 $BENCH --config gpt2 $g > gpurun_out/bench_jgpt2.json 2>/dev/null; python -c "
import json; d=json.loads(open('gpurun_out/bench_jgpt2.json').read().strip().splitlines()[-1]); print('gpt2 [$g]', d['stage_ms'], d['ms_per_step'])"; done
