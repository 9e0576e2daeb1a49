# Round 2: first run of the ping-pong kernel (SFA_KERNEL_SM100_PP): watchdog parity, then bench vs OT.
mkdir -p gpurun_out
B() { python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }; }
SFA_NVCC_FLAGS="-DSFA_WATCHDOG" B
timeout 300 python -m pytest tests/test_gpu_sm100.py -x -q -k "pp" > gpurun_out/pytest_pp_wd.log 2>&1; echo "pytest wd rc=$?"; tail -5 gpurun_out/pytest_pp_wd.log
B
timeout 300 python -m pytest tests/test_gpu_sm100.py -q -k "pp" > gpurun_out/pytest_pp.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_pp.log
BENCH="python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --no-long"
for kn in pp ot pp ot; do timeout 300 $BENCH --kernel $kn > gpurun_out/bench_k_$kn.json 2>gpurun_out/bench_k_$kn.err; echo "bench $kn rc=$?"; python -c "
import json; d=json.loads(open('gpurun_out/bench_k_$kn.json').read().strip().splitlines()[-1]); print('$kn', d['stage_ms'], d['clocks']['sm_mhz'])"; done
for kn in pp sm100; do timeout 300 $BENCH --config gpt2 --kernel $kn > gpurun_out/bench_gpt2_$kn.json 2>/dev/null; echo "gpt2 $kn rc=$?"; python -c "
import json; d=json.loads(open('gpurun_out/bench_gpt2_$kn.json').read().strip().splitlines()[-1]); print('gpt2 $kn', d['stage_ms'])"; done
