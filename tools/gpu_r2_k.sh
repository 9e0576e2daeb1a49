# Round 2: first run of SFA_KERNEL_SM100_OTH (Q~ in TMEM, 64-key score halves): watchdog parity, bench vs OT, ncu SMEM.
mkdir -p gpurun_out
B() { python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }; }
SFA_NVCC_FLAGS="-DSFA_WATCHDOG" B
timeout 240 python -m pytest tests/test_gpu_sm100.py -x -q -k "oth" > gpurun_out/pytest_k_wd.log 2>&1; echo "pytest wd rc=$?"; tail -4 gpurun_out/pytest_k_wd.log; grep -m2 "watchdog" gpurun_out/pytest_k_wd.log
B
BENCH="python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --no-long"
for kn in oth ot oth; do timeout 120 $BENCH --kernel $kn > gpurun_out/bench_k_$kn.json 2>gpurun_out/bench_k_$kn.err; echo "bench $kn rc=$?"; python -c "
import json; d=json.loads(open('gpurun_out/bench_k_$kn.json').read().strip().splitlines()[-1]); print('$kn', d['stage_ms'], d['clocks']['sm_mhz'], d['context']['dense_sdpa_ms'])"; done
NCUM=l1tex__data_pipe_tc_wavefronts_mem_shared.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,gpu__time_duration.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed,l1tex__data_pipe_tc_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active
timeout 300 ncu --metrics $NCUM --clock-control none -k regex:attn_sm100_oth -s 1 -c 1 python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-long --no-dense-context --kernel oth > gpurun_out/ncu_smem_oth.log 2>&1; echo "ncu rc=$?"; grep -E "wavefronts|duration|tensor|xu|issue" gpurun_out/ncu_smem_oth.log
