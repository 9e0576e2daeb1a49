# Round 2: backward with Q~ / K~ by TMA (SFA_BWD_TMA): watchdog parity, bench A/B, ncu SMEM.
mkdir -p gpurun_out
B() { python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }; }
SFA_NVCC_FLAGS="-DSFA_WATCHDOG" B
timeout 300 python -m pytest tests/test_gpu_bwd.py -x -q > gpurun_out/pytest_o_wd.log 2>&1; echo "pytest wd rc=$?"; tail -3 gpurun_out/pytest_o_wd.log; grep -m2 watchdog gpurun_out/pytest_o_wd.log
B
for i in 1 2; do timeout 200 python bench.py --mode bwd --steps 5 --warmup 3 > gpurun_out/bench_o.json 2>/dev/null; python -c "
import json; d=json.loads(open('gpurun_out/bench_o.json').read().strip().splitlines()[-1]); print('tma', round(d['ms_per_step'],3), round(d['roofline']['frac'],3))"; done
NCUM=l1tex__data_pipe_tc_wavefronts_mem_shared.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,gpu__time_duration.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed,l1tex__data_pipe_tc_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum
timeout 600 ncu --metrics $NCUM --clock-control none -k regex:bwd_d -s 2 -c 2 python bench.py --mode bwd --steps 1 --warmup 1 > gpurun_out/ncu_bwd_tma.log 2>&1; grep -E "bwd_d|wavefronts|duration|tensor|conflicts" gpurun_out/ncu_bwd_tma.log
SFA_NVCC_FLAGS="-DSFA_BWD_TMA=0" B
for i in 1 2; do timeout 200 python bench.py --mode bwd --steps 5 --warmup 3 > gpurun_out/bench_o.json 2>/dev/null; python -c "
import json; d=json.loads(open('gpurun_out/bench_o.json').read().strip().splitlines()[-1]); print('decomp', round(d['ms_per_step'],3), round(d['roofline']['frac'],3))"; done
B
