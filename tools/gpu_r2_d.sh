# Round 2: warp-cooperative K~ decompression (SFA_DZ_WARP) A/B + parity of the SM100_OT paths.
mkdir -p gpurun_out
B() { python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }; }
BENCH="python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --no-long"
B
timeout 900 python -m pytest tests/test_gpu_sm100.py tests/test_gpu_attn.py tests/test_gpu_window.py tests/test_gpu_edges.py -x -q -m "gpu and not slow" > gpurun_out/pytest_d.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_d.log
for i in 1 2; do timeout 300 $BENCH > gpurun_out/bench_dz1_$i.json 2>/dev/null; echo "dz1 rc=$?"; done
timeout 900 ncu --metrics l1tex__data_pipe_tc_wavefronts_mem_shared.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum,gpu__time_duration.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed,l1tex__data_pipe_tc_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed --clock-control none -k regex:attn_sm100_ot -s 1 -c 1 python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-long --no-dense-context > gpurun_out/ncu_smem_dz1.log 2>&1; echo "ncu rc=$?"
SFA_NVCC_FLAGS="-DSFA_DZ_CLEAR_OLD=0" B
for i in 1 2; do timeout 300 $BENCH > gpurun_out/bench_dzfull_$i.json 2>/dev/null; echo "dzfull rc=$?"; done
SFA_NVCC_FLAGS="-DSFA_DZ_WARP=0" B
for i in 1 2; do timeout 300 $BENCH > gpurun_out/bench_dz0_$i.json 2>/dev/null; echo "dz0 rc=$?"; done
timeout 900 ncu --metrics l1tex__data_pipe_tc_wavefronts_mem_shared.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum,gpu__time_duration.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed,l1tex__data_pipe_tc_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed --clock-control none -k regex:attn_sm100_ot -s 1 -c 1 python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-long --no-dense-context > gpurun_out/ncu_smem_dz0.log 2>&1; echo "ncu rc=$?"
B
