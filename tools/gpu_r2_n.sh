# Round 2: where the backward kernels stand (shared-memory path, tensor pipe) before moving Q~ / K~ to TMA.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
NCUM=l1tex__data_pipe_tc_wavefronts_mem_shared.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,gpu__time_duration.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed,l1tex__data_pipe_tc_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active,l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum
timeout 600 ncu --metrics $NCUM --clock-control none -k regex:bwd_ -s 3 -c 2 python bench.py --mode bwd --steps 1 --warmup 1 > gpurun_out/ncu_bwd.log 2>&1; echo "ncu rc=$?"; grep -E "bwd_|wavefronts|duration|tensor|xu|issue|conflicts" gpurun_out/ncu_bwd.log
