# Round 2: K~ by TMA from the decompressed rows (SFA_OT_KTMA) A/B, parity of the OT paths, SMEM counters, MUFU bench.
mkdir -p gpurun_out
B() { python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }; }
BENCH="python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --no-long"
NCUM=l1tex__data_pipe_tc_wavefronts_mem_shared.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum,gpu__time_duration.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed,l1tex__data_pipe_tc_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active,dram__bytes_read.sum,dram__bytes_write.sum
B
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o gpurun_out/mufu_bench tools/mufu_bench.cu && ./gpurun_out/mufu_bench > gpurun_out/mufu_bench.txt 2>&1; echo "mufu rc=$?"
timeout 900 python -m pytest tests/test_gpu_sm100.py tests/test_gpu_attn.py tests/test_gpu_window.py tests/test_gpu_edges.py tests/test_gpu_fused_q.py tests/test_gpu_dist.py -x -q -m "gpu and not slow" > gpurun_out/pytest_e.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_e.log
for i in 1 2; do timeout 300 $BENCH > gpurun_out/bench_kt1_$i.json 2>/dev/null; echo "kt1 rc=$?"; done
timeout 900 ncu --metrics $NCUM --clock-control none -k regex:attn_sm100_ot -s 1 -c 1 python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-long --no-dense-context > gpurun_out/ncu_smem_kt1.log 2>&1; echo "ncu rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_kt1.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-long --no-dense-context > /dev/null 2>&1; echo "launches rc=$?"
SFA_NVCC_FLAGS="-DSFA_OT_KTMA=0" B
for i in 1 2; do timeout 300 $BENCH > gpurun_out/bench_kt0_$i.json 2>/dev/null; echo "kt0 rc=$?"; done
B
