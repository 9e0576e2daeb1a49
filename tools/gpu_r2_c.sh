# Round 2: A/B of the OT kernel's P hand-off (SFA_OT_PHALF=1 halves vs 0 whole tile), launch list and
# one ncu --set full capture of the default attention kernel, SASS counts.
mkdir -p gpurun_out
B() { python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }; }
BENCH="python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --no-long"
B
timeout 900 python -m pytest tests/test_gpu_sm100.py tests/test_gpu_attn.py -x -q -m "gpu and not slow" > gpurun_out/pytest_c.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_c.log
for i in 1 2; do timeout 300 $BENCH > gpurun_out/bench_phalf1_$i.json 2>/dev/null; echo "phalf1 rc=$?"; done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_c.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-long --no-dense-context > gpurun_out/launches_c.log 2>&1; echo "launches rc=$?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:attn_sm100_ot -s 1 -c 1 -o gpurun_out/ot_r2c -f python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-long --no-dense-context > gpurun_out/ncu_full_c.log 2>&1; echo "ncu full rc=$?"
SFA_NVCC_FLAGS="-DSFA_OT_PHALF=0" B
for i in 1 2; do timeout 300 $BENCH > gpurun_out/bench_phalf0_$i.json 2>/dev/null; echo "phalf0 rc=$?"; done
B
