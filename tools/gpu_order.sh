mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_sm100.py tests/test_gpu_attn.py tests/test_gpu_window.py -q -x > gpurun_out/pytest_order.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/pytest_order.log
for o in 1 0 1 0; do
  if [ $o = 0 ]; then SFA_NVCC_FLAGS="-DSFA_OT_ORDER=0" python -m paper_2603_22300_b200.build --force > /dev/null 2>&1; else python -m paper_2603_22300_b200.build --force > /dev/null 2>&1; fi
  echo "order=$o $(timeout 600 python bench.py --no-cpu-baseline --no-e2e --no-dense-context 2>/dev/null | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["ms_per_step"], d["stage_ms"]["attn"])')"
done
python -m paper_2603_22300_b200.build --force > /dev/null 2>&1
timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:attn_sm100_ot -s 1 -c 1 python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-dense-context > gpurun_out/ncu_order.log 2>&1; grep -E 'dram__bytes|gpu__time' gpurun_out/ncu_order.log
