mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 600 python -m pytest tests/test_gpu_decode.py -q -x > gpurun_out/pytest_dec.log 2>&1; echo "dec rc=$?"; tail -2 gpurun_out/pytest_dec.log
for pf in 2 0 4 8 2; do
  SFA_NVCC_FLAGS="-DSFA_DEC_PF=$pf" python -m paper_2603_22300_b200.build --force > /dev/null 2>&1
  echo "pf=$pf $(timeout 300 python bench.py --mode decode --no-dense-context 2>/dev/null | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["ms_per_step"], d["roofline"]["frac"])') b1 $(timeout 300 python bench.py --mode decode --decode-batch 1 --no-dense-context 2>/dev/null | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["ms_per_step"], d["roofline"]["frac"])')"
done
