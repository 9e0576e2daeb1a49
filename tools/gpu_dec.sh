mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 600 python -m pytest tests/test_gpu_decode.py tests/test_gpu_topk.py -q -x > gpurun_out/pytest_dec.log 2>&1; echo "dec+topk rc=$?"; tail -2 gpurun_out/pytest_dec.log
timeout 300 python bench.py --mode decode > gpurun_out/bench_decode.json 2>&1; tail -1 gpurun_out/bench_decode.json | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["ms_per_step"], d["roofline"]["frac"], d["context"])'
timeout 300 python bench.py --mode decode --decode-batch 1 > gpurun_out/bench_decode_b1.json 2>&1; tail -1 gpurun_out/bench_decode_b1.json | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["ms_per_step"], d["roofline"]["frac"], d["context"])'
