mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 600 python -m pytest tests/test_gpu_bwd.py -q -x > gpurun_out/pytest_bwd.log 2>&1; echo "bwd rc=$?"; tail -2 gpurun_out/pytest_bwd.log
timeout 600 python bench.py --mode bwd > gpurun_out/bench_bwd.json 2>&1; tail -1 gpurun_out/bench_bwd.json | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print("bwd", d["ms_per_step"], d["roofline"]["frac"])'
rm -f gpurun_out/sweep.jsonl
for k in 4 8 16 32 64 128; do
  timeout 300 python bench.py --config sweep --k $k --no-e2e --no-cpu-baseline 2>gpurun_out/sweep_err_$k.log | tail -1 >> gpurun_out/sweep.jsonl
done
timeout 300 python bench.py --config gpt2 --no-e2e --no-cpu-baseline 2>gpurun_out/gpt2.err | tail -1 > gpurun_out/bench_gpt2.json
timeout 300 python bench.py --config tiny --no-e2e --no-cpu-baseline 2>gpurun_out/tiny.err | tail -1 > gpurun_out/bench_tiny.json
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -1 gpurun_out/bench.json | cut -c1-200
