# Round 2, session 3 re-entry check: build, smoke, the GPU suite, the default bench line, GPT-2 line.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_a.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke_a.log
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench_a.json 2> gpurun_out/bench_a.err; echo "bench rc=$?"; tail -c 1500 gpurun_out/bench_a.json
timeout 300 python bench.py --config gpt2 --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --graph > gpurun_out/bench_gpt2_a.json 2>/dev/null; echo "gpt2 rc=$?"; tail -c 800 gpurun_out/bench_gpt2_a.json
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_a.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_a.log
