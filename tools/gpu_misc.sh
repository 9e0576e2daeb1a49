mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu.log
for k in 64 128; do timeout 300 python bench.py --config sweep --k $k --no-e2e --no-cpu-baseline 2>/dev/null | tail -1 > gpurun_out/sweep_k$k.json; done
timeout 300 python bench.py --mode decode > gpurun_out/bench_decode.json 2>&1; tail -1 gpurun_out/bench_decode.json | cut -c1-100
timeout 600 compute-sanitizer --tool memcheck python tools/sanitize_smoke.py > gpurun_out/san_memcheck.log 2>&1; echo "memcheck rc=$?"; tail -3 gpurun_out/san_memcheck.log
timeout 900 compute-sanitizer --tool racecheck python tools/sanitize_smoke.py > gpurun_out/san_racecheck.log 2>&1; echo "racecheck rc=$?"; tail -3 gpurun_out/san_racecheck.log
timeout 900 compute-sanitizer --tool synccheck python tools/sanitize_smoke.py > gpurun_out/san_synccheck.log 2>&1; echo "synccheck rc=$?"; tail -3 gpurun_out/san_synccheck.log
