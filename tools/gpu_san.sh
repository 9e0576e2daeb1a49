mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 900 compute-sanitizer --tool synccheck python tools/sanitize_smoke.py --no-ablations > gpurun_out/san_synccheck.log 2>&1; echo "synccheck rc=$?"; tail -3 gpurun_out/san_synccheck.log
timeout 900 compute-sanitizer --tool initcheck python tools/sanitize_smoke.py --no-ablations > gpurun_out/san_initcheck.log 2>&1; echo "initcheck rc=$?"; tail -3 gpurun_out/san_initcheck.log
