mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
for b in 1 2 4 8; do timeout -k 5 120 python tools/dec_fault.py $b 2>&1 | tail -1; done
timeout -k 5 600 compute-sanitizer --tool memcheck python tools/dec_fault.py 8 > gpurun_out/dec_memcheck.log 2>&1; echo "memcheck rc=$?"; grep -m 20 -E "Invalid|at 0x|by thread|Address|ERROR SUMMARY" gpurun_out/dec_memcheck.log
