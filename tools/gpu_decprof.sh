mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 600 python bench.py --mode decode > gpurun_out/bench_decode.json 2>&1; tail -1 gpurun_out/bench_decode.json | cut -c1-300
timeout 900 ncu --set full --import-source on --clock-control none -k regex:decode_partial -s 3 -c 1 -o gpurun_out/decode -f python bench.py --mode decode --steps 2 --warmup 3 > gpurun_out/ncu_dec.log 2>&1; echo "ncu rc=$?"
