mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 900 ncu --set full --import-source on --clock-control none -k regex:decode_partial -s 3 -c 1 -o gpurun_out/decode3 -f python bench.py --mode decode --steps 2 --warmup 3 --no-dense-context > gpurun_out/ncu_dec.log 2>&1; echo "ncu rc=$?"
