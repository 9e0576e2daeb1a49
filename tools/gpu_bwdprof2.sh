mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 900 ncu --set full --import-source on --clock-control none -k regex:bwd_dkdv -s 1 -c 1 -o gpurun_out/bwd_dkdv3 -f python bench.py --mode bwd --steps 1 --warmup 1 > gpurun_out/ncu_dkdv.log 2>&1; echo "ncu dkdv rc=$?"
