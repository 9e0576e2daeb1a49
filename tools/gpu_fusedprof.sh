mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 900 ncu --set full --import-source on --clock-control none -k regex:attn_sm100_ot -s 1 -c 1 -o gpurun_out/ot_fused -f python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-dense-context > gpurun_out/ncu_fused.log 2>&1; echo "ncu rc=$?"
