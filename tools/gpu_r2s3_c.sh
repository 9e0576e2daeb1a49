# ncu --set full of the top-k kernel at Qwen3-32K (one launch: Q and K rows)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 600 ncu --set full --import-source on --clock-control none -k regex:topk_rows -s 2 -c 1 -o gpurun_out/topk_v3 -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-long --no-dense-context > gpurun_out/ncu_topk.log 2>&1; echo "ncu rc=$?"; tail -3 gpurun_out/ncu_topk.log
