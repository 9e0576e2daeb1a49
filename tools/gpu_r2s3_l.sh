# GPT-2-shaped attention vs batch size (fixed vs per-tile cost), SM100 and SM100_OT kernels
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout -k 10 600 python tools/gpt2_scaling.py sm100 ot 2>&1 | tee gpurun_out/gpt2_scaling.txt
