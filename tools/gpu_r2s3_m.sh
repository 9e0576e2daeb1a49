# SM100_OT hand-off timelines over several work items of CTA 0 (SFA_TIMELINE build), GPT-2 heads
mkdir -p gpurun_out
SFA_NVCC_FLAGS="-DSFA_TIMELINE" python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout -k 10 300 python tools/timeline_ot_items.py 8 1024 > gpurun_out/tl_ot_gpt2.txt 2>&1; echo "tl rc=$?"
timeout -k 10 300 python tools/timeline_ot_items.py 1 8192 > gpurun_out/tl_ot_8k.txt 2>&1; echo "tl8k rc=$?"
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
head -60 gpurun_out/tl_ot_gpt2.txt
