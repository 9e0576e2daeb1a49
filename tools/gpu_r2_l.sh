mkdir -p gpurun_out
SFA_NVCC_FLAGS="-DSFA_TIMELINE" python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
timeout 120 python tools/timeline.py 32768 oth qwen > gpurun_out/timeline_oth.txt 2>&1; echo "tl rc=$?"; head -40 gpurun_out/timeline_oth.txt
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
