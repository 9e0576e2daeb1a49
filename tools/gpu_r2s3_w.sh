# where the first tile's clocks go in an SFA_TIMELINE build (the debug score-tile dump; tools/timeline_ot_coldstart.py)
mkdir -p gpurun_out
SFA_NVCC_FLAGS="-DSFA_TIMELINE" python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout -k 10 300 python tools/timeline_ot_coldstart.py 2>&1 | tee gpurun_out/tl_coldstart.txt
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
