# Round-end evidence: full GPU suite, smoke, every bench mode, launch list + full ncu capture of the
# dominant kernel.  Outputs under gpurun_out/ (copied to profiles/ by hand).
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "ref rc=$?"
timeout 600 python bench.py --mode bwd > gpurun_out/bench_bwd.json 2>/dev/null; echo "bwd rc=$?"
timeout 600 python bench.py --mode decode > gpurun_out/bench_decode.json 2>/dev/null; echo "decode rc=$?"
timeout 600 python bench.py --edges-only --no-cpu-baseline --no-e2e > gpurun_out/bench_edges.json 2>/dev/null; echo "edges rc=$?"
timeout 600 python bench.py --window 4096 --no-cpu-baseline --no-e2e > gpurun_out/bench_window.json 2>/dev/null; echo "window rc=$?"
timeout 600 python bench.py --fused-q --no-cpu-baseline --no-e2e --no-dense-context > gpurun_out/bench_fusedq.json 2>/dev/null; echo "fusedq rc=$?"
timeout 600 python bench.py --config gpt2 --no-cpu-baseline --no-e2e > gpurun_out/bench_gpt2.json 2>/dev/null; echo "gpt2 rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-dense-context > gpurun_out/b_ncu.log 2>&1; echo "ncu list rc=$?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:attn_sm100_ot -s 1 -c 1 -o gpurun_out/ot_final -f python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-dense-context > gpurun_out/ncu_full.log 2>&1; echo "ncu full rc=$?"
