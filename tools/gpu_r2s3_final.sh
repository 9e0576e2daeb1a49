# Round 2 (session 3) evidence: full GPU suite, smoke, the default bench line, the reference arm, launch
# list, one ncu --set full capture of the attention kernel and of the top-k kernel, backward / decode /
# GPT-2 / sweep-point benches.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout -k 10 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_final.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_final.log
timeout -k 10 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_final.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke_final.log
timeout -k 10 900 python bench.py > gpurun_out/bench_final.json 2> gpurun_out/bench_final.err; echo "bench rc=$?"; tail -c 400 gpurun_out/bench_final.json
timeout -k 10 600 python bench.py --impl reference > gpurun_out/bench_reference.json 2>/dev/null; echo "ref rc=$?"
timeout -k 10 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/launches_final.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-long --no-dense-context > /dev/null 2>&1; echo "launches rc=$?"
timeout -k 10 900 ncu --set full --import-source on --clock-control none -k regex:attn_sm100_ot -s 1 -c 1 -o gpurun_out/ot_final_r2s3 -f python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-long --no-dense-context > gpurun_out/ncu_final.log 2>&1; echo "ncu ot rc=$?"
timeout -k 10 300 python bench.py --mode bwd --steps 5 --warmup 3 > gpurun_out/bench_bwd_final.json 2>/dev/null; echo "bwd rc=$?"
timeout -k 10 300 python bench.py --mode decode --steps 20 --warmup 5 > gpurun_out/bench_decode_final.json 2>/dev/null; echo "decode rc=$?"
timeout -k 10 300 python bench.py --config gpt2 --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/bench_gpt2_final.json 2>/dev/null; echo "gpt2 rc=$?"
timeout -k 10 300 python bench.py --config gpt2 --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --graph > gpurun_out/bench_gpt2_graph.json 2>/dev/null; echo "gpt2 graph rc=$?"
for kk in 4 16 128; do timeout -k 10 300 python bench.py --config sweep --k $kk --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_sweep_k$kk.json 2>/dev/null; echo "sweep $kk rc=$?"; done
timeout -k 10 300 python bench.py --window 4096 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-long > gpurun_out/bench_window4096.json 2>/dev/null; echo "window rc=$?"
timeout -k 10 300 python bench.py --edges-only --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-long > gpurun_out/bench_edges.json 2>/dev/null; echo "edges rc=$?"
