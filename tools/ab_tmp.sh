mkdir -p gpurun_out
b() { SFA_NVCC_FLAGS="$1" python -m paper_2603_22300_b200.build --force >/dev/null; }
bench() { timeout 300 python bench.py --steps 10 --warmup 3 --kernel $1 --no-cpu-baseline > gpurun_out/bench_$2.json 2>gpurun_out/bench_$2.err; echo "$2 rc=$? $(grep -o '"attn": [0-9.]*' gpurun_out/bench_$2.json)"; }
b ""
timeout 300 python -m pytest tests/test_gpu_sm100.py -m gpu -x -q -k ot > gpurun_out/t_q.log 2>&1; echo "pytest rc=$? $(tail -1 gpurun_out/t_q.log)"
bench ot late1
b "-DSFA_OT_PVLATE=0"
bench ot late0
SFA_NVCC_FLAGS="-DSFA_TIMELINE" python -m paper_2603_22300_b200.build --force >/dev/null && timeout 120 python tools/timeline.py 32768 ot qwen > gpurun_out/tl_qt.txt 2>&1
sed -n 30,36p gpurun_out/tl_qt.txt
