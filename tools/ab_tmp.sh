mkdir -p gpurun_out
python -m paper_2603_22300_b200.build --force >/dev/null
timeout 600 python -m pytest tests/test_gpu_bwd.py -m gpu -x -q > gpurun_out/t_bwd.log 2>&1; echo "pytest rc=$? $(tail -1 gpurun_out/t_bwd.log)"
timeout 600 python bench.py --mode bwd --steps 5 --warmup 3 > gpurun_out/bench_bwd.json 2>gpurun_out/bench_bwd.err; echo "bench rc=$?"; cat gpurun_out/bench_bwd.json | head -c 1500; tail -3 gpurun_out/bench_bwd.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_bwd.csv python bench.py --mode bwd --steps 1 --warmup 1 > /dev/null 2>&1; echo "ncu rc=$?"
