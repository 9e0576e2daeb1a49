mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 600 python -m pytest tests/test_gpu_bwd.py -q -x > gpurun_out/pytest_bwd.log 2>&1; echo "bwd rc=$?"; tail -2 gpurun_out/pytest_bwd.log
for i in 1 2; do timeout 600 python bench.py --mode bwd > gpurun_out/bench_bwd.json 2>&1; tail -1 gpurun_out/bench_bwd.json | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print("bwd", d["ms_per_step"], d["roofline"]["frac"])'; done
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_bwd.csv python bench.py --mode bwd --steps 2 --warmup 1 > gpurun_out/b_ncu_bwd.log 2>&1; echo "ncu rc=$?"
