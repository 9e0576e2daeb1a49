mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 900 python bench.py --config long --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-dense-context > gpurun_out/bench_long.json 2> gpurun_out/bench_long.err; tail -1 gpurun_out/bench_long.json | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print("long", d["ms_per_step"], d["stage_ms"], d["roofline"]["frac"])'
timeout 900 python bench.py --config long --shard-seq --steps 3 --warmup 3 > gpurun_out/bench_long_shard.json 2> gpurun_out/bench_long_shard.err; tail -1 gpurun_out/bench_long_shard.json | cut -c1-600
