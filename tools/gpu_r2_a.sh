# Round 2, first GPU check: the new multi-GPU/host-plan tests, tiny/huge V, long-context parity to 1M,
# the new bench line (head-sharded headline + long_context block), long benches, MUFU microbenchmark.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o gpurun_out/mufu_bench tools/mufu_bench.cu && ./gpurun_out/mufu_bench > gpurun_out/mufu_bench.txt 2>&1; echo "mufu rc=$?"
export SFA_PARITY_LOG=$PWD/gpurun_out/parity_headroom.jsonl
timeout 600 python -m pytest tests/test_gpu_vscale.py tests/test_gpu_multi.py tests/test_gpu_dist.py -q -x > gpurun_out/pytest_new.log 2>&1; echo "pytest new rc=$?"; tail -3 gpurun_out/pytest_new.log
timeout 300 python bench.py --steps 10 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"; tail -3 gpurun_out/bench.err
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
for n in 262144 1048576; do
  timeout 600 python bench.py --config long --seq-len $n --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-dense-context > gpurun_out/bench_long_$n.json 2> gpurun_out/bench_long_$n.err; echo "long $n rc=$?"
done
