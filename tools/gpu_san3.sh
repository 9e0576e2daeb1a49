# Round 2: racecheck of the tcgen05.commit / cross-warp patterns (repro) and of the product kernels after the
# backward's explicit epilogue barriers; backward parity + bench.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -I paper_2603_22300_b200/csrc tools/racecheck_commit_repro.cu -o gpurun_out/rcr
for m in 0 1 2 3; do timeout 120 compute-sanitizer --tool racecheck ./gpurun_out/rcr $m $m > gpurun_out/rcr_mode$m.txt 2>&1; echo "mode $m: $(grep -E 'read|SUMMARY' gpurun_out/rcr_mode$m.txt | tr '\n' ' ')"; done
timeout 1500 compute-sanitizer --tool racecheck --print-limit 20 python tools/sanitize_smoke.py > gpurun_out/san_racecheck2.txt 2>&1; echo "racecheck rc=$?"; tail -3 gpurun_out/san_racecheck2.txt
timeout 600 python -m pytest tests/test_gpu_bwd.py -q > gpurun_out/pytest_bwd2.log 2>&1; echo "bwd pytest rc=$?"; tail -1 gpurun_out/pytest_bwd2.log
timeout 300 python bench.py --mode bwd --steps 5 --warmup 3 > gpurun_out/bench_bwd2.json 2>/dev/null; python -c "
import json; d=json.loads(open('gpurun_out/bench_bwd2.json').read().strip().splitlines()[-1]); print('bwd', d['ms_per_step'], d['roofline']['frac'])"
