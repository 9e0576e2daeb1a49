# decode combine kernel with the split loops unrolled by 8
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout -k 10 900 python -m pytest tests/test_gpu_decode.py tests/test_gpu_repeat.py -q -x -p no:cacheprovider > gpurun_out/pytest_u.log 2>&1; rc=$?; echo "pytest rc=$rc"; tail -2 gpurun_out/pytest_u.log
[ $rc -eq 0 ] || exit 1
for i in 1 2 3; do timeout -k 10 300 python bench.py --mode decode --steps 20 --warmup 5 > gpurun_out/bench_dec_u.json 2>/dev/null; python -c "import json;d=json.loads(open('gpurun_out/bench_dec_u.json').read().strip().splitlines()[-1]);print('decode', d['ms_per_step'], round(d['roofline']['frac'],4))"; done
