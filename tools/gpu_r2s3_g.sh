# decode: one consumer group per V block (fixes the two-group stage-phase aliasing of the round-1
# 16-warp shape); 128-key blocks x 2 CTAs per SM (default) vs 256-key blocks x 1 CTA per SM
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
for db in 643 642; do SFA_DEC_DB=$db timeout -k 10 600 python -m pytest tests/test_gpu_decode.py -q -x -p no:cacheprovider > gpurun_out/pytest_g_$db.log 2>&1; echo "pytest db=$db rc=$?"; tail -1 gpurun_out/pytest_g_$db.log; done
for db in 1282 643 642 1282 643 642; do SFA_DEC_DB=$db timeout -k 10 300 python bench.py --mode decode --steps 20 --warmup 5 > gpurun_out/bench_dec_$db.json 2>gpurun_out/bench_dec_$db.err; echo "decode db=$db rc=$?"; python - $db <<'P'
import json,sys
d=json.loads(open(f"gpurun_out/bench_dec_{sys.argv[1]}.json").read().strip().splitlines()[-1]); print(d["ms_per_step"], d["roofline"]["frac"])
P
done
