python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 300 python -m pytest tests/test_gpu_bwd.py -q -x > /tmp/b.log 2>&1; echo "bwd tests rc=$?"; tail -2 /tmp/b.log
timeout 300 python bench.py --mode bwd 2>/dev/null | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print("bwd", d["ms_per_step"], d["roofline"]["frac"])'
