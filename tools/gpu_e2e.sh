python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 600 python -m pytest tests/test_gpu_attn.py -q -x -k "forward_composition or forward_host" > /tmp/t.log 2>&1; echo "tests rc=$?"; tail -2 /tmp/t.log
for c in 8 16 32 64 8 16 32; do echo "chunks=$c $(timeout 600 python bench.py --no-cpu-baseline --no-dense-context --steps 5 --e2e-chunks $c 2>/dev/null | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["ms_per_step"], d["e2e"]["ms_per_step"], d["e2e"]["value"])')"; done
