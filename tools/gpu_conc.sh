python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for m in "" "--serial-stages" "" "--serial-stages"; do echo "mode=[$m] $(timeout 600 python bench.py --no-cpu-baseline --no-e2e --no-dense-context $m 2>/tmp/e.log | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["ms_per_step"], d["stage_ms"])')"; tail -2 /tmp/e.log; done
