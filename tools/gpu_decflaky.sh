python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for i in 1 2 3 4 5 6; do timeout 300 python bench.py --mode decode > /tmp/d.json 2> /tmp/d.err; echo "run $i rc=$? $(tail -1 /tmp/d.json | cut -c1-60)"; if [ -s /tmp/d.err ]; then tail -5 /tmp/d.err; fi; done
timeout 600 python bench.py --mode bwd > /dev/null 2>&1; timeout 300 python bench.py --mode decode > /tmp/d.json 2> /tmp/d.err; echo "after bwd rc=$?"; tail -5 /tmp/d.err
