python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
rm -f gpurun_out/sweep2.jsonl
for k in 4 8 16 32 64 128; do
  timeout 300 python bench.py --config sweep --k $k --no-e2e --no-cpu-baseline 2>/dev/null | tail -1 >> gpurun_out/sweep2.jsonl
done
echo done
