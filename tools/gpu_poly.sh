for p in 2 1 3 2 1 3; do
  SFA_NVCC_FLAGS="-DSFA_OT_POLY=$p" python -m paper_2603_22300_b200.build --force > /dev/null 2>&1
  echo "poly=$p $(timeout 600 python bench.py --no-cpu-baseline --no-e2e --no-dense-context 2>/dev/null | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["ms_per_step"], d["stage_ms"]["attn"])')"
done
