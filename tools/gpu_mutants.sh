# Negative controls: build the library with one injected fault at a time (SFA_FAULT_*, see the #ifdefs in
# topk_row.cuh, attn_sm100_ot.cu, vprep.cu) and run the parity tests that should catch it.  A mutant is
# "caught" when at least one test fails; the unmodified build must pass the same selection.
mkdir -p gpurun_out
out=gpurun_out/mutants.txt
: > $out
B() { python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }; }
SEL_ATTN="tests/test_gpu_attn.py tests/test_gpu_sm100.py tests/test_gpu_window.py"
run() {  # $1 = fault macro (or none), $2 = tests
  if [ "$1" = none ]; then SFA_NVCC_FLAGS="" B; else SFA_NVCC_FLAGS="-D$1" B; fi
  timeout -k 10 400 python -m pytest $2 -q -m "gpu and not slow" -k "not pp and not pair and not wide" -p no:cacheprovider > gpurun_out/mut_$1.log 2>&1
  res=$(tail -1 gpurun_out/mut_$1.log)
  echo "$1 | $2 | $res" | tee -a $out
}
run none "tests/test_gpu_topk.py $SEL_ATTN"
run SFA_FAULT_TOPK_TIE_HIGH "tests/test_gpu_topk.py"
run SFA_FAULT_CAUSAL_PLUS1 "$SEL_ATTN"
run SFA_FAULT_NO_O_RESCALE "$SEL_ATTN"
run SFA_FAULT_SCALE "$SEL_ATTN"
run SFA_FAULT_KDENSE_DROP_LAST "$SEL_ATTN"
run SFA_FAULT_VSCALE "$SEL_ATTN"
SFA_NVCC_FLAGS="" B
