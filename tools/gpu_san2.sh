# Round 2: compute-sanitizer over the product kernels incl. the round-2 ones, and the tcgen05.commit racecheck repro.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -I paper_2603_22300_b200/csrc tools/racecheck_commit_repro.cu -o gpurun_out/rcr
./gpurun_out/rcr > gpurun_out/rcr_plain.txt 2>&1; cat gpurun_out/rcr_plain.txt
for mode in 0 1; do :; done
timeout 300 compute-sanitizer --tool racecheck ./gpurun_out/rcr > gpurun_out/rcr_racecheck.txt 2>&1; echo "rcr racecheck rc=$?"; tail -25 gpurun_out/rcr_racecheck.txt
for tool in memcheck synccheck initcheck racecheck; do
  timeout 1500 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize_smoke.py > gpurun_out/san_$tool.txt 2>&1; echo "$tool rc=$?"; tail -4 gpurun_out/san_$tool.txt
done
