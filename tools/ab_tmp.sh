mkdir -p gpurun_out
python -m paper_2603_22300_b200.build --force >/dev/null
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$? $(tail -1 gpurun_out/pytest_gpu.log)"
grep -E "FAILED" gpurun_out/pytest_gpu.log | head
