SFA_NVCC_FLAGS="-DSFA_WATCHDOG" python -m paper_2603_22300_b200.build --force > /tmp/build.log 2>&1; tail -3 /tmp/build.log
timeout 120 python -m pytest tests/test_gpu_bwd.py -q -x > /tmp/b.log 2>&1; echo "bwd tests rc=$?"; grep -m5 'watchdog\|passed\|failed\|Error' /tmp/b.log
