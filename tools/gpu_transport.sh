cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_transport_gpu.py -q -s --timeout 600 -p no:cacheprovider > gpurun_out/pytest_transport.log 2>&1; echo pytest_transport=$?
grep -E "identical|passed|failed|Error|assert" gpurun_out/pytest_transport.log | head -30
timeout 1200 python -m pytest tests -m gpu -q --timeout 600 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
tail -3 gpurun_out/pytest_gpu.log
