cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_callback.py tests/test_transport_gpu.py -q -s --timeout 600 -p no:cacheprovider > gpurun_out/pytest_new.log 2>&1; echo pytest_new=$?
grep -E "identical|differ|passed|failed|Error|assert " gpurun_out/pytest_new.log | head -40
timeout 1200 python -m pytest tests -m gpu -q --timeout 600 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
tail -3 gpurun_out/pytest_gpu.log
timeout 900 python tools/sweep.py --which tr --out gpurun_out/sweep_tr.jsonl > gpurun_out/sweep_tr.log 2>&1; echo sweep=$?; cut -c1-400 gpurun_out/sweep_tr.log
