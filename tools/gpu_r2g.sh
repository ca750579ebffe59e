cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 600 python tools/e2e_breakdown.py > gpurun_out/e2e_breakdown.txt 2>&1; echo e2e=$?; cat gpurun_out/e2e_breakdown.txt
timeout 600 python -m pytest tests/test_gpu_api.py -q -x --timeout 900 -p no:cacheprovider > gpurun_out/pytest_api.log 2>&1; echo api=$?; tail -3 gpurun_out/pytest_api.log
