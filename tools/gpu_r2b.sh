# round 2: new parity tests + the full GPU suite + bench
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_api.py tests/test_gpu_scale_parity.py -q --timeout 900 -p no:cacheprovider -x > gpurun_out/pytest_new.log 2>&1; echo new=$?
tail -15 gpurun_out/pytest_new.log
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider --deselect tests/test_gpu_scale_parity.py > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
tail -5 gpurun_out/pytest_gpu.log
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench=$?; cat gpurun_out/bench.json
