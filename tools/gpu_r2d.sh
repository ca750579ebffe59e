# round 2: multi-GPU handle, bench N>1 smoke, full GPU suite, L2 microbenchmark
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
./tools/micro/l2bw > gpurun_out/l2_peak.json 2> gpurun_out/l2_peak.err; echo l2bw=$?; cat gpurun_out/l2_peak.json
timeout 1200 python -m pytest tests/test_gpu_multi.py tests/test_gpu_bench_dist.py -q -x --timeout 900 -p no:cacheprovider > gpurun_out/pytest_multi.log 2>&1; echo multi=$?
tail -30 gpurun_out/pytest_multi.log
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
tail -5 gpurun_out/pytest_gpu.log
