# full GPU suite after the round-2 changes + locate kernel ncu capture
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider -rs > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
tail -15 gpurun_out/pytest_gpu.log
timeout 300 python -m pytest tests/test_transport_gpu.py -q -s -p no:cacheprovider 2>&1 | grep -E "mean diff|K\*se|identical|passed|failed" | head -40
timeout 900 ncu --set full --clock-control none --import-source on -k regex:locate_grid -c 1 -o gpurun_out/locate_full python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_locate.log 2>&1; echo ncu_locate=$?
