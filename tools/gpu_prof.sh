# GPU session: parity tests + ncu full profile of the walk kernel + bench
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q --timeout 600 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
tail -8 gpurun_out/pytest_gpu.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:walk_kernel -s 2 -c 1 -o gpurun_out/walk_full python bench.py --steps 1 --warmup 2 --no-e2e --no-cpu-baseline > gpurun_out/ncu_full.log 2>&1; echo ncu2=$?
tail -3 gpurun_out/ncu_full.log
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench=$?; cat gpurun_out/bench.json
