# round 2: parity, microbench, bench (pinned + pageable e2e), ncu capture of the bench kernel
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
./tools/micro/l2bw > gpurun_out/l2_peak.json 2> gpurun_out/l2_peak.err; echo l2bw=$?; cat gpurun_out/l2_peak.json
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 900 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
tail -5 gpurun_out/pytest_gpu.log
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench=$?; cat gpurun_out/bench.json
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base mangled -k regex:walk_staged_kernelILi192ELi2ELb0ELb1 -s 2 -c 1 -o gpurun_out/walk_full python bench.py --steps 1 --warmup 2 --no-e2e --no-cpu-baseline > gpurun_out/ncu_walk_full.log 2>&1; echo ncu_full=$?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_launch_bench.log 2>&1; echo ncu_launches=$?
