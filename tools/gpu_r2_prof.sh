# round 2 profile pass: L2/HBM microbenchmark, bench, ncu launch list of the
# bench command, one ncu --set full capture of the walk kernel
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
./tools/micro/l2bw > gpurun_out/l2_peak.json 2> gpurun_out/l2_peak.err; echo l2bw=$?; cat gpurun_out/l2_peak.json
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench=$?; cat gpurun_out/bench.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_launch_bench.log 2>&1; echo ncu_launches=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:walk_staged -s 2 -c 1 -o gpurun_out/walk_full python bench.py --steps 1 --warmup 2 --no-e2e --no-cpu-baseline > gpurun_out/ncu_walk_full.log 2>&1; echo ncu_full=$?
ls -la gpurun_out
