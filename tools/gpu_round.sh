# standard GPU session: smoke, parity tests, bench (+ reference arm), sweeps (C3/C4/C5),
# launch list and one ncu --set full capture of the walk kernel
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 300 python __graft_entry__.py > gpurun_out/smoke.log 2>&1; echo smoke=$?; tail -1 gpurun_out/smoke.log
timeout 1200 python -m pytest tests -m gpu -q --timeout 600 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
tail -3 gpurun_out/pytest_gpu.log
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench=$?; cat gpurun_out/bench.json
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo ref=$?; cat gpurun_out/bench_ref.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-transport > gpurun_out/ncu_launch_bench.log 2>&1; echo ncu_launches=$?
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base mangled -k regex:walk_staged_kernelILi192ELi2ELb0ELb1 -s 2 -c 1 -o gpurun_out/walk_full python bench.py --steps 1 --warmup 2 --no-e2e --no-cpu-baseline > gpurun_out/ncu_walk_full.log 2>&1; echo ncu_full=$?
timeout 1500 python tools/sweep.py --out gpurun_out/sweep.jsonl > gpurun_out/sweep.log 2>&1; echo sweep=$?; cut -c1-300 gpurun_out/sweep.log
