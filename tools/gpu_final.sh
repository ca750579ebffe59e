# final round-2 measurement pass: walk ncu capture (for walk_sol.json), transport ncu capture
# (transport_sol.json), launch list, sweeps, short moves, transport line, bench (both arms)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base mangled -k regex:walk_staged_kernelILi192ELi2ELb0ELb1 -s 2 -c 1 -o gpurun_out/walk_full python bench.py --steps 1 --warmup 2 --no-e2e --no-cpu-baseline > gpurun_out/ncu_walk_full.log 2>&1; echo ncu_full=$?
bash tools/gpu_prof_tr.sh
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-transport > gpurun_out/ncu_launch_bench.log 2>&1; echo ncu_launches=$?
timeout 1500 python tools/sweep.py --out gpurun_out/sweep.jsonl > gpurun_out/sweep.log 2>&1; echo sweep=$?
timeout 600 python tools/short_moves.py > gpurun_out/short.jsonl 2>&1; echo short=$?
timeout 900 python tools/transport_line.py > gpurun_out/tr_line.json 2> gpurun_out/tr_line.err; echo line=$?
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench=$?
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo ref=$?
