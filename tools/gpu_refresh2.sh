# round-2 refresh: transport line, sweeps (library-only batch times), walk ncu capture
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python tools/transport_line.py > gpurun_out/tr_line.json 2> gpurun_out/tr_line.err; echo line=$?; cut -c1-400 gpurun_out/tr_line.json
timeout 1500 python tools/sweep.py --out gpurun_out/sweep.jsonl > gpurun_out/sweep.log 2>&1; echo sweep=$?; cut -c1-250 gpurun_out/sweep.log
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base mangled -k regex:walk_staged_kernelILi192ELi2ELb0ELb1 -s 2 -c 1 -o gpurun_out/walk_full python bench.py --steps 1 --warmup 2 --no-e2e --no-cpu-baseline > gpurun_out/ncu_walk_full.log 2>&1; echo ncu_full=$?
