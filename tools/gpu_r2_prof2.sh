# walk kernel full ncu capture (the direct-refill, digest-free bench kernel) + host copy rates
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
./tools/micro/hostcopy > gpurun_out/hostcopy.json 2> gpurun_out/hostcopy.err; echo hostcopy=$?; cat gpurun_out/hostcopy.json
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base mangled -k regex:walk_staged_kernelILi192ELi2ELb0ELb1 -s 2 -c 1 -o gpurun_out/walk_full python bench.py --steps 1 --warmup 2 --no-e2e --no-cpu-baseline > gpurun_out/ncu_walk_full.log 2>&1; echo ncu_full=$?
tail -3 gpurun_out/ncu_walk_full.log
