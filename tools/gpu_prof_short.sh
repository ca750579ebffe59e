# ncu capture of the walk kernel on a paper-physics move (sigma_t = 100, 1e7 particles)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
python tools/short_walk_once.py
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base mangled -k regex:walk_staged_kernelILi192ELi2ELb0ELb1 -s 2 -c 1 -o gpurun_out/walk_short python tools/short_walk_once.py > gpurun_out/ncu_short.log 2>&1; echo ncu=$?
