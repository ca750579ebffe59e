# ncu full capture of one locate_grid_kernel launch of the bench workload
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:locate_grid -c 1 -o gpurun_out/locate python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/ncu_locate.log 2>&1; echo ncu=$?
