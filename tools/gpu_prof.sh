# ncu full capture (with source) of one walk launch of the bench workload
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
tag=${1:-walk}
[ -n "$2" ] && export BT_LIB_PATH=$2
timeout 900 ncu --set full --clock-control none --import-source on -k regex:walk_staged -s 2 -c 1 -o gpurun_out/$tag python bench.py --steps 1 --warmup 2 --no-e2e --no-cpu-baseline > gpurun_out/ncu_$tag.log 2>&1; echo ncu=$?
tail -3 gpurun_out/ncu_$tag.log
