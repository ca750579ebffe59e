# localization after the pruned-grid change: lanes sweep at the default density, C2 and 10.1M cube
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for n in 55 119; do timeout 300 python tools/locate_sweep.py $n 10000000 2>&1 | head -5; done
