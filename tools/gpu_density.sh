# localization grid: density x pruning sweep (tools/locate_sweep.py) + the localization parity tests
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -k "locali or grid or pruning" 2>&1 | tail -3
for pr in 1; do
for d in 0.5 1 2 4 8; do
  for n in 55 119; do
    B200TALLY_GRID_PRUNE=$pr B200TALLY_GRID_DENSITY=$d timeout 300 python tools/locate_sweep.py $n 10000000 2>&1 | sed -n 2p | sed "s/^/prune=$pr density=$d n=$n /"
  done
done
done
