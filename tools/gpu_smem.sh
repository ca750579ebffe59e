#!/bin/bash
# walk time per variant on the L2-resident (n=55) and HBM-resident (n=95, 119)
# cubes: does the direct refill's shared memory (three stages) cost L1?
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for r in 1 2; do
  for v in default "$@"; do
    if [ "$v" = default ]; then lib=""; else lib=build/variants/libb200tally_$v.so; fi
    for p in "2 119" "2 95" "2 55" "100 55"; do
      read sg nc <<< "$p"
      echo -n "r$r $v "; BT_LIB_PATH=$lib timeout 300 python tools/variant_walk.py $sg 0 $nc
    done
  done
done
