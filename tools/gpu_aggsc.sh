#!/bin/bash
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for r in 1 2; do
  for v in default "$@"; do
    if [ "$v" = default ]; then lib=""; else lib=build/variants/libb200tally_$v.so; fi
    echo -n "r$r $v "; BT_LIB_PATH=$lib timeout 300 python tools/point_walk_once.py 2
    echo -n "r$r $v "; BT_LIB_PATH=$lib timeout 300 python tools/point_walk_once.py 100
    echo -n "r$r $v "; BT_LIB_PATH=$lib timeout 300 python tools/variant_walk.py 2 0 12
    echo -n "r$r $v "; BT_LIB_PATH=$lib timeout 300 python tools/variant_walk.py 2 0 55
  done
done
