#!/bin/bash
# host-input move pipeline depth (BT_OPT_MOVE_CHUNKS) vs the e2e step
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for c in 4 1 2 3 6 8 4; do
  echo "== move_chunks=$c"; timeout 600 python tools/e2e_breakdown.py $c 2>&1 | grep "defer=0"
done
