#!/bin/bash
# GPU suite + smoke on the in-tree library, then ncu of the C4 n=119 walk for the
# in-tree library and the given variants (why the async refill loses there)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 300 python __graft_entry__.py > gpurun_out/smoke.log 2>&1; echo smoke=$?; tail -1 gpurun_out/smoke.log
timeout 1200 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?; tail -2 gpurun_out/pytest_gpu.log
for v in default "$@"; do
  if [ "$v" = default ]; then lib=""; else lib=build/variants/libb200tally_$v.so; fi
  BT_LIB_PATH=$lib timeout 900 ncu --section SpeedOfLight --section MemoryWorkloadAnalysis --section WarpStateStats --section SchedulerStats --section LaunchStats --clock-control none -k regex:walk_staged_kernel -s 1 -c 1 -o gpurun_out/w119_$v python tools/walk119_once.py > gpurun_out/ncu_w119_$v.log 2>&1; echo ncu_$v=$?
done
