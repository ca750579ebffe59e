#!/bin/bash
# A/B of the default build against variants (build/variants/libb200tally_NAME.so):
#   tools/gpu_ab.sh NAME1 NAME2 ...   (run under gpurun; "default" = the in-tree library)
# Alternates the walk-only bench (3 rounds) and prints kernel ms per step.
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for r in 1 2 3; do
  for v in default "$@"; do
    if [ "$v" = default ]; then lib=""; else lib=build/variants/libb200tally_$v.so; fi
    BT_LIB_PATH=$lib timeout 300 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline \
      > gpurun_out/ab_${v}_$r.json 2> gpurun_out/ab_${v}_$r.err
    python -c "import json;d=json.load(open('gpurun_out/ab_${v}_$r.json'));print('ab $v round $r', '%.4e'%d['value'], '%.3f ms'%d['roofline']['kernel_ms_per_step'], d['ms_per_step'])" || tail -3 gpurun_out/ab_${v}_$r.err
  done
done
