#!/bin/bash
# transport line: aggregation hold 4 (default) vs 128 (variant), alternating
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for r in 1 2; do
  for v in default trhold; do
    if [ "$v" = default ]; then lib=""; else lib=build/variants/libb200tally_$v.so; fi
    BT_LIB_PATH=$lib timeout 900 python tools/transport_line.py > gpurun_out/trh_$v.json 2>/dev/null
    python -c "import json;d=json.load(open('gpurun_out/trh_$v.json'));print('r$r $v %.4e'%d['value'])"
  done
done
timeout 1200 python -m pytest -q -x -p no:cacheprovider -m gpu tests/test_transport_gpu.py > gpurun_out/trh_tests.log 2>&1; echo tr_tests=$?; tail -1 gpurun_out/trh_tests.log
