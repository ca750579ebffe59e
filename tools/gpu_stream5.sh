#!/bin/bash
# streamed move from 2^18 particles: parity, then e2e at 1e6 / 3e6 particles
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest -q -x -p no:cacheprovider -m gpu tests/test_gpu_parity.py -k "pipelined or options_keep_parity" > gpurun_out/stream_tests.log 2>&1; rc=$?; echo tests=$rc; tail -2 gpurun_out/stream_tests.log
[ $rc = 0 ] || exit 1
for P in 1000000 3000000; do for r in 1 2; do for sm in 1 0; do timeout 600 python tools/e2e_breakdown.py 0 $sm $P 2>&1 | grep "pinned.*defer=0"; done; done; done
timeout 1500 python -m pytest tests -x -q -m gpu -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?; tail -1 gpurun_out/pytest_gpu.log
