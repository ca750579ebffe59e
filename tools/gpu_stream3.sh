#!/bin/bash
# streamed move: tools detection, the ncu launch list (must finish), parity, e2e, bench
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 300 ncu --metrics gpu__time_duration.sum python -c "import os; print('ncu env', os.environ.get('CUDA_INJECTION64_PATH'))" 2>&1 | grep "ncu env"
timeout 300 compute-sanitizer python -c "import os; print('sanitizer env', os.environ.get('CUDA_INJECTION64_PATH'))" 2>&1 | grep "sanitizer env"
timeout 900 python -m pytest -q -x -p no:cacheprovider -m gpu tests/test_gpu_parity.py -k "pipelined or options_keep_parity" > gpurun_out/stream_tests.log 2>&1; rc=$?; echo tests=$rc; tail -2 gpurun_out/stream_tests.log
[ $rc = 0 ] || exit 1
timeout -k 20 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-transport > gpurun_out/ncu_launch_bench.log 2>&1; echo ncu_launches=$?
for r in 1 2; do for sm in 1 0; do timeout 600 python tools/e2e_breakdown.py 0 $sm 2>&1 | grep "defer=0"; done; done
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench=$?
python -c "import json;d=json.load(open('gpurun_out/bench.json'));print('value %.4e e2e %.4e e2e_ms %.3f pageable %.4e walk %.3f'%(d['value'],d['e2e']['value'],d['e2e']['ms_per_step'],d['e2e']['pageable']['value'],d['roofline']['kernel_ms_per_step']))"
