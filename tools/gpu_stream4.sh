#!/bin/bash
# streamed move (pinned inputs): parity, ncu launch list, memcheck, full GPU suite,
# e2e breakdown, both bench arms
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest -q -x -p no:cacheprovider -m gpu tests/test_gpu_parity.py -k "pipelined or options_keep_parity" > gpurun_out/stream_tests.log 2>&1; rc=$?; echo tests=$rc; tail -2 gpurun_out/stream_tests.log
[ $rc = 0 ] || exit 1
timeout -k 20 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-transport > gpurun_out/ncu_launch_bench.log 2>&1; echo ncu_launches=$?
timeout 1500 compute-sanitizer --print-limit 20 --tool memcheck --leak-check no python -m pytest -q -p no:cacheprovider -m gpu tests/test_gpu_parity.py -k "pipelined" > gpurun_out/stream_mem.log 2>&1; echo mem=$?; tail -2 gpurun_out/stream_mem.log
timeout 1500 python -m pytest -q -x -p no:cacheprovider -m gpu tests > gpurun_out/pytest_gpu.log 2>&1; echo gpu_all=$?; tail -2 gpurun_out/pytest_gpu.log
timeout 300 python __graft_entry__.py > gpurun_out/smoke.log 2>&1; echo smoke=$?; tail -1 gpurun_out/smoke.log
timeout 600 python tools/e2e_breakdown.py > gpurun_out/e2e_breakdown.txt 2>&1; echo e2e=$?; cat gpurun_out/e2e_breakdown.txt
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench=$?
python -c "import json;d=json.load(open('gpurun_out/bench.json'));print('value %.4e e2e %.4e e2e_ms %.3f pageable %.4e walk %.3f'%(d['value'],d['e2e']['value'],d['e2e']['ms_per_step'],d['e2e']['pageable']['value'],d['roofline']['kernel_ms_per_step']))"
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo ref=$?
