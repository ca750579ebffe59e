#!/bin/bash
# streamed host-input move (one walk launch waiting on the copy stream's
# chunk marks): parity first, then the e2e step against per-chunk launches
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest -q -x -p no:cacheprovider -m gpu tests/test_gpu_parity.py -k "pipelined or options_keep_parity" > gpurun_out/stream_tests.log 2>&1; rc=$?; echo tests=$rc; tail -3 gpurun_out/stream_tests.log
[ $rc = 0 ] || exit 1
for r in 1 2; do
  for sm in 1 0; do
    timeout 600 python tools/e2e_breakdown.py 0 $sm 2>&1 | grep "defer=0"
  done
done
for c in 8 16; do timeout 600 python tools/e2e_breakdown.py $c 1 2>&1 | grep "pinned.*defer=0"; done
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-transport > gpurun_out/stream_bench.json 2> gpurun_out/stream_bench.err; echo bench=$?
python -c "import json;d=json.load(open('gpurun_out/stream_bench.json'));print('value %.4e e2e %.4e e2e_ms %.3f pageable %.4e'%(d['value'],d['e2e']['value'],d['e2e']['ms_per_step'],d['e2e']['pageable']['value']))"
timeout 1500 python -m pytest -q -x -p no:cacheprovider -m gpu tests > gpurun_out/stream_gpu_all.log 2>&1; echo gpu_all=$?; tail -2 gpurun_out/stream_gpu_all.log
