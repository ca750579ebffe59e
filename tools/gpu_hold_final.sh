#!/bin/bash
# aggregation hold 128: GPU suite, smoke, options sweep, transport line, both bench arms
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 1500 python -m pytest tests -x -q -m gpu -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?; tail -2 gpurun_out/pytest_gpu.log
timeout 300 python __graft_entry__.py > gpurun_out/smoke.log 2>&1; echo smoke=$?; tail -1 gpurun_out/smoke.log
timeout 1500 python tools/options_sweep.py --out gpurun_out/options.jsonl > gpurun_out/options.log 2>&1; echo options=$?
timeout 900 python tools/transport_line.py > gpurun_out/tr_line.json 2> gpurun_out/tr_line.err; echo line=$?
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench=$?
python -c "import json;d=json.load(open('gpurun_out/bench.json'));print('value %.4e e2e %.4e (%.2f ms) walk %.3f transport %.4e'%(d['value'],d['e2e']['value'],d['e2e']['ms_per_step'],d['roofline']['kernel_ms_per_step'],d['transport']['value']))"
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo ref=$?
