#!/bin/bash
# final check of the committed library: smoke, the GPU suite, the default bench line
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 300 python __graft_entry__.py > gpurun_out/smoke.log 2>&1; echo smoke=$?; tail -1 gpurun_out/smoke.log
timeout 1500 python -m pytest tests -x -q -m gpu -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?; tail -2 gpurun_out/pytest_gpu.log
timeout 600 python bench.py > gpurun_out/bench_check.json 2> gpurun_out/bench_check.err; echo bench=$?
python -c "import json;d=json.load(open('gpurun_out/bench_check.json'));print('value %.4e e2e %.4e (%.2f ms) walk %.3f launches %d opts %s'%(d['value'],d['e2e']['value'],d['e2e']['ms_per_step'],d['roofline']['kernel_ms_per_step'],d['gpu_launches'],d['config']['options']))"
