# deferred initialize: parity + e2e
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_api.py tests/test_gpu_parity.py -q -x --timeout 900 -p no:cacheprovider > gpurun_out/pytest_api.log 2>&1; echo api=$?
tail -15 gpurun_out/pytest_api.log
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench=$?; python -c "
import json; d=json.load(open('gpurun_out/bench.json')); print('value %.4e kernel %.3f step %.3f e2e %.4e (%.2f ms) pageable %.4e (%.2f ms)' % (d['value'], d['roofline']['kernel_ms_per_step'], d['ms_per_step'], d['e2e']['value'], d['e2e']['ms_per_step'], d['e2e']['pageable']['value'], d['e2e']['pageable']['ms_per_step']))"
tail -3 gpurun_out/bench.err
