cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 300 python __graft_entry__.py > gpurun_out/smoke.log 2>&1; echo smoke=$?; tail -1 gpurun_out/smoke.log
timeout 1200 python -m pytest tests -m gpu -q --timeout 600 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
tail -8 gpurun_out/pytest_gpu.log
for b in 1 2 3; do
  timeout 300 python bench.py --steps 3 --warmup 2 --no-e2e --no-cpu-baseline --blocks-per-sm $b > gpurun_out/fast_b${b}.json 2>gpurun_out/fast_b${b}.err
  python -c "import json;d=json.load(open('gpurun_out/fast_b${b}.json'));print('fast b=$b', '%.3e'%d['value'], '%.2f ms'%d['roofline']['kernel_ms_per_step'])"
done
