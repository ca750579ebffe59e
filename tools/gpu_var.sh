# parity tests + walk-kernel launch-variant sweep (kernel-only bench lines)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x --timeout 600 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
tail -3 gpurun_out/pytest_gpu.log
for v in 1 6 2 5; do
  timeout 300 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --blocks-per-sm $v > gpurun_out/var_$v.json 2>&1
  python -c "import json;d=json.load(open('gpurun_out/var_$v.json'));print($v, d['value'], d['roofline']['kernel_ms_per_step'], d['clocks'])"
done
