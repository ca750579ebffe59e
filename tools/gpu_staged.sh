cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q --timeout 600 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
tail -8 gpurun_out/pytest_gpu.log
for st in 1 0; do for b in 2 1; do
  timeout 300 python bench.py --steps 3 --warmup 2 --no-e2e --no-cpu-baseline --staged $st --blocks-per-sm $b > gpurun_out/st${st}_b${b}.json 2>gpurun_out/st${st}_b${b}.err
  python -c "import json;d=json.load(open('gpurun_out/st${st}_b${b}.json'));print('staged=$st b=$b', '%.3e'%d['value'], '%.2f ms'%d['roofline']['kernel_ms_per_step'])"
done; done
