# perf iteration: parity tests, variant sweep, ncu full of the default walk
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x --timeout 600 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
tail -3 gpurun_out/pytest_gpu.log
for v in ${VARIANTS:-1 4 6}; do
  timeout 300 python bench.py --steps 3 --warmup 2 --no-e2e --no-cpu-baseline --blocks-per-sm $v > gpurun_out/perf_v${v}.json 2>gpurun_out/perf_v${v}.err
  python -c "import json;d=json.load(open('gpurun_out/perf_v${v}.json'));print('variant=$v', '%.4e'%d['value'], '%.2f ms'%d['roofline']['kernel_ms_per_step'])"
done
if [ -n "$NCU" ]; then
timeout 900 ncu --set full --clock-control none --import-source on -k regex:walk_staged -s 2 -c 1 -o gpurun_out/walk_prof python bench.py --steps 1 --warmup 2 --no-e2e --no-cpu-baseline > gpurun_out/ncu_full.log 2>&1; echo ncu=$?
fi
