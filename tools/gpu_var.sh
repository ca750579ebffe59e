cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x --timeout 600 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
tail -3 gpurun_out/pytest_gpu.log
for v in 1 2 4 5 6; do for so in 0 1; do
  timeout 300 python bench.py --steps 3 --warmup 2 --no-e2e --no-cpu-baseline --blocks-per-sm $v --sort $so > gpurun_out/var_${v}_s${so}.json 2>gpurun_out/var_${v}.err
  python -c "import json;d=json.load(open('gpurun_out/var_${v}_s${so}.json'));print('variant=$v sort=$so', '%.3e'%d['value'], '%.2f ms'%d['roofline']['kernel_ms_per_step'])"
done; done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:walk_staged -s 2 -c 1 -o gpurun_out/walk_fast_full python bench.py --steps 1 --warmup 2 --no-e2e --no-cpu-baseline > gpurun_out/ncu_full.log 2>&1; echo ncu=$?
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench=$?; cat gpurun_out/bench.json
