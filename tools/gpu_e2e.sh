cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q --timeout 600 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
tail -3 gpurun_out/pytest_gpu.log
for gd in 0.1667 0.5 1.0; do
  B200TALLY_GRID_DENSITY=$gd timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/e2e_gd${gd}.json 2>gpurun_out/e2e.err
  python -c "import json;d=json.load(open('gpurun_out/e2e_gd${gd}.json'));print('density=$gd value %.4e'%d['value'], 'e2e %.4e'%d['e2e']['value'], '%.2f ms'%d['e2e']['ms_per_step'], 'walk %.2f'%d['roofline']['kernel_ms_per_step'])"
done
B200TALLY_GRID_DENSITY=0.5 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_gd.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > /dev/null 2>&1; echo ncu=$?
