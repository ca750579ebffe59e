# GPU session: parity tests, launch-config sweep, ncu launch list + full profile
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 300 python __graft_entry__.py > gpurun_out/smoke.log 2>&1; echo smoke=$?; tail -1 gpurun_out/smoke.log
timeout 1200 python -m pytest tests -m gpu -q --timeout 600 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
tail -15 gpurun_out/pytest_gpu.log
for b in 1 2 3; do for s in 1 0; do for w in 1 0; do
  timeout 300 python bench.py --steps 3 --warmup 2 --no-e2e --no-cpu-baseline --blocks-per-sm $b --sort $s --warp-agg $w > gpurun_out/sweep_b${b}_s${s}_w${w}.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/sweep_b${b}_s${s}_w${w}.json'));print('b=$b s=$s w=$w', '%.3e'%d['value'], '%.2f ms'%d['roofline']['kernel_ms_per_step'])"
done; done; done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/ncu_launch_bench.log 2>&1; echo ncu1=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:walk_kernel -s 3 -c 1 -o gpurun_out/walk_full python bench.py --steps 1 --warmup 2 --no-e2e --no-cpu-baseline > gpurun_out/ncu_full.log 2>&1; echo ncu2=$?
tail -3 gpurun_out/ncu_full.log
