# kernel-only bench lines for each experimental library build x launch variant
# usage: bash tools/gpu_libvar.sh "r1c1 r0c0" "6 2 1"
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for lib in $1; do for v in $2; do
  BT_LIB_PATH=build/variants/libb200tally_$lib.so timeout 300 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --blocks-per-sm $v > gpurun_out/lv_${lib}_$v.json 2>&1
  python -c "import json;d=json.load(open('gpurun_out/lv_${lib}_$v.json'));print('$lib', $v, round(d['value']/1e9,3), round(d['roofline']['kernel_ms_per_step'],3), d['clocks']['sm_mhz'], d['clocks']['reasons'])" || tail -3 gpurun_out/lv_${lib}_$v.json
done; done
