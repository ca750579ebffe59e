# full bench lines for experimental library builds: bash tools/gpu_libbench.sh "libA libB" "bench args"
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for lib in $1; do
  BT_LIB_PATH=build/variants/libb200tally_$lib.so timeout 300 python bench.py --no-cpu-baseline $2 > gpurun_out/lb_$lib.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/lb_$lib.json')); print('$lib', round(d['value']/1e9,3), round(d['ms_per_step'],3), round(d['roofline']['kernel_ms_per_step'],3), round(d['e2e']['value']/1e9,3), round(d['e2e']['ms_per_step'],3))"
done
