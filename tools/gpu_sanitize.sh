# compute-sanitizer pass over the final library: smoke under memcheck / racecheck / synccheck,
# then memcheck over a spread of small GPU tests (multi handle, API paths, grid localization,
# callback path, transport, GPU adjacency) and racecheck over the refill options
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
CS="compute-sanitizer --print-limit 20"
for t in memcheck racecheck synccheck; do
  extra=""; [ $t = memcheck ] && extra="--leak-check no"
  timeout 900 $CS --tool $t $extra python __graft_entry__.py > gpurun_out/san_smoke_$t.log 2>&1; echo smoke_$t=$?; tail -2 gpurun_out/san_smoke_$t.log
done
timeout 2400 $CS --tool memcheck --leak-check no python -m pytest -q -p no:cacheprovider -m gpu \
  tests/test_gpu_multi.py tests/test_gpu_api.py tests/test_gpu_callback.py tests/test_transport_gpu.py \
  "tests/test_gpu_parity.py::test_grid_localize_random_meshes" "tests/test_gpu_parity.py::test_localize_pathologies" \
  "tests/test_gpu_parity.py::test_ragged_moves_and_edge_inputs" \
  -k "not two_gpus" > gpurun_out/san_mem_tests.log 2>&1; echo mem_tests=$?; tail -4 gpurun_out/san_mem_tests.log
grep -c "========= ERROR\|Invalid" gpurun_out/san_mem_tests.log
timeout 1800 $CS --tool racecheck python -m pytest -q -p no:cacheprovider -m gpu tests/test_gpu_parity.py -k "options_keep_parity or ragged" > gpurun_out/san_race_tests.log 2>&1; echo race_tests=$?; tail -4 gpurun_out/san_race_tests.log
