#!/bin/bash
# Bulk (TMA) direct refill variant: parity tests through it, then walk times
# against the in-tree library on the L2- and HBM-resident meshes
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
V=build/variants/libb200tally_bulk.so
BT_LIB_PATH=$V timeout 1200 python -m pytest -q -x -p no:cacheprovider -m gpu tests/test_gpu_parity.py tests/test_gpu_api.py tests/test_gpu_multi.py > gpurun_out/bulk_tests.log 2>&1; echo tests=$?; tail -3 gpurun_out/bulk_tests.log
for r in 1 2; do
  for v in default bulk; do
    if [ "$v" = default ]; then lib=""; else lib=$V; fi
    for p in "2 55" "100 55" "10 55" "2 95" "2 119"; do
      read sg nc <<< "$p"
      echo -n "r$r $v "; BT_LIB_PATH=$lib timeout 300 python tools/variant_walk.py $sg 0 $nc
    done
  done
done
BT_LIB_PATH=$V timeout 1500 compute-sanitizer --print-limit 20 --tool memcheck --leak-check no python -m pytest -q -p no:cacheprovider -m gpu \
  tests/test_gpu_api.py "tests/test_gpu_parity.py::test_ragged_moves_and_edge_inputs" -k "not two_gpus" > gpurun_out/bulk_mem.log 2>&1; echo mem=$?; tail -2 gpurun_out/bulk_mem.log
BT_LIB_PATH=$V timeout 900 compute-sanitizer --tool racecheck python -m pytest -q -p no:cacheprovider -m gpu "tests/test_gpu_parity.py::test_ragged_moves_and_edge_inputs" > gpurun_out/bulk_race.log 2>&1; echo race=$?; tail -2 gpurun_out/bulk_race.log
