#!/bin/bash
# Async direct refill vs HEAD: alternating bench A/B, short-move walk times,
# then memcheck over the API tests (the padded 4-byte flag copies)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
bash tools/gpu_ab.sh head
for v in default head; do
  if [ "$v" = default ]; then lib=""; else lib=build/variants/libb200tally_$v.so; fi
  for s in 100 10; do echo -n "$v "; BT_LIB_PATH=$lib timeout 300 python tools/variant_walk.py $s 0; done
done
timeout 1500 compute-sanitizer --print-limit 20 --tool memcheck --leak-check no python -m pytest -q -p no:cacheprovider -m gpu \
  tests/test_gpu_api.py "tests/test_gpu_parity.py::test_ragged_moves_and_edge_inputs" -k "not two_gpus" \
  > gpurun_out/async_mem.log 2>&1; echo mem=$?; tail -3 gpurun_out/async_mem.log
grep -c "========= ERROR\|Invalid" gpurun_out/async_mem.log
timeout 1200 python -m pytest -q -x -p no:cacheprovider -m gpu tests > gpurun_out/async_gpu_tests.log 2>&1; echo gpu_tests=$?; tail -3 gpurun_out/async_gpu_tests.log
