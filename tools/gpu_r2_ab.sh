# A/B of the vertex/record load variants + parity of the new default
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
bash tools/gpu_ab.sh old xr8 vtx 2>&1 | tee gpurun_out/ab.log
timeout 1200 python -m pytest tests -m gpu -q -x --timeout 900 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
tail -5 gpurun_out/pytest_gpu.log
