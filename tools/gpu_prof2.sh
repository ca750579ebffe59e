cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:walk_staged -s 2 -c 1 -o gpurun_out/walk_v1 python bench.py --steps 1 --warmup 2 --no-e2e --no-cpu-baseline > gpurun_out/ncu_v1.log 2>&1; echo ncu=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:transport_kernel -c 1 -o gpurun_out/transport python -c "
import sys; sys.path.insert(0,'.')
from paper_2504_19048_b200 import transport as T, build_cube_mesh
T.run(T.RunConfig(mesh_n=10, num_particles=1000000, num_batches=1, seed=42), build_cube_mesh(10))
" > gpurun_out/ncu_tr.log 2>&1; echo ncu_tr=$?
timeout 1200 compute-sanitizer --tool memcheck --leak-check full python -m pytest tests/test_gpu_parity.py -q -x -k "c1_point_s2 or straight_ray or error" -p no:cacheprovider > gpurun_out/memcheck.log 2>&1; echo memcheck=$?
grep -E "ERROR SUMMARY|passed|failed" gpurun_out/memcheck.log | tail -5
timeout 1200 compute-sanitizer --tool racecheck python -m pytest tests/test_gpu_callback.py -q -x -k cb_n6 -p no:cacheprovider > gpurun_out/racecheck.log 2>&1; echo racecheck=$?
grep -E "ERROR SUMMARY|RACECHECK SUMMARY|passed|failed" gpurun_out/racecheck.log | tail -5
