# ncu full capture (with source) of one transport_kernel launch (paper physics, 1e6 histories)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:transport_kernel -c 1 -o gpurun_out/transport python -c "
import sys; sys.path.insert(0,'.')
from paper_2504_19048_b200 import transport as T, build_cube_mesh
T.run(T.RunConfig(mesh_n=10, num_particles=1000000, num_batches=1, seed=42), build_cube_mesh(10))
" > gpurun_out/ncu_tr.log 2>&1; echo ncu_tr=$?
