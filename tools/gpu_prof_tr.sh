# ncu full capture (with source) of one transport_kernel launch (paper physics, 1e6 histories);
# the run's events go to gpurun_out/tr_events.txt (for tools/ncu_walk_sol.py ... transport_sol.json)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:transport_kernel -c 1 -o gpurun_out/transport python -c "
import sys; sys.path.insert(0,'.')
from paper_2504_19048_b200 import transport as T, build_cube_mesh
r = T.run(T.RunConfig(mesh_n=10, num_particles=1000000, num_batches=1, seed=42), build_cube_mesh(10))
open('gpurun_out/tr_events.txt', 'w').write(f'{r.events} {r.collisions}\n')
" > gpurun_out/ncu_tr.log 2>&1; echo ncu_tr=$?; cat gpurun_out/tr_events.txt
