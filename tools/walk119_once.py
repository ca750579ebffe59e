"""Two moves of 1e7 particles on the 10.1M-tet cube (C4 n=119, Σt = 2): an ncu capture target."""
import sys, math, torch
sys.path.insert(0, '.')
from paper_2504_19048_b200 import MeshTally, build_cube_mesh
n=10_000_000; dev=torch.device("cuda",0); g=torch.Generator(device=dev); g.manual_seed(3)
pos=0.05+0.9*torch.rand(n,3,generator=g,device=dev,dtype=torch.float64)
mu=2*torch.rand(n,generator=g,device=dev,dtype=torch.float64)-1; phi=2*math.pi*torch.rand(n,generator=g,device=dev,dtype=torch.float64)
s=torch.sqrt(1-mu*mu); d=torch.stack([s*torch.cos(phi),s*torch.sin(phi),mu],1)
dest=(pos-torch.log(torch.rand(n,generator=g,device=dev,dtype=torch.float64))[:,None]/2.0*d).contiguous()
fly=torch.ones(n,dtype=torch.int8,device=dev); w=torch.ones(n,dtype=torch.float64,device=dev)
mt=MeshTally(build_cube_mesh(119),n)
for _ in range(2):
    mt.initialize_particle_location(pos); mt.move_to_next_location(dest,fly,w)
torch.cuda.synchronize()
