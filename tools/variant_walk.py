import sys, math, torch
sys.path.insert(0, '.')
from paper_2504_19048_b200 import MeshTally, _lib, build_cube_mesh
n=10_000_000; sig=float(sys.argv[1]); v=int(sys.argv[2]); ncube=int(sys.argv[3]) if len(sys.argv)>3 else 55
dev=torch.device("cuda",0); g=torch.Generator(device=dev); g.manual_seed(3)
pos=0.05+0.9*torch.rand(n,3,generator=g,device=dev,dtype=torch.float64)
mu=2*torch.rand(n,generator=g,device=dev,dtype=torch.float64)-1; phi=2*math.pi*torch.rand(n,generator=g,device=dev,dtype=torch.float64)
s=torch.sqrt(1-mu*mu); d=torch.stack([s*torch.cos(phi),s*torch.sin(phi),mu],1)
dest=(pos-torch.log(torch.rand(n,generator=g,device=dev,dtype=torch.float64))[:,None]/sig*d).contiguous()
fly=torch.ones(n,dtype=torch.int8,device=dev); w=torch.ones(n,dtype=torch.float64,device=dev)
mt=MeshTally(build_cube_mesh(ncube),n); mt.set_option(_lib.BT_OPT_BLOCKS_PER_SM, v)
ts=[]
for _ in range(4):
    mt.initialize_particle_location(pos); r=mt.move_to_next_location(dest,fly,w); ts.append(mt.last_timing()[0])
print(f"n={ncube} sigma={sig} variant={v} walk_ms={min(ts[1:]):.3f}")
