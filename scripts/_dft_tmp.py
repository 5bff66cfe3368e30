import sys
sys.path.insert(0, "/root/repo")
import torch
from fsfem_inputs import config_mesh
from paper_2001_08849_b200 import FsFem, fsfem_spmv
m = config_mesh(4)
g = FsFem(device=0, stream=torch.cuda.current_stream().cuda_stream)
g.build_faces(m.xyz, m.tets)
g.assemble_csr(1.0e6, 0.3)
x = torch.randn(3 * m.n_nodes, dtype=torch.float64, device="cuda")
y = torch.empty_like(x)
for _ in range(3):
    fsfem_spmv(g.ctx, x, y)
torch.cuda.synchronize()
print("=== timed", flush=True)
fsfem_spmv(g.ctx, x, y)
torch.cuda.synchronize()
