import numpy as np, torch, sys
sys.path.insert(0,'.')
import synth, oracle, paper_2604_10357_b200 as T
sys.path.insert(0,'tests')
from test_gpu_parity import CASES, state
mesh, mat, rule = CASES["t10_single_element_svk"]()
x, v, vn, fext = state(mesh)
d=lambda a: None if a is None else torch.from_numpy(np.ascontiguousarray(a)).cuda()
gs=[]
for rep in range(3):
    c=T.Context.from_mesh(mesh,mat,rule,gravity=(0,-9.81,0.3))
    g,H,f=c.empty_outputs(); g.fill_(12345.0); f.fill_(12345.0)
    c.eval(d(x),d(v),d(vn),d(fext),1e-3,g,H,f); torch.cuda.synchronize()
    print(rep, "info", c.info["fused_eval"], "unwritten g", np.where(g.cpu().numpy()==12345.0)[0], "f", np.where(f.cpu().numpy()==12345.0)[0])
