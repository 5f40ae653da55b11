import numpy as np, torch, sys, time
sys.path.insert(0,'.')
import synth, oracle, paper_2604_10357_b200 as T
def rel(a,b): return float(np.linalg.norm(a-b)/max(np.linalg.norm(b),1e-300))
for (nx,ny,nz,rule) in [(8,2,2,0),(6,4,3,1),(12,8,4,1)]:
    mesh=synth.kuhn_t10_box(nx,ny,nz,3,2,1)
    x,v,vn,fe=synth.t10_state(mesh)
    mat=dict(synth.SVK_PAPER)
    d=lambda a: None if a is None else torch.from_numpy(a).cuda()
    c1=T.Context.from_mesh(mesh,mat,rule)
    c0=T.Context.from_mesh(mesh,mat,rule,reference_layout="tables")
    print(mesh.name, "fused", c1.info["fused_eval"], "old", c0.info["fused_eval"])
    out=[]
    for name,c in (("tile",c1),("old",c0)):
        print(" eval", name, flush=True)
        g,H,f=c.empty_outputs()
        c.eval(d(x),d(v),d(vn),d(fe),1e-3,g,H,f); torch.cuda.synchronize()
        out.append((g.cpu().numpy(),H.cpu().numpy(),f.cpu().numpy()))
    pr=oracle.Problem(mesh,mat,rule)
    g0,H0,f0=pr.eval(x,v,vn,fe,1e-3)
    print(" tile vs oracle g/H/f", rel(out[0][0],g0), rel(out[0][1],H0), rel(out[0][2],f0))
    print(" old  vs oracle g/H/f", rel(out[1][0],g0), rel(out[1][1],H0), rel(out[1][2],f0))
