"""The one-launch small-mesh evaluation (k_eval_small) against the three-launch
path: runs the same evaluations with libtlfea.so and libtlfea_nosmall.so
(built with -DTLFEA_SMALL_MAX_EL=0) and checks g, H, f bitwise equal."""
import os, sys, numpy as np, torch
sys.path.insert(0, os.getcwd())
import synth
res = {}
for lib in ["paper_2604_10357_b200/libtlfea.so", "paper_2604_10357_b200/libtlfea_nosmall.so"]:
    import subprocess, json
    code = f'''
import os, sys, numpy as np, torch
os.environ["TLFEA_LIB"] = "{lib}"
sys.path.insert(0, os.getcwd())
import paper_2604_10357_b200 as T, synth
out = {{}}
for name, mesh, rule in [("cfg1", synth.config(1).mesh, 0), ("k6x4x3", synth.kuhn_t10_box(6, 4, 3, 0.6, 0.4, 0.3), 1), ("k10x7x7", synth.kuhn_t10_box(10, 7, 7, 1.0, 0.7, 0.7), 1)]:
    x, v, vn, fe = synth.t10_state(mesh, with_fext=True)
    ctx = T.Context.from_mesh(mesh, dict(synth.SVK_PAPER), rule)
    d = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
    g, H, f = ctx.empty_outputs()
    ctx.eval(d(x), d(v), d(vn), d(fe), 1e-3, g, H, f)
    torch.cuda.synchronize()
    np.save(f"/tmp/{{name}}_{os.path.basename(lib)}.npy", np.concatenate([g.cpu().numpy(), H.cpu().numpy(), f.cpu().numpy()]))
    out[name] = ctx.info["fused_eval"]
print(out)
'''
    print(lib, subprocess.run([sys.executable, "-c", code], capture_output=True, text=True).stdout.strip())
for name in ["cfg1", "k6x4x3", "k10x7x7"]:
    a = np.load(f"/tmp/{name}_libtlfea.so.npy"); b = np.load(f"/tmp/{name}_libtlfea_nosmall.so.npy")
    print(name, "bitwise equal:", np.array_equal(a, b), float(np.abs(a - b).max()))
