import sys, time, numpy as np, torch
sys.path.insert(0, "/root/repo")
from paper_2504_12908_b200 import scenes as S, taccel as T
sc = S.make_scene("C2")
E = 16
ei = S.env_inputs(sc, np.arange(E), n_steps=14)
b = T.Batch(sc, E)
print("set_state", b.set_state(ei.x0, ei.y0))
for k in range(14):
    b.set_targets(ei.ykin[k]); t=time.time(); st = b.step(1); torch.cuda.synchronize()
    s = b.stats()
    print(k, f"{time.time()-t:.2f}s", "status", st.tolist())
    print("   newton", [x["newton_iters"] for x in s], "al", [x["al_rounds"] for x in s])
    print("   pcg", [x["pcg_iters"] for x in s])
    print("   nact", [x["n_active"] for x in s], "ncand", [x["n_candidates"] for x in s])
    print("   res", ["%.1e" % x["constraint_residual"] for x in s[:6]], "amin", ["%.1e" % x["alpha_min"] for x in s[:6]])
