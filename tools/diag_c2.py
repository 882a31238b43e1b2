"""Diagnostic: run a C2 batch and print per-step status histograms and iteration statistics."""
import sys, time, collections
import numpy as np, torch
sys.path.insert(0, "/root/repo")
from paper_2504_12908_b200 import scenes as S, taccel as T
E = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
NS = int(sys.argv[2]) if len(sys.argv) > 2 else 23
sc = S.make_scene("C2")
ei = S.env_inputs(sc, np.arange(E), n_steps=NS)
b = T.Batch(sc, E)
print("set_state", collections.Counter(b.set_state(ei.x0, ei.y0).tolist()))
first_fail = {}
for k in range(NS):
    b.set_targets(ei.ykin[k]); t = time.time(); st = b.step(1); torch.cuda.synchronize()
    s = b.stats()
    new = [i for i, x in enumerate(st.tolist()) if x != 0 and i not in first_fail]
    for i in new:
        first_fail[i] = (k, int(st[i]), s[i]["newton_iters"], s[i]["n_active"], s[i]["n_candidates"], s[i]["al_rounds"],
                         ["%.3e" % v for v in s[i]["diag"]])
    nw = np.array([x["newton_iters"] for x in s]); pc = np.array([x["pcg_iters"] for x in s])
    print(k, f"{time.time()-t:.2f}s", dict(collections.Counter(st.tolist())), "newton max/mean %d/%.1f" % (nw.max(), nw.mean()),
          "pcg max/mean %d/%.0f" % (pc.max(), pc.mean()), "nact max", max(x["n_active"] for x in s),
          "ncand max", max(x["n_candidates"] for x in s), flush=True)
    act, ms = b.profile_iterations()
    print("    iters", len(act), "active:", act[:12], "... ms:", ["%.1f" % v for v in ms[:12]], "... tail ms/iter %.2f" %
          (sum(ms[12:]) / max(len(ms) - 12, 1)), "bulk(first 12) %.0f ms, tail %.0f ms" % (sum(ms[:12]), sum(ms[12:])))
print("first failures (step, status, newton, nact, ncand, al):")
for i, v in list(first_fail.items())[:30]:
    print("  env", i, v)
