"""PCG iteration distribution on C2 (lockstep tac_step, one step at a time): per env-step Newton and
PCG iterations, PCG per Newton iteration, active pairs; percentiles and the per-step maximum."""
import json, sys
import numpy as np
sys.path.insert(0, "/root/repo")
from paper_2504_12908_b200 import scenes as S, taccel as T
E = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
K = int(sys.argv[2]) if len(sys.argv) > 2 else 16
cfg = sys.argv[3] if len(sys.argv) > 3 else "C2"
sc = S.make_scene(cfg)
ei = S.env_inputs(sc, np.arange(E), n_steps=K)
b = T.Batch(sc, E)
b.set_state(ei.x0, ei.y0)
rows = []
for k in range(K):
    b.set_targets(ei.ykin[k])
    b.step(1)
    st = b.stats()
    nw = np.array([s["newton_iters"] for s in st]); pc = np.array([s["pcg_iters"] for s in st])
    na = np.array([s["n_active"] for s in st])
    act, ms = b.profile_iterations()
    per = pc / np.maximum(nw, 1)
    rows.append({"step": k, "newton_p50": float(np.median(nw)), "newton_max": int(nw.max()),
                 "pcg_step_p50": float(np.median(pc)), "pcg_step_p99": float(np.percentile(pc, 99)), "pcg_step_max": int(pc.max()),
                 "pcg_per_newton_p50": float(np.median(per)), "pcg_per_newton_p99": float(np.percentile(per, 99)),
                 "pcg_per_newton_max": float(per.max()), "n_active_p50": float(np.median(na)), "n_active_max": int(na.max()),
                 "iters_lockstep": len(act), "active_per_iter": act, "ms_per_iter": [round(x, 2) for x in ms]})
    print(json.dumps({kk: v for kk, v in rows[-1].items() if kk not in ("active_per_iter", "ms_per_iter")}), flush=True)
json.dump(rows, open("gpurun_out/pcg_dist.json", "w"))
