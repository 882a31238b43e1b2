"""Newton iterations per env-step of the CPU oracle on the first steps of a workload (env 0), for the
extrapolated oracle baseline of C3 (bench.py): an oracle C3 env-step takes minutes, so the bench times
oracle Newton iterations and converts with these counts.  Writes profiles/r2_oracle_newton_<cfg>.json."""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main(cfg="C3", n_steps=13, env=0):
    import torch
    torch.set_num_threads(1)
    from paper_2504_12908_b200 import scenes as S
    from oracle import mesh as M
    from oracle import solver as SO
    sc = S.make_scene(cfg)
    mod = M.prepare(sc)
    ei = S.env_inputs(sc, [env], n_steps=n_steps)
    st = SO.State(ei.x0[0].copy(), np.zeros_like(ei.x0[0]), ei.y0[0].copy(), np.zeros_like(ei.y0[0]))
    L = M.env_scale(mod, st.x, st.y)
    rows = []
    for k in range(n_steps):
        t0 = time.perf_counter()
        st, stats = SO.step(mod, st, ei.ykin[k, 0], L_env=L)
        rows.append({"step": k, "newton_iters": stats.newton_iters, "seconds": time.perf_counter() - t0,
                     "status": stats.status, "n_active": stats.n_active})
        print(rows[-1], flush=True)
        out = {"cfg": cfg, "env": env, "steps": rows,
               "what": "CPU oracle (1 thread, exact direct Newton solve): Newton iterations and seconds per env-step"}
        json.dump(out, open(os.path.join(ROOT, "profiles", f"r2_oracle_newton_{cfg}.json"), "w"), indent=1)


if __name__ == "__main__":
    main(*(sys.argv[1:2] or ["C3"]))
