"""Relaxed PCG tolerance study (reading R24, NEXT 4): oracle steps (PCG solver) from dumped GPU states with
fixed η and with the Eisenstat–Walker forcing at several η_max; prints Newton / PCG counts and the position
difference against the fixed-η result (in L_env).

python tools/forcing_study.py gpurun_out/states_C2.npz env step [step ...]
"""
import dataclasses
import sys
import time

import numpy as np

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
from paper_2504_12908_b200 import scenes as S
from oracle import mesh as M
from oracle import solver as SO


def main(path, env, *steps):
    D = np.load(path)
    name = path.rsplit("states_", 1)[1].split(".")[0]
    sc0 = S.make_scene(name)
    st = list(D["steps"])
    x0 = D["x"][0][int(env)]; y0 = D["y"][0][int(env)]
    for k in map(int, steps):
        i = st.index(k)
        state = SO.State(D["x"][i][int(env)], D["v"][i][int(env)], D["y"][i][int(env)], D["ydot"][i][int(env)])
        ref = None
        for em in (0.0, 1e-2, 1e-1, 0.5):
            sc = S.make_scene(name)
            sc.config = dataclasses.replace(sc0.config, pcg_eta_max=em)
            mod = M.prepare(sc)
            L = M.env_scale(mod, x0, y0)
            t = time.time()
            new, stats = SO.step(mod, state, D["ykin"][i][int(env)], solver="pcg", L_env=L)
            P = M.all_positions(mod, new.x, new.y)
            d = 0.0 if ref is None else np.abs(P - ref).max() / L
            ref = P if ref is None else ref
            print(f"step {k} eta_max {em:g}: status {stats.status} newton {stats.newton_iters} pcg {stats.pcg_iters} "
                  f"al {stats.al_rounds} |dP|/L {d:.2e} ({time.time() - t:.0f}s)", flush=True)


if __name__ == "__main__":
    main(*sys.argv[1:])
