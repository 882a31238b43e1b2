"""Dump GPU states of a few envs along the scripted episode (for the preconditioner study, NEXT 4).

python tools/dump_states.py C3 8 40 5   -> gpurun_out/states_C3.npz with x, v, y, ydot at steps 0, 5, ..., 40
(state BEFORE step k, plus the step's kinematic target) for envs 0..7, and the per-step Newton / PCG counts.
"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2504_12908_b200 import scenes as S
from paper_2504_12908_b200 import taccel as T


def main(cfg="C3", E=8, k_end=40, every=5):
    E, k_end, every = int(E), int(k_end), int(every)
    sc = S.make_scene(cfg)
    ei = S.env_inputs(sc, np.arange(E), n_steps=k_end + 1)
    b = T.Batch(sc, E)
    b.set_state(ei.x0, ei.y0)
    yk = torch.tensor(ei.ykin, device="cuda")
    out = {"steps": [], "x": [], "v": [], "y": [], "ydot": [], "ykin": [], "newton": [], "pcg": []}
    for k in range(k_end + 1):
        if k % every == 0 or k % every == 1:
            x, v, y, yd = (t.cpu().numpy() for t in b.get_state())
            out["steps"].append(k); out["x"].append(x); out["v"].append(v); out["y"].append(y); out["ydot"].append(yd)
            out["ykin"].append(ei.ykin[k])
        if k == k_end:
            break
        b.set_targets(yk[k])
        b.step(1)
        ss = b.stats()
        out["newton"].append([s["newton_iters"] for s in ss])
        out["pcg"].append([s["pcg_iters"] for s in ss])
        print(k, "newton", out["newton"][-1], "pcg", out["pcg"][-1], flush=True)
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    np.savez_compressed(os.path.join(ROOT, "gpurun_out", f"states_{cfg}.npz"), **{k: np.array(v) for k, v in out.items()})


if __name__ == "__main__":
    main(*sys.argv[1:])
