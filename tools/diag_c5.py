"""C5 AL diagnostic: lockstep 128 envs until an env fails, then re-run that step for the failing env with a
Newton/AL trace (tac_debug_trace) and more AL rounds; prints the active pairs' bodies at the failure."""
import dataclasses
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2504_12908_b200 import scenes as S
from paper_2504_12908_b200 import taccel as T


def run(E=128, k_end=80, al_rounds=None, rho0=None):
    E, k_end = int(E), int(k_end)
    sc = S.make_scene("C5")
    over = {}
    if al_rounds:
        over["max_al_rounds"] = int(al_rounds)
    if rho0:
        over["al_rho0"] = float(rho0)
    if over:
        sc.config = dataclasses.replace(sc.config, **over)
    print("config", {k: getattr(sc.config, k) for k in ("al_rho0", "max_al_rounds", "al_tol_rel")}, flush=True)
    ei = S.env_inputs(sc, np.arange(E), n_steps=k_end)
    b = T.Batch(sc, E)
    assert (b.set_state(ei.x0, ei.y0) == 0).all()
    b.set_chain(S.hand_chain())
    yp = np.repeat(S.hand_palm_pose()[None], E, 0)
    scripts = np.stack([S.hand_script(e, k_end).reshape(k_end, -1) for e in range(E)], 1)
    qdev = torch.tensor(scripts, device="cuda")
    for k in range(k_end):
        prev = [t.clone() for t in b.get_state()]
        b.set_joint_targets(qdev[k], base=yp)
        st = b.step(1)
        ss = b.stats()
        bad = np.nonzero(st)[0]
        nw = np.array([s["newton_iters"] for s in ss])
        al = np.array([s["al_rounds"] for s in ss])
        print(k, "newton mean %.1f max %d" % (nw.mean(), nw.max()), "al max", al.max(), "failed", bad[:8], flush=True)
        if len(bad):
            e = int(bad[0])
            print("failed env", e, ss[e], flush=True)
            x, v, y, yd = (t.cpu().numpy() for t in prev)
            b1 = T.Batch(sc, 1)
            b1.set_state(x[e:e + 1], y[e:e + 1], v[e:e + 1], yd[e:e + 1])
            b1.set_chain(S.hand_chain())
            b1.set_joint_targets(qdev[k][e:e + 1], base=yp[:1])
            b1.debug_trace_start(0)
            s1 = b1.step(1)
            print("solo status", s1, b1.stats()[0], flush=True)
            for row in b1.debug_trace_read():
                print("   ", " ".join("%.4g" % v for v in row), flush=True)
            xs, _, ys, _ = (t.cpu().numpy()[0] for t in b1.get_state())
            pairs = b1.debug_active_pairs(0, xs, ys)
            print("active pairs", len(pairs), flush=True)
            break


if __name__ == "__main__":
    run(*[a for a in sys.argv[1:]])
