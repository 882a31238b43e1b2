"""GPU diagnostics (round 2): capacity detection per env, C3 failing env, cluster PCG plan."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import dataclasses
from paper_2504_12908_b200 import scenes as S
from paper_2504_12908_b200 import taccel as T


def capacity():
    sc = S.make_scene("C1")
    sc.config = dataclasses.replace(sc.config, cand_capacity_per_env=64)
    ei = S.env_inputs(sc, range(2), n_steps=2)
    y0 = ei.y0.copy()
    y0[1, 1, 2] += 20e-3
    y0[0, 1, 2] -= 0.2e-3 - 0.04e-3
    b = T.Batch(sc, 2)
    print("set_state", b.set_state(ei.x0, y0))
    for s in b.stats():
        print({k: s[k] for k in ("status", "n_candidates", "n_active")})
    b2 = T.Batch(S.make_scene("C1"), 2)
    print("default-capacity set_state", b2.set_state(ei.x0, y0))
    for s in b2.stats():
        print({k: s[k] for k in ("status", "n_candidates", "n_active")})


def c3_fail(k_end=38):
    sc = S.make_scene("C3")
    E = 4096
    ei = S.env_inputs(sc, np.arange(E), n_steps=k_end)
    b = T.Batch(sc, E)
    print("pcg kernel", b.pcg_kernel, flush=True)
    b.set_state(ei.x0, ei.y0)
    yk = torch.tensor(ei.ykin, device="cuda")
    for k in range(k_end):
        b.set_targets(yk[k])
        st = b.step(1)
        ss = b.stats()
        nw = np.array([s["newton_iters"] for s in ss])
        bad = np.nonzero(st)[0]
        print(k, "newton mean %.1f max %d argmax %d" % (nw.mean(), nw.max(), nw.argmax()), "failed", bad[:8], flush=True)
        for e in bad[:3]:
            print("   ", e, ss[e])
        if len(bad):
            break


if __name__ == "__main__":
    which = sys.argv[1] if len(sys.argv) > 1 else "capacity"
    {"capacity": capacity, "c3": c3_fail}[which]()
