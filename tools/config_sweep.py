"""Time C2 (E envs, steps W..W+K-1) under config overrides: python tools/config_sweep.py E W K key=val[,key=val] ..."""
import sys, time
import numpy as np, torch
sys.path.insert(0, "/root/repo")
from paper_2504_12908_b200 import scenes as S, taccel as T
E, W, K = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
for spec in sys.argv[4:]:
    sc = S.make_scene("C2")
    for kv in filter(None, spec.split(",")):
        k, v = kv.split("=")
        setattr(sc.config, k, type(getattr(sc.config, k))(float(v)) if isinstance(getattr(sc.config, k), float) else int(v))
    ei = S.env_inputs(sc, np.arange(E), n_steps=W + K)
    b = T.Batch(sc, E)
    b.set_state(ei.x0, ei.y0)
    for k in range(W):
        b.set_targets(ei.ykin[k]); b.step(1)
    torch.cuda.synchronize()
    s0 = b.stats()
    b.profile(True); b.profile_read(reset=True)
    t = time.time(); fails = 0; newton = 0
    for k in range(W, W + K):
        b.set_targets(ei.ykin[k]); st = b.step(1); fails += int((st != 0).sum())
        newton += sum(x["newton_iters"] for x in b.stats())
    torch.cuda.synchronize(); dt = time.time() - t
    prof = b.profile_read(reset=True)
    s1 = b.stats()
    pcg = sum(x["pcg_iters_total"] - y["pcg_iters_total"] for x, y in zip(s1, s0))
    top = sorted(((k, v[0]) for k, v in prof.items() if v[1]), key=lambda kv: -kv[1])[:6]
    print(f"{spec or 'default':40s} {E*K/dt:8.1f} env-steps/s  {1e3*dt/K:7.1f} ms/step  fails {fails}  newton/env-step {newton/(E*K):.1f}"
          f"  pcg/env-step {pcg/(E*K):.0f}  " + " ".join(f"{k}={v/K:.0f}" for k, v in top), flush=True)
