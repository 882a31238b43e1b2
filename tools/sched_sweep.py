"""Time C2 in scheduled mode (E envs, W warm-up steps, K timed steps) under config overrides."""
import sys, time
import numpy as np, torch
sys.path.insert(0, "/root/repo")
from paper_2504_12908_b200 import scenes as S, taccel as T
E, W, K = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
for spec in sys.argv[4:] or [""]:
    sc = S.make_scene("C2")
    for kv in filter(None, spec.split(",")):
        k, v = kv.split("=")
        cur = getattr(sc.config, k)
        setattr(sc.config, k, type(cur)(float(v)) if isinstance(cur, float) else int(v))
    ei = S.env_inputs(sc, np.arange(E), n_steps=W + K)
    b = T.Batch(sc, E)
    b.set_state(ei.x0, ei.y0)
    yk = torch.tensor(ei.ykin, device="cuda")
    b.step_schedule(yk[:W])
    torch.cuda.synchronize()
    s0 = b.stats()
    b.profile(True); b.profile_read(reset=True)
    t = time.time()
    st = b.step_schedule(yk[W:W + K])
    torch.cuda.synchronize(); dt = time.time() - t
    prof = b.profile_read(reset=True)
    s1 = b.stats()
    pcg = sum(x["pcg_iters_total"] - y["pcg_iters_total"] for x, y in zip(s1, s0))
    top = sorted(((k, v[0]) for k, v in prof.items() if v[1]), key=lambda kv: -kv[1])[:7]
    n_it = prof["pcg"][1]
    act, ims = b.profile_iterations()
    q = len(act) // 8 or 1
    print("   active by octile:", [int(np.mean(act[i:i + q])) for i in range(0, len(act), q)],
          " ms by octile:", [round(sum(ims[i:i + q])) for i in range(0, len(ims), q)])
    print(f"{spec or 'default':34s} {E*K/dt:8.1f} env-steps/s {1e3*dt/K:6.1f} ms/step fails {int((st != 0).sum())} host-iters {n_it}"
          f" pcg/env-step {pcg/(E*K):.0f} | " + " ".join(f"{k}={v/K:.0f}" for k, v in top), flush=True)
