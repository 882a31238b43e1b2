"""Full C2 episode in scheduled mode: failures and throughput over all 200 steps (+ invariant spot checks)."""
import sys, time
import numpy as np, torch
sys.path.insert(0, "/root/repo")
from paper_2504_12908_b200 import scenes as S, taccel as T
name = sys.argv[1] if len(sys.argv) > 1 else "C2"
E = int(sys.argv[2]) if len(sys.argv) > 2 else 1024
NS = int(sys.argv[3]) if len(sys.argv) > 3 else 200
CH = int(sys.argv[4]) if len(sys.argv) > 4 else 40
sc = S.make_scene(name)
t0 = time.time()
ei = S.env_inputs(sc, np.arange(E), n_steps=NS)
print(f"inputs {time.time() - t0:.1f}s", flush=True)
b = T.Batch(sc, E)
print("workspace GB", b.workspace.numel() / 1e9, "set_state", np.unique(b.set_state(ei.x0, ei.y0), return_counts=True))
yk = torch.tensor(ei.ykin, device="cuda")
for k0 in range(0, NS, CH):
    t = time.time()
    st = b.step_schedule(yk[k0:k0 + CH])
    torch.cuda.synchronize()
    dt = time.time() - t
    s = b.stats()
    print(f"steps {k0}-{k0 + CH - 1}: {E * CH / dt:8.1f} env-steps/s  status {dict(zip(*np.unique(st, return_counts=True)))}"
          f"  newton(last) max {max(x['newton_iters'] for x in s)}  nact max {max(x['n_active'] for x in s)}"
          f"  ncand max {max(x['n_candidates'] for x in s)}", flush=True)
