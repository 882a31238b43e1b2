"""Per-phase latency with few envs (the lockstep tail regime): ms per launch of each phase."""
import sys, time
import numpy as np, torch
sys.path.insert(0, "/root/repo")
from paper_2504_12908_b200 import scenes as S, taccel as T
E = int(sys.argv[1]) if len(sys.argv) > 1 else 8
NS = int(sys.argv[2]) if len(sys.argv) > 2 else 14
sc = S.make_scene("C2")
ei = S.env_inputs(sc, np.arange(E), n_steps=NS)
b = T.Batch(sc, E)
b.set_state(ei.x0, ei.y0)
for k in range(NS - 4):
    b.set_targets(ei.ykin[k]); b.step(1)
b.profile(True); b.profile_read(reset=True)
t = time.time()
for k in range(NS - 4, NS):
    b.set_targets(ei.ykin[k]); b.step(1)
torch.cuda.synchronize()
wall = time.time() - t
prof = b.profile_read(reset=True)
tot = sum(v[0] for v in prof.values())
print(f"E={E} wall {wall*1e3:.0f} ms for 4 steps, device phase sum {tot:.0f} ms")
for k, (ms, n) in sorted(prof.items(), key=lambda kv: -kv[1][0]):
    if n:
        print(f"  {k:14s} {ms:9.1f} ms  {n:6d} launches  {1e3*ms/n:8.1f} us/launch")
s = b.stats()
print("pcg per newton", sum(x["pcg_iters"] for x in s) / max(1, sum(x["newton_iters"] for x in s)))
