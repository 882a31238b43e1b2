"""Run C2 for W steps, then wrap ONE step in cudaProfilerStart/Stop so that
`ncu --profile-from-start off --metrics gpu__time_duration.sum` lists every launch of that step."""
import sys
import numpy as np, torch
sys.path.insert(0, "/root/repo")
from paper_2504_12908_b200 import scenes as S, taccel as T
E = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
W = int(sys.argv[2]) if len(sys.argv) > 2 else 12
sc = S.make_scene("C2")
ei = S.env_inputs(sc, np.arange(E), n_steps=W + 1)
b = T.Batch(sc, E)
b.set_state(ei.x0, ei.y0)
for k in range(W):
    b.set_targets(ei.ykin[k]); b.step(1)
torch.cuda.synchronize()
b.set_targets(ei.ykin[W])
torch.cuda.profiler.start()
b.step(1)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
act, ms = b.profile_iterations()
print("active per iteration:", act)
