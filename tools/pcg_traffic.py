"""One C2 step (after W warm-up steps) inside cudaProfilerStart/Stop, for
`ncu --profile-from-start off -k regex:k_pcg_r --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum`.
Prints the algorithmic PCG bytes of that step (device counters) so traffic/algorithmic can be compared."""
import json, sys
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
s0 = b.stats()
b.set_targets(ei.ykin[W])
torch.cuda.synchronize()
torch.cuda.profiler.start()
b.step(1)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
s1 = b.stats()
alg = sum(x["pcg_alg_bytes_total"] - y["pcg_alg_bytes_total"] for x, y in zip(s1, s0))
its = sum(x["pcg_iters_total"] - y["pcg_iters_total"] for x, y in zip(s1, s0))
print("ALG", json.dumps({"alg_bytes_step": alg, "pcg_iters_step": its, "envs": E, "step": W}))
