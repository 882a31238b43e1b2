"""One lockstep step of a workload (after W warm-up steps) inside cudaProfilerStart/Stop, for
`ncu --profile-from-start off -k regex:'^k_pcg' --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum`.
Prints the device-counted algorithmic PCG bytes of that step so DRAM traffic / algorithmic bytes can be compared.

  python tools/pcg_traffic.py CFG E W"""
import json, os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2504_12908_b200 import scenes as S, taccel as T
cfg = sys.argv[1] if len(sys.argv) > 1 else "C2"
E = int(sys.argv[2]) if len(sys.argv) > 2 else 1024
W = int(sys.argv[3]) if len(sys.argv) > 3 else 12
sc = S.make_scene(cfg)
ei = S.env_inputs(sc, np.arange(E), n_steps=W + 1)
b = T.Batch(sc, E)
b.set_state(ei.x0, ei.y0)
yk = torch.tensor(ei.ykin, device="cuda")
for k in range(W):
    b.set_targets(yk[k]); b.step(1)
s0 = b.stats()
b.set_targets(yk[W])
torch.cuda.synchronize()
torch.cuda.profiler.start()
b.step(1)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
s1 = b.stats()
alg = sum(x["pcg_alg_bytes_total"] - y["pcg_alg_bytes_total"] for x, y in zip(s1, s0))
its = sum(x["pcg_iters_total"] - y["pcg_iters_total"] for x, y in zip(s1, s0))
print("ALG", json.dumps({"cfg": cfg, "kernel": b.pcg_kernel, "alg_bytes_step": alg, "pcg_iters_step": its, "envs": E, "step": W}))
