"""Per-section clock64 cycles of one k_pcg iteration (thread 0 of each CTA, averaged over iterations).
Needs the instrumented build: nvcc ... -DTAC_CLOCKS (see tools/build_clocks.sh); usage: pcg_clocks.py E W K."""
import ctypes, sys
import numpy as np, torch
sys.path.insert(0, "/root/repo")
from paper_2504_12908_b200 import scenes as S, taccel as T
T.LIB_PATH = T.LIB_PATH.replace("libtaccel_cuda.so", "libtaccel_cuda_clk.so")   # the -DTAC_CLOCKS build
E, W, K = (int(a) for a in sys.argv[1:4])
CFG = sys.argv[4] if len(sys.argv) > 4 else "C2"
NAMES = ["zero+sync", "pass A (pairs, couplings)", "B2 barrier", "soft rows", "body rows", "dAd warp sum", "B3 wait", "update+precond+rz", "B4 wait", "beta, d upd, B1"]
sc = S.make_scene(CFG)
ei = S.env_inputs(sc, np.arange(E), n_steps=W + K)
b = T.Batch(sc, E)
b.set_state(ei.x0, ei.y0)
yk = torch.tensor(ei.ykin, device="cuda")
for k in range(W):
    b.set_targets(yk[k]); b.step(1)
lib = T.load()
buf = (ctypes.c_ulonglong * 32)()
lib.tac_debug_clocks(buf)
for k in range(W, W + K):
    b.set_targets(yk[k]); b.step(1)
lib.tac_debug_clocks(buf)
n = buf[15]
tot = sum(buf[i] for i in range(10))
print(f"E={E}: {n} CTA-iterations, {tot / max(n, 1):.0f} cycles/iteration")
for i, nm in enumerate(NAMES):
    print(f"  {nm:16s} {buf[i] / max(n, 1):9.0f} cyc  {100 * buf[i] / max(tot, 1):5.1f}%")
na = max(buf[14], 1)
print(f"k_assemble: {buf[14]} CTA launches")
for i, nm in zip(range(10, 14), ["edge blocks", "vertex loop", "body warps", "body pair terms"]):
    print(f"  {nm:16s} {buf[i] / na:9.0f} cyc")
print(f"  vertex loop split: phase 1 {buf[16] / na:9.0f}  phase 2 {buf[17] / na:9.0f} cyc (phase 3 = rest)")
s = b.stats()
print("n_active mean", np.mean([x["n_active"] for x in s]), "max", max(x["n_active"] for x in s))
