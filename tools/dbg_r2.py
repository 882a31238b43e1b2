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


def pcg():
    """debug_pcg with the cluster kernel vs the oracle PCG, per block (C1 press, C2)."""
    from oracle import contact as C, energy as En, mesh as M, solver as SO
    for name in ("C1", "C2"):
        sc = S.make_scene(name)
        mod = M.prepare(sc)
        ei = S.env_inputs(sc, [0], n_steps=1)
        rng = np.random.default_rng(11)
        xn, yn = ei.x0[0], ei.y0[0]
        v = rng.normal(size=xn.shape) * 1e-3
        x = xn + rng.normal(size=xn.shape) * 2e-5
        y = yn.copy()
        if name == "C1":
            y[1, 2] -= 0.2e-3 - 0.04e-3
        ctx = En.make_context(mod, xn, v, yn, np.zeros_like(yn), ei.ykin[0, 0], sc.config.dt)
        b = T.Batch(sc, 1)
        b.set_state(xn[None], yn[None], v[None])
        b.set_targets(ei.ykin[0])
        print(name, "kernel", b.pcg_kernel)
        p_gpu, it, mu = b.debug_pcg(0, x, y, with_mu=True)
        pairs = C.active_pairs(mod, M.all_positions(mod, x, y))
        g, H = En.assemble(mod, ctx, x, y, pairs)
        p_ref, it_ref = SO.block_jacobi_pcg(mod, H, g, sc.config.pcg_eta, sc.config.max_pcg)
        V = mod.V
        d = np.abs(p_gpu - p_ref)
        print("  it", it, it_ref, "mu", mu, "max|p|", np.abs(p_ref).max(), "soft diff", d[:3 * V].max(), "body diff", d[3 * V:].max() if len(d) > 3 * V else 0)
        print("  body gpu", p_gpu[3 * V:3 * V + 12])
        print("  body ref", p_ref[3 * V:3 * V + 12])
        print("  argmax", d.argmax(), p_gpu[d.argmax()], p_ref[d.argmax()])


def trace(name="C3", k_end=37, E=4096):
    """Lockstep to step k_end; run step k_end once to find the slowest env, restore the state, trace that
    env's Newton iterations while re-running the step."""
    sc = S.make_scene(name)
    ei = S.env_inputs(sc, np.arange(E), n_steps=k_end + 1)
    b = T.Batch(sc, E)
    b.set_state(ei.x0, ei.y0)
    yk = torch.tensor(ei.ykin, device="cuda")
    for k in range(k_end):
        b.set_targets(yk[k])
        b.step(1)
    x, xd, y, yd = b.get_state()
    b.set_targets(yk[k_end])
    b.step(1)
    nw = np.array([s["newton_iters"] for s in b.stats()])
    e = int(nw.argmax())
    print("step", k_end, "slowest env", e, "newton", nw[e], "p50", np.median(nw), flush=True)
    b.set_state(x[e:e + 1], y[e:e + 1], xd[e:e + 1], yd[e:e + 1], env0=e)
    b.set_targets(yk[k_end][e:e + 1], env0=e)
    b.debug_trace_start(e, 4096)
    b.step(1)
    rows = b.debug_trace_read(4096)
    print("newton pcg mu p_inf gm gp alpha E0 E1 bt")
    for r in rows:
        print(" ".join("%.4g" % v for v in r), flush=True)


def sanity():
    """Small runs through every kernel family, for compute-sanitizer: C2 lockstep + schedule (resident PCG),
    C3 one step (streamed PCG with the ELL copy), C1 with friction + depth maps, C5 with device FK."""
    import dataclasses
    sched(E=4, K=6)
    sc = S.make_scene("C3")
    ei = S.env_inputs(sc, np.arange(2), n_steps=1)
    b = T.Batch(sc, 2)
    b.set_state(ei.x0, ei.y0)
    b.set_targets(ei.ykin[0])
    print("C3", b.pcg_kernel, b.step(1), flush=True)
    sc = S.make_scene("C1")
    sc.config = dataclasses.replace(sc.config, mu_friction=0.5)
    ei = S.env_inputs(sc, np.arange(2), n_steps=3)
    b = T.Batch(sc, 2)
    b.set_state(ei.x0, ei.y0)
    for k in range(3):
        b.set_targets(ei.ykin[k])
        print("C1 friction", b.step(1), flush=True)
    d, n = b.get_depth_maps(12, 16)
    print("depth max", float(torch.nan_to_num(d).max()), flush=True)
    sc = S.make_scene("C5")
    ei = S.env_inputs(sc, np.arange(2), n_steps=2)
    b = T.Batch(sc, 2)
    b.set_state(ei.x0, ei.y0)
    b.set_chain(S.hand_chain())
    for k in range(2):
        q = np.stack([S.hand_script(e, 2)[k].reshape(-1) for e in range(2)])
        b.set_joint_targets(q, base=np.repeat(S.hand_palm_pose()[None], 2, 0))
        print("C5", b.step(1), flush=True)


def sched(E=8, K=12):
    sc = S.make_scene("C2")
    ei = S.env_inputs(sc, np.arange(E), n_steps=K)
    b = T.Batch(sc, E)
    b.set_state(ei.x0, ei.y0)
    yk = torch.tensor(ei.ykin, device="cuda")
    for k in range(K // 2):
        b.set_targets(yk[k])
        print("lockstep", k, b.step(1), flush=True)
    print("schedule", b.step_schedule(yk[K // 2:]), flush=True)


def grasp(name="C4:0", E=256, k_end=30):
    """Lockstep a grasp workload; on a failure print the env's stats (capacity flags)."""
    sc = S.make_scene(name)
    ei = S.env_inputs(sc, np.arange(E), n_steps=k_end)
    b = T.Batch(sc, E)
    print("set_state", np.unique(b.set_state(ei.x0, ei.y0), return_counts=True), flush=True)
    chain = name == "C5"
    if chain:
        b.set_chain(S.hand_chain())
        q = torch.tensor(np.stack([S.hand_script(e, k_end).reshape(k_end, -1) for e in range(E)], 1), device="cuda")
        yp = np.repeat(S.hand_palm_pose()[None], E, 0)
    yk = torch.tensor(ei.ykin, device="cuda")
    for k in range(k_end):
        if chain:
            b.set_joint_targets(q[k], base=yp)
        else:
            b.set_targets(yk[k])
        st = b.step(1)
        ss = b.stats()
        bad = np.nonzero(st)[0]
        nc = np.array([s["n_candidates"] for s in ss]); na = np.array([s["n_active"] for s in ss])
        print(k, "cand max", nc.max(), "active max", na.max(), "newton max", max(s["newton_iters"] for s in ss), "failed", bad[:6], flush=True)
        for e in bad[:2]:
            print("   ", e, ss[e], flush=True)
        if len(bad):
            break


def iters(name="C2", E=1024, k_end=12):
    """Per Newton iteration of lockstep step k_end: envs still active and host wall ms; phase split of
    that step (CUDA events)."""
    sc = S.make_scene(name)
    ei = S.env_inputs(sc, np.arange(E), n_steps=k_end + 1)
    b = T.Batch(sc, E)
    b.set_state(ei.x0, ei.y0)
    yk = torch.tensor(ei.ykin, device="cuda")
    for k in range(k_end):
        b.set_targets(yk[k])
        b.step(1)
    b.set_targets(yk[k_end])
    b.profile(True)
    b.profile_read(reset=True)
    b.step(1)
    prof = b.profile_read(reset=True)
    act, ms = b.profile_iterations()
    print("step", k_end, "iterations", len(act), "total ms %.1f" % sum(ms))
    for i, (a, m) in enumerate(zip(act, ms)):
        print("  it %3d active %5d  %.3f ms" % (i, a, m))
    print({k: (round(v[0], 2), v[1]) for k, v in prof.items() if v[1]})


def tail(name="C2", E=1024, k_end=12):
    """Lockstep steps 0..k_end of `name`; per step the slowest envs' stats; then the oracle traces the
    slowest env's step from the shared GPU state (per Newton iteration: α, ‖p‖, μ, energies)."""
    from oracle import mesh as M, solver as SO
    sc = S.make_scene(name)
    ei = S.env_inputs(sc, np.arange(E), n_steps=k_end + 1)
    b = T.Batch(sc, E)
    b.set_state(ei.x0, ei.y0)
    yk = torch.tensor(ei.ykin, device="cuda")
    worst = None
    for k in range(k_end + 1):
        x, xd, y, yd = (t.cpu().numpy() for t in b.get_state())
        b.set_targets(yk[k])
        st = b.step(1)
        ss = b.stats()
        nw = np.array([s["newton_iters"] for s in ss])
        order = np.argsort(-nw)[:3]
        print(k, "newton p50 %d max %d" % (np.median(nw), nw.max()), "failed", np.nonzero(st)[0][:5], flush=True)
        for e in order:
            s = ss[e]
            print("   env", e, {kk: s[kk] for kk in ("newton_iters", "pcg_iters", "ls_backtracks", "al_rounds", "alpha_min", "lm_mu", "n_active")}, flush=True)
        if worst is None or nw.max() > worst[0]:
            worst = (nw.max(), k, int(order[0]), (x[order[0]], xd[order[0]], y[order[0]], yd[order[0]]))
    n, k, e, (x, xd, y, yd) = worst
    print("oracle trace: step", k, "env", e, "GPU newton", n, flush=True)
    mod = M.prepare(sc)
    L = M.env_scale(mod, ei.x0[e], ei.y0[e])
    trace = []
    ost, ostats = SO.step(mod, SO.State(x.copy(), xd.copy(), y.copy(), yd.copy()), ei.ykin[k, e], L_env=L, trace=trace)
    print("oracle stats", ostats, flush=True)
    for t in trace:
        print("  ", {kk: (round(v, 6) if isinstance(v, float) and abs(v) > 1e-3 else v) for kk, v in t.items()}, flush=True)


if __name__ == "__main__":
    which = sys.argv[1] if len(sys.argv) > 1 else "capacity"
    if which == "tail":
        tail(*(sys.argv[2:3] or ["C2"]))
    elif which == "trace":
        trace(*(sys.argv[2:3] or ["C3"]), *(int(a) for a in sys.argv[3:4]))
    elif which == "iters":
        iters(*(sys.argv[2:3] or ["C2"]))
    elif which == "grasp":
        grasp(*(sys.argv[2:3] or ["C4:0"]))
    else:
        {"capacity": capacity, "c3": c3_fail, "pcg": pcg, "sched": sched, "sanity": sanity}[which]()
