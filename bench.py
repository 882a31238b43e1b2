#!/usr/bin/env python
"""bench.py — throughput of the batched IPC + ABD Newton step (Taccel, arXiv 2504.12908) on B200.

Metric (BASELINE.json): peg-insertion env-steps/s and ×real-time, dual sensors, at 1/2/4/8 B200.

A "step" is one backward-Euler time step of EVERY env of the workload, advanced in LOCKSTEP the way an
RL loop drives the C ABI: per step tac_set_targets (from a device-resident target table of the scripted
episode), tac_step (host-blocking; all envs finish the step) and tac_get_gel_deformation (coated-vertex
displacements, marker positions and flows of every env, into device buffers).

Workloads:
  C3  (primary line; BASELINE configs[2], the 1/2/4/8-GPU axis): peg insertion with dual HIGH-res pads,
      4096 envs in total, env-sharded over the N GPUs (strong scaling: rank r owns [⌊rE/N⌋, ⌊(r+1)E/N⌋)).
  C2  (alongside; BASELINE configs[1]): dual low-res pads, 1024 envs per GPU (weak scaling).
Both run the scripted 200-step episode; the timed steps are W..W+K-1 (closing phase, pads pressing
the peg; contact-rich from step ~3).  Inputs are larger than L2 (per-step working set ≫ 126 MB).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl taccel|reference] [--config C3|C2]
                  [--envs-total E | --envs-per-gpu E] [--no-alongside]

With --gpus N > 1 and no WORLD_SIZE in the environment, bench.py launches itself under
torch.distributed.run with N ranks (one per GPU, NCCL); the world size must equal --gpus.
value = whole-job env-steps/s = Σ_ranks envs · K / (max over ranks of the CUDA-event time).
"""
import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "peg-insertion env-steps/s and ×real-time, dual sensors, at 1/2/4/8 B200"
WORKLOADS = {
    "C4": "C4: parallel-gripper grasp, dual 40x40x4 mm pads (14x14x3 lattice, 588 nodes/1690 tets each), 8 procedural "
          "star-shaped objects (perturbed level-3 icospheres, 642 v/1280 t; 256 envs per shape, one batch each), "
          "2 kinematic fingers + static table, frictional contact mu=0.5 (lagged D_k), dt=0.02 s",
    "C5": "C5: Allegro-like hand, four 24x24x3 mm fingertip pads (9x9x4 lattice, 324 nodes/960 tets each), palm + 16 "
          "kinematic links driven by on-device forward kinematics of a 16-joint script, dynamic engraved tile "
          "(16x30x22 mm, 8676 triangles), static table, frictional contact mu=0.5 (lagged D_k), dt=0.02 s",
    "C2": "C2: peg insertion, dual low-res sensors (2 pads x 8x6x3 lattice, 144 nodes/350 tets each), "
          "1 dynamic peg + 2 kinematic fingers + static blind hole, frictional contact mu=0.5 (lagged D_k), dt=0.02 s",
    "C3": "C3: peg insertion, dual high-res sensors (2 pads x 19x16x5 lattice, 1520 nodes/5400 tets each), "
          "1 dynamic peg + 2 kinematic fingers + static blind hole, frictional contact mu=0.5 (lagged D_k), dt=0.02 s",
}
DEFAULTS = {  # config: (scaling, envs, default steps)
    "C3": ("strong", 4096, 10),
    "C2": ("weak", 1024, 20),
    "C4": ("weak", 2048, 10),
    "C5": ("strong", 1024, 10),
}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=None)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="taccel", choices=["taccel", "reference"])
    ap.add_argument("--config", default="C3", choices=sorted(WORKLOADS))
    ap.add_argument("--envs-total", type=int, default=None, help="strong scaling: total envs split over the ranks")
    ap.add_argument("--envs-per-gpu", type=int, default=None, help="weak scaling: envs per rank")
    ap.add_argument("--no-alongside", action="store_true", help="skip the C2 line reported alongside C3")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-schedule", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--phases", action="store_true", help="add the per-phase breakdown to the JSON line")
    ap.add_argument("--set", action="append", default=[], metavar="KEY=VALUE",
                    help="override a solver constant of the scene config (experiments; recorded in the line)")
    a = ap.parse_args()
    if a.steps is None:
        a.steps = DEFAULTS[a.config][2]
    return a


def load_peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        return None


def relaunch_distributed(a):
    """--gpus N > 1 without a torchrun environment: run this script under torch.distributed.run."""
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={a.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


# ----------------------------------------------------------------------------------------------
# clocks sampler (nvidia-smi during the timed region)
# ----------------------------------------------------------------------------------------------
class Clocks:
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index):
        self.idx = gpu_index
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        self.p = None

    def start(self):
        try:
            self.p = subprocess.Popen(["nvidia-smi", f"--id={self.idx}", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                                       "-lms", "100"], stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:
            self.p = None

    def stop(self):
        if self.p is None:
            return None
        time.sleep(0.25)
        self.p.terminate()
        try:
            self.p.wait(timeout=5)
        except Exception:
            self.p.kill()
        self.f.flush()
        rows = [r.split(",") for r in open(self.f.name).read().strip().splitlines() if r.strip()]
        os.unlink(self.f.name)
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in rows:
            try:
                sm.append(float(r[1]))
                mx = float(r[2])
                for nm, v in zip(names, r[5:9]):
                    if v.strip() == "Active":
                        reasons.add(nm)
            except Exception:
                pass
        if not sm:
            return None
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": len(sm)}


# ----------------------------------------------------------------------------------------------
# CPU oracle baseline: the oracle as it stands (numpy/torch-autograd fp64, exact direct Newton
# solve), one env per process, one thread per process, on every host core (bounded sample)
# ----------------------------------------------------------------------------------------------
def _oracle_job(args):
    """One oracle process: env `env_id` of `cfg_name` from its initial state, `n_steps` full steps, or
    (n_newton > 0) only the first n_newton Newton iterations of step 0 (the step is cut there).
    Returns (seconds, env-steps done, Newton iterations done)."""
    cfg_name, env_id, n_steps, n_newton = args
    import dataclasses
    import torch
    torch.set_num_threads(1)
    from paper_2504_12908_b200 import scenes as S
    from oracle import mesh as M
    from oracle import solver as SO
    sc = S.make_scene(cfg_name)
    if n_newton > 0:
        sc.config = dataclasses.replace(sc.config, max_newton=n_newton)
    mod = M.prepare(sc)
    ei = S.env_inputs(sc, [env_id], n_steps=max(n_steps, 1))
    st = SO.State(ei.x0[0].copy(), np.zeros_like(ei.x0[0]), ei.y0[0].copy(), np.zeros_like(ei.y0[0]))
    L = M.env_scale(mod, st.x, st.y)
    t0 = time.perf_counter()
    done, newton = 0, 0
    for k in range(max(n_steps, 1)):
        yk = ei.ykin[k, 0] if ei.ykin.shape[2] else np.zeros((0, 12))
        st, stats = SO.step(mod, st, yk, L_env=L)
        newton += stats.newton_iters
        done += 1
    return time.perf_counter() - t0, done, newton


def oracle_pool(jobs):
    """Run oracle jobs in one single-thread process each (spawned, all host cores); returns the
    per-job results and the wall time."""
    import multiprocessing as mp
    for k in ("OMP_NUM_THREADS", "OPENBLAS_NUM_THREADS", "MKL_NUM_THREADS", "NUMEXPR_NUM_THREADS"):
        os.environ[k] = "1"                           # one thread per oracle process (spawned children inherit)
    ctx = mp.get_context("spawn")
    with ctx.Pool(len(jobs)) as pool:
        t0 = time.perf_counter()
        res = pool.map(_oracle_job, jobs)
        wall = time.perf_counter() - t0
    return res, wall


def cpu_cores():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


ORACLE_SAMPLE = {  # cfg: (full steps per process, Newton iterations per process (0 = full steps))
    "C2": (3, 0),
    "C3": (1, 2),
}


def oracle_rate(cfg_name, cores, env0, newton_per_step):
    """The bounded oracle sample of one bench "step": `cores` processes × ORACLE_SAMPLE[cfg].  C2: full
    env-steps (env-steps/s = Σ steps / max process time).  C3: an oracle env-step takes minutes
    (profiles/r2_oracle_newton_C3.json), so each process runs the first 2 Newton iterations of its env's
    step and the rate is EXTRAPOLATED: env-steps/s = cores / (seconds per Newton iteration ×
    Newton iterations per env-step)."""
    n_steps, n_newton = ORACLE_SAMPLE[cfg_name]
    res, wall = oracle_pool([(cfg_name, env0 + i, n_steps, n_newton) for i in range(cores)])
    tmax = max(r[0] for r in res)
    if n_newton == 0:
        return sum(r[1] for r in res) / tmax, wall, tmax, None
    s_per_it = statistics.mean(r[0] / max(r[2], 1) for r in res)
    return cores / (s_per_it * newton_per_step), wall, tmax, s_per_it


def oracle_newton_per_step(cfg_name):
    """Oracle Newton iterations per env-step from the committed offline oracle run (env 0, first steps)."""
    try:
        j = json.load(open(os.path.join(ROOT, "profiles", f"r2_oracle_newton_{cfg_name}.json")))
        return statistics.mean(r["newton_iters"] for r in j["steps"]), "profiles/r2_oracle_newton_%s.json" % cfg_name
    except Exception:
        return 12.0, "oracle C3 env 0 step 0 (12 Newton iterations, measured offline)"


def cpu_baseline(cfg_name, gpu_newton_mean):
    """nproc single-thread oracle processes (one env each) on the host cores, plus the C1 run
    (BASELINE configs[0]) in seconds on one core."""
    cores = cpu_cores()
    nps, src = (gpu_newton_mean, "the GPU run's mean Newton iterations per env-step over the same timed steps") \
        if gpu_newton_mean else oracle_newton_per_step(cfg_name)
    v, wall, tmax, s_it = oracle_rate(cfg_name, cores, 0, nps)
    n_steps, n_newton = ORACLE_SAMPLE[cfg_name]
    if n_newton:
        sample = (f"{cfg_name}: {cores} processes x 1 thread, envs 0-{cores - 1}, the first {n_newton} Newton iterations of "
                  f"episode step 0 each ({s_it:.2f} s per Newton iteration); EXTRAPOLATED to env-steps with "
                  f"{nps:.2f} Newton iterations per env-step ({src}); max process time {tmax:.1f} s")
    else:
        sample = (f"{cfg_name}: {cores} processes x 1 thread, envs 0-{cores - 1}, episode steps 0-{n_steps - 1} each; "
                  f"max process time {tmax:.1f} s")
    c1_s = _oracle_job(("C1", 0, 10, 0))[0]
    return {"value": v, "unit": "env-steps/s", "cores": cores, "kind": "oracle",
            "sample": sample + "; the CPU oracle as it stands (numpy/torch-autograd fp64, exact sparse direct Newton solve)",
            "x_realtime": v * 0.02, "c1_oracle_seconds": c1_s,
            "c1_note": "BASELINE configs[0]: C1 (1 env, 490-tet pad pressed 1 mm by a kinematic cube), all 10 steps "
                       "at dt=0.01 on 1 core"}


def run_reference(a):
    """Reference arm of this tier = the CPU oracle as it stands, on the host cores (rank 0 only):
    each timed step is one bounded oracle sample of the workload (oracle_rate)."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    cores = cpu_cores()
    nps, src = oracle_newton_per_step(a.config)
    W = min(a.warmup, 1)
    for w in range(W):
        oracle_rate(a.config, cores, 100000 + w * cores, nps)
    secs = 0.0
    n_equiv = 0.0
    for k in range(a.steps):
        v, wall, tmax, s_it = oracle_rate(a.config, cores, k * cores, nps)
        secs += cores / v                      # seconds of this sample's env-step equivalents
        n_equiv += cores
    v = n_equiv / secs
    n_steps, n_newton = ORACLE_SAMPLE[a.config]
    sample = (f"{a.config}: per timed step {cores} processes x 1 thread, distinct env ids, " +
              (f"the first {n_newton} Newton iterations of episode step 0 each, extrapolated with {nps:.2f} oracle Newton "
               f"iterations per env-step ({src})" if n_newton else f"episode steps 0-{n_steps - 1} each"))
    line = {"metric": METRIC, "value": v, "unit": "env-steps/s", "impl": "reference", "n_gpus": 0,
            "steps": a.steps, "warmup": W, "ms_per_step": 1e3 * secs / a.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": WORKLOADS[a.config] + " — reference arm: the CPU oracle, one env per host core",
                       "envs_per_step": cores, "dt": 0.02},
            "x_realtime": v * 0.02,
            "cpu_baseline": {"value": v, "unit": "env-steps/s", "cores": cores, "kind": "oracle", "sample": sample},
            "e2e": {"value": v, "unit": "env-steps/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------------------------------------
# the CUDA path
# ----------------------------------------------------------------------------------------------
def _pcts(v):
    if not len(v):
        return None
    v = np.asarray(v, float)
    return {"mean": float(v.mean()), "p50": float(np.percentile(v, 50)), "p99": float(np.percentile(v, 99)),
            "max": float(v.max())}


class Part:
    """One homogeneous batch of the workload (C4 has one per object shape) on its own CUDA stream."""

    def __init__(self, sc, ids, W, K, dev, chain=False, overrides=None):
        import dataclasses
        import torch
        from paper_2504_12908_b200 import scenes as S
        from paper_2504_12908_b200 import taccel as T
        if overrides:
            sc.config = dataclasses.replace(sc.config, **overrides)
        self.sc, self.ids, self.E = sc, ids, len(ids)
        self.stream = torch.cuda.Stream(dev)
        self.ei = S.env_inputs(sc, ids, n_steps=W + K)
        self.batch = T.Batch(sc, self.E, device=dev.index, stream=self.stream)
        st = self.batch.set_state(self.ei.x0, self.ei.y0)
        assert (st == 0).all(), f"bad initial states: {np.unique(st)}"
        self.ykin_dev = torch.tensor(self.ei.ykin, device=dev)
        self.chain = chain
        if chain:                                          # C5: targets compiled on the device from joint targets
            self.batch.set_chain(S.hand_chain())
            q = np.stack([S.hand_script(int(g), W + K).reshape(W + K, -1) for g in ids], 1)
            self.q_dev = torch.tensor(q, device=dev)
            self.base_dev = torch.tensor(np.repeat(S.hand_palm_pose()[None], self.E, 0), device=dev)
        NC, NM = self.batch.n_coated, self.batch.n_markers
        self.out_dev = [tuple(torch.empty((self.E, n, 3), dtype=torch.float64, device=dev) for n in (NC, NM, NM))
                        for _ in range(K)]

    def step(self, k, targets, outs, stats=None):
        """One lockstep step: targets (tac_set_targets, or joint targets → tac_set_joint_targets), tac_step,
        gel readout."""
        import torch
        with torch.cuda.stream(self.stream):
            if self.chain:
                self.batch.set_joint_targets(targets[k], base=self.base_dev)
            else:
                self.batch.set_targets(targets[k])
            f = int((self.batch.step(1) != 0).sum())
            self.batch.get_gel_deformation(out=outs)
            if stats is not None:
                stats.append(self.batch.stats())
        return f


def run_parts(parts, fn):
    """Run fn(part) for every part concurrently (one host thread per batch: tac_step is host-blocking and
    releases the GIL inside the C call); returns the results in part order."""
    if len(parts) == 1:
        return [fn(parts[0])]
    from concurrent.futures import ThreadPoolExecutor
    with ThreadPoolExecutor(len(parts)) as ex:
        return list(ex.map(fn, parts))


def run_config(cfg_name, a, rank, world, dev, envs_total=None, envs_per_gpu=None, steps=None, primary=True):
    import torch
    import torch.distributed as dist
    from paper_2504_12908_b200 import scenes as S
    from paper_2504_12908_b200.shard import env_range, reduce_run_stats, split_range

    scaling = DEFAULTS[cfg_name][0]
    if envs_per_gpu is not None:
        scaling = "weak"
    elif envs_total is not None:
        scaling = "strong"
    if scaling == "strong":
        total = envs_total or DEFAULTS[cfg_name][1]
        ids = np.asarray(list(split_range(rank, world, total)))
    else:
        per = envs_per_gpu or DEFAULTS[cfg_name][1]
        ids = np.asarray(list(env_range(rank, world, per)))
    W, K = a.warmup, (steps or a.steps)
    ov = {}
    for kv in a.set:
        k, v = kv.split("=", 1)
        ov[k] = type(getattr(S.Config(), k))(v)
    if cfg_name == "C4":                   # 8 object shapes, one homogeneous batch each (env id → shape)
        per_shape = max(1, (len(ids) + 7) // 8) if scaling == "strong" else max(1, (envs_per_gpu or DEFAULTS["C4"][1]) // 8)
        groups = {}
        for g in ids:
            groups.setdefault(int((g % (8 * per_shape)) // per_shape), []).append(int(g))
        parts = [Part(S.make_scene(f"C4:{sh}"), np.asarray(gl), W, K, dev, overrides=ov) for sh, gl in sorted(groups.items())]
    else:
        parts = [Part(S.make_scene(cfg_name), ids, W, K, dev, chain=(cfg_name == "C5"), overrides=ov)]
    E = sum(p.E for p in parts)
    sc = parts[0].sc
    main = torch.cuda.current_stream(dev)
    fails = 0

    def lockstep(part, k0, n, targets, outs, stats_out=None):
        f = 0
        for k in range(n):
            f += part.step(k0 + k, targets, outs[k], stats_out)
        return f

    tables = lambda p: p.q_dev if p.chain else p.ykin_dev
    # warm-up (untimed): W lockstep steps
    fails += sum(run_parts(parts, lambda p: lockstep(p, 0, W, tables(p), [p.out_dev[0]] * W)))
    saved = [p.batch.get_state() for p in parts]
    stats0 = [p.batch.stats() for p in parts]
    torch.cuda.synchronize(dev)
    if world > 1:
        dist.barrier()

    def timed(fn):
        """CUDA-event time on the main stream with every part's stream joined in (device-side)."""
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(main)
        for p in parts:
            p.stream.wait_event(e0)
        res = run_parts(parts, fn)
        for p in parts:
            ej = torch.cuda.Event()
            ej.record(p.stream)
            main.wait_event(ej)
        e1.record(main)
        torch.cuda.synchronize(dev)
        return e0.elapsed_time(e1), res

    # ---- timed: K lockstep steps, device-resident inputs/outputs ----
    clocks = Clocks(dev.index)
    clocks.start()
    for p in parts:
        p.batch.profile(True)
        p.batch.profile_read(reset=True)
    per_step = {id(p): [] for p in parts}
    torch.cuda.synchronize(dev)
    if world > 1:
        dist.barrier()
    ms, fl = timed(lambda p: lockstep(p, W, K, tables(p), p.out_dev, per_step[id(p)]))
    fails += sum(fl)
    profs = [p.batch.profile_read(reset=True) for p in parts]
    for p in parts:
        p.batch.profile(False)
    clk = clocks.stop()
    stats1 = [p.batch.stats() for p in parts]
    pcg_local = sum(s1["pcg_alg_bytes_total"] - s0["pcg_alg_bytes_total"] for S0, S1 in zip(stats0, stats1) for s0, s1 in zip(S0, S1))
    pcg_iters_local = sum(s1["pcg_iters_total"] - s0["pcg_iters_total"] for S0, S1 in zip(stats0, stats1) for s0, s1 in zip(S0, S1))
    allst = [s for p in parts for ss in per_step[id(p)] for s in ss]
    newton = [s["newton_iters"] for s in allst]
    pcg_per_step = [s["pcg_iters"] for s in allst]
    n_active = [s["n_active"] for s in allst]
    n_res = [s["n_residual"] for s in allst]
    n_fr = [s["n_friction"] for s in allst]
    min_d = min((s["min_dist"] for s in allst), default=float("inf"))

    # ---- scheduled mode (context): the same K steps, envs advance independently ----
    ms_sched = 0.0
    if not a.no_schedule and not parts[0].chain:
        for p, sv in zip(parts, saved):
            x, xd, y, yd = sv
            p.batch.set_state(x, y, xd, yd)
        outs = {id(p): tuple(torch.empty((K, p.E) + t.shape[1:], dtype=torch.float64, device=dev) for t in p.out_dev[0])
                for p in parts}
        torch.cuda.synchronize(dev)
        if world > 1:
            dist.barrier()

        def sched(p):
            with torch.cuda.stream(p.stream):
                p.batch.step_schedule(p.ykin_dev[W:W + K], out=outs[id(p)])
        ms_sched, _ = timed(sched)

    # ---- e2e: the same K lockstep steps through the C ABI with pinned HOST buffers (targets or joint
    #      targets in, per-step gel readout out, both copied inside the timed region) ----
    ms_e2e, h2d, d2h = 0.0, 0, 0
    if not a.no_e2e:
        for p, sv in zip(parts, saved):
            x, xd, y, yd = sv
            p.batch.set_state(x, y, xd, yd)
        host = {}
        for p in parts:
            tab = (p.q_dev if p.chain else p.ykin_dev)[W:W + K].cpu().pin_memory()
            outs_h = [tuple(torch.empty(t.shape, dtype=torch.float64).pin_memory() for t in p.out_dev[0]) for _ in range(K)]
            host[id(p)] = (tab, outs_h)
            h2d += tab[0].numel() * 8
            d2h += sum(t.numel() * 8 for t in outs_h[0])
        torch.cuda.synchronize(dev)
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        ms_dev, _ = timed(lambda p: lockstep(p, 0, K, host[id(p)][0], host[id(p)][1]))
        wall = time.perf_counter() - t0
        ms_e2e = max(ms_dev, 1e3 * wall)

    tot, cnt, mins = reduce_run_stats([ms, ms_e2e, ms_sched], [float(fails), float(pcg_iters_local), float(E)], world,
                                      device=dev, mins=[min_d])
    ms, ms_e2e, ms_sched = (float(v) for v in tot)
    fails, pcg_iters_all, n_env_total = (float(v) for v in cnt)
    n_env_total = int(n_env_total)
    dt = sc.config.dt
    value = n_env_total * K / (ms / 1e3)
    prof = {}
    for pr in profs:
        for k, v in pr.items():
            m0, n0 = prof.get(k, (0.0, 0))
            prof[k] = (m0 + v[0], n0 + v[1])
    res = {"cfg": cfg_name, "overrides": ov, "E_local": E, "n_env_total": n_env_total, "scaling": scaling, "K": K, "W": W, "ms": ms,
           "value": value, "dt": dt, "clocks": clk, "fails": fails, "min_dist": float(mins[0]), "n_batches": len(parts),
           "workspace_gb": sum(p.batch.workspace.numel() for p in parts) / 1e9, "pcg_kernel": parts[0].batch.pcg_kernel,
           "prof": prof}
    res["e2e"] = None if a.no_e2e else {"value": n_env_total * K / (ms_e2e / 1e3), "unit": "env-steps/s",
                                        "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                                        "path": ("tac_set_joint_targets" if parts[0].chain else "tac_set_targets") +
                                                " (pinned host) + tac_step + tac_get_gel_deformation (pinned host) per step"}
    res["schedule"] = None if (a.no_schedule or parts[0].chain) else {
        "value": n_env_total * K / (ms_sched / 1e3), "ms_per_step": ms_sched / K,
        "mode": "tac_step_schedule: envs advance independently through the same K steps"}
    res["solver"] = {"newton_iters_per_env_step": _pcts(newton), "pcg_iters_per_env_step": _pcts(pcg_per_step),
                     "pcg_iters_per_newton_iter": pcg_iters_all / max(sum(newton) * world, 1) if newton else None,
                     "active_pairs_per_env": _pcts(n_active), "residual_pairs_per_env": _pcts(n_res),
                     "friction_pairs_per_env": _pcts(n_fr), "mu_friction": sc.config.mu_friction,
                     "failed_env_steps": fails, "min_dist_m": float(mins[0]),
                     "sample": "rank-0 per-env stats of every timed step" if world > 1 else "every env, every timed step"}
    phases = {k: {"ms": v[0], "launches": v[1]} for k, v in prof.items() if v[1] > 0}
    res["phases"] = phases
    res["launches"] = int(sum(v["launches"] for v in phases.values()))
    res["roofline"] = roofline(cfg_name, res["pcg_kernel"], phases, pcg_local, ms * len(parts), K)
    return res


def roofline(cfg_name, kernel, phases, pcg_bytes, ms_step_total, K):
    if "pcg" not in phases or phases["pcg"]["ms"] <= 0:
        return None
    peaks = load_peaks()
    if peaks:
        peak, src = peaks["hbm_gbs"], "MEASURED_PEAKS.json hbm_gbs (1 GiB copy, read+write bytes, burst)"
    else:
        peak, src = 6650.0, "fallback 6.65 TB/s (B200_PROFILING.md)"
    pcg_ms = phases["pcg"]["ms"]
    launches = max(phases["pcg"]["launches"], 1)
    ach = pcg_bytes / (pcg_ms / 1e3) / 1e9
    traffic, tsrc, t_alg, t_ratio = None, None, None, None
    tfile = os.path.join(ROOT, "profiles", "r2_pcg_traffic.json")
    if os.path.exists(tfile):
        tj = json.load(open(tfile)).get(cfg_name)
        if tj and tj.get("kernel") == kernel.split(" ")[0]:
            traffic, t_alg, t_ratio = tj["dram_bytes_per_launch"], tj["alg_bytes_per_launch"], tj["traffic_over_alg"]
            tsrc = (f"profiles/r2_pcg_traffic.json: ncu dram__bytes_read.sum+write.sum per {tj['kernel']} launch, "
                    f"{tj['what']}; traffic_alg_bytes_per_launch = the device-counted algorithmic bytes of the same "
                    f"launches (the launches of one step differ in size, so compare the ratio)")
    resident = kernel.startswith("k_pcg_r")
    return {"kernel": kernel, "bound": "hbm", "achieved": ach, "peak": peak, "unit": "GB/s", "frac": ach / peak,
            "traffic": traffic, "traffic_alg_bytes_per_launch": t_alg, "traffic_over_alg": t_ratio,
            "traffic_source": tsrc, "peak_source": src,
            "share_of_step": pcg_ms / ms_step_total, "alg_bytes_per_launch": pcg_bytes / launches,
            "alg_model": "per PCG iteration per env: 72(V+E_s)+4E_s+640*P_res+296*N_cpl+1248*ND+48V+96n "
                         "(SURVEY sec 8(d) B_pcg on the condensed operator; DESIGN.md sec 5)",
            "reading": ("effective algorithmic bandwidth: the operator is staged in shared memory once per launch "
                        "and reused by every PCG iteration, so frac > 1 means on-chip reuse beats streaming it from HBM "
                        "each iteration; measured DRAM traffic is the `traffic` field") if resident else
                       ("streamed operator: achieved = algorithmic bytes / kernel time, an HBM-bandwidth fraction "
                        "when the operator is re-read from L2/HBM every iteration")}


def main():
    a = parse()
    if a.impl == "reference":
        run_reference(a)
        return
    if a.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(relaunch_distributed(a))
    import torch
    import torch.distributed as dist
    from paper_2504_12908_b200.build import build

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    assert world == a.gpus, f"world size {world} != --gpus {a.gpus}"
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    if rank == 0:
        build()
    if world > 1:
        dist.barrier()

    main_res = run_config(a.config, a, rank, world, dev, envs_total=a.envs_total, envs_per_gpu=a.envs_per_gpu)
    side = None
    if not a.no_alongside and a.config != "C2":
        side = run_config("C2", a, rank, world, dev, steps=DEFAULTS["C2"][2], primary=False)
    cpu = None
    if rank == 0 and world == 1 and not a.no_cpu_baseline:
        nm = main_res["solver"]["newton_iters_per_env_step"]
        cpu = cpu_baseline(a.config, nm["mean"] if nm else None)
    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return
    r = main_res
    E_note = (f"{r['n_env_total']} envs in total split over {world} GPU(s)" if r["scaling"] == "strong"
              else f"{r['E_local']} envs per GPU")
    line = {
        "metric": METRIC, "value": r["value"], "unit": "env-steps/s", "n_gpus": world, "steps": r["K"], "warmup": r["W"],
        "ms_per_step": r["ms"] / r["K"], "higher_is_better": True, "scaling": r["scaling"], "vs_baseline": None,
        "dtype": "f64", "data": "synthetic",
        "config": {"workload": WORKLOADS[r["cfg"]], "envs_total": r["n_env_total"], "envs_per_gpu": r["E_local"],
                   "solver_overrides": r["overrides"] or None,
                   "envs": E_note, "dt": r["dt"],
                   "stepping": "lockstep: per step tac_set_targets (device target table) + tac_step + tac_get_gel_deformation "
                               "(device buffers) for every env",
                   "episode_steps_timed": f"{r['W']}-{r['W'] + r['K'] - 1}", "parallelism": f"env-sharded x{world}",
                   "l2": "inputs larger than L2: per-step working set ~%.1f GB/GPU > 126 MB L2" % r["workspace_gb"],
                   "timing_note": "per-kernel CUDA events are recorded inside the device-timed region (roofline, "
                                  "gpu_launches) and per-env stats are read after every timed step; the e2e replay runs "
                                  "without events"},
        "x_realtime": r["value"] * r["dt"],
        "paper_context": "Taccel: 915 env-steps/s = 18.30x real-time (low-res peg, >4096 envs) and 64 envs at 0.25x "
                         "(high-res peg), 1x H100 FP64 (P:L230, P:L49 Table 1) — context, not this workload",
        "roofline": r["roofline"],
        "gpu_launches": r["launches"],
        "solver": r["solver"],
        "schedule": r["schedule"],
        "clocks": r["clocks"],
    }
    if r["e2e"]:
        line["e2e"] = r["e2e"]
    if side:
        line["alongside"] = {
            "config": {"workload": WORKLOADS["C2"], "envs_per_gpu": side["E_local"], "envs_total": side["n_env_total"],
                       "scaling": side["scaling"], "episode_steps_timed": f"{side['W']}-{side['W'] + side['K'] - 1}"},
            "value": side["value"], "unit": "env-steps/s", "x_realtime": side["value"] * side["dt"],
            "ms_per_step": side["ms"] / side["K"], "steps": side["K"], "e2e": side["e2e"], "schedule": side["schedule"],
            "roofline": side["roofline"], "solver": side["solver"], "gpu_launches": side["launches"], "clocks": side["clocks"]}
        if a.phases:
            line["alongside"]["phases"] = side["phases"]
    if a.phases:
        line["phases"] = r["phases"]
    if cpu:
        line["cpu_baseline"] = cpu
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
