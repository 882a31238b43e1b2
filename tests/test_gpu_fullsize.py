"""GPU parity at BASELINE.json's full sizes, in the launch configurations bench.py times (lockstep
tac_set_targets + tac_step + tac_get_gel_deformation over a device-resident target table, and
tac_step_schedule): C2 at 1024 envs and C3 (high-res pads) at 4096 envs, including single steps from
shared states deep in the contact-rich phase (the GPU state after k steps is loaded
into the oracle, both advance one step, sampled envs are compared).  Sampled envs are compared with the CPU oracle one by one; every env is
checked against properties that hold at any size (status, inversion- and intersection-free, P:L30,
P:L60).  Bars (BASELINE.json north_star): active sets bit-exact; energies/gradients/HVPs within 1e-9
relative; positions after each converged step within 1e-6·L_env."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2504_12908_b200 import scenes as S
from paper_2504_12908_b200 import taccel as T
from paper_2504_12908_b200.build import build
from oracle import contact as C
from oracle import energy as En
from oracle import mesh as M
from oracle import readout as R
from oracle import solver as SO

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _built():
    build()


@pytest.fixture(autouse=True)
def _free_device_memory():
    yield
    import gc
    gc.collect()
    torch.cuda.empty_cache()


def _schedule(sc, E, K):
    ei = S.env_inputs(sc, np.arange(E), n_steps=K)
    b = T.Batch(sc, E)
    assert (b.set_state(ei.x0, ei.y0) == 0).all()
    dev = torch.device("cuda", 0)
    yk = torch.tensor(ei.ykin, device=dev)
    out = (torch.empty((K, E, b.n_coated, 3), dtype=torch.float64, device=dev),
           torch.empty((K, E, b.n_markers, 3), dtype=torch.float64, device=dev),
           torch.empty((K, E, b.n_markers, 3), dtype=torch.float64, device=dev))
    st = b.step_schedule(yk, out=out)
    return ei, b, st, [t.cpu().numpy() for t in out]


def test_c2_full_batch_sampled_steps_match_oracle():
    """C2 (BASELINE configs[1]): 1024 envs, 2 scheduled steps (peg resting 0.08 mm above the hole
    floor: ABD–static contact from step 0); envs 0, 517, 1023 against the oracle step by step."""
    sc = S.make_scene("C2")
    E, K = 1024, 2
    ei, b, st, out = _schedule(sc, E, K)
    assert (st == 0).all(), np.unique(st, return_counts=True)
    mod = M.prepare(sc)
    x_all, _, y_all, _ = (t.cpu().numpy() for t in b.get_state())
    for e in (0, 517, 1023):
        ost = SO.State(ei.x0[e].copy(), np.zeros_like(ei.x0[e]), ei.y0[e].copy(), np.zeros_like(ei.y0[e]))
        L = M.env_scale(mod, ost.x, ost.y)
        for k in range(K):
            ost, ostats = SO.step(mod, ost, ei.ykin[k, e], L_env=L)
            assert ostats.status == 0
        P = M.all_positions(mod, x_all[e], y_all[e])
        Po = M.all_positions(mod, ost.x, ost.y)
        assert np.abs(P - Po).max() <= 1e-6 * L, (e, np.abs(P - Po).max() / L)
        # per-step readout of the last step (scheduled output buffers) against the oracle readout
        o = R.gel_deformation(mod, ost.x, ost.y)
        oc = np.concatenate([a[0] for a in o])
        assert np.abs(out[0][K - 1, e] - oc).max() <= 1e-6 * L
    # properties that hold at any size: every env inversion- and intersection-free
    for e in range(0, E, 97):
        assert not SO.any_inverted(mod, x_all[e])
        assert C.min_distance(mod, M.all_positions(mod, x_all[e], y_all[e])) > 0


def _perturbed_state(sc, mod, ei, e, seed, amp=2e-5):
    rng = np.random.default_rng(seed)
    xn, yn = ei.x0[e], ei.y0[e]
    v = rng.normal(size=xn.shape) * 1e-3
    yd = np.zeros_like(yn)
    x = xn + rng.normal(size=xn.shape) * amp
    y = yn.copy()
    for bi in range(len(y)):
        if mod.dof_slot[bi] >= 0:
            yd[bi] = rng.normal(size=12) * 1e-3 * np.r_[np.ones(3), np.full(9, 0.01)]
            y[bi] += rng.normal(size=12) * amp * np.r_[np.full(3, 0.25), np.full(9, 0.01)]
    ctx = En.make_context(mod, xn, v, yn, yd, ei.ykin[0, e], sc.config.dt)
    ctx.lam_att = rng.normal(size=ctx.lam_att.shape) * 1e-6
    ctx.lam_kin = rng.normal(size=ctx.lam_kin.shape) * 1e-6
    ctx.rho = sc.config.al_rho0 * 2.0
    return (xn, v, yn, yd), ctx, x, y


def _lockstep(b, ykin_dev, k0, n):
    for k in range(k0, k0 + n):
        b.set_targets(ykin_dev[k])
        st = b.step(1)
        assert (st == 0).all(), (k, np.unique(st, return_counts=True))
        b.get_gel_deformation()


def _guard_band_ok(sc, mod, P):
    _, d2 = C.classify(mod, P, C.candidate_pairs(mod, P))
    dh2 = sc.config.dhat ** 2
    return bool(np.all(np.abs(d2 - dh2) > 1e-9 * dh2))


def _shared_state_step(sc, mod, ei, b, ykin_dev, k, envs, require_contact=True):
    """At the GPU state after k steps: for each sampled env, the active set (bit-exact), energy terms,
    gradient and exact-Hessian HVP (1e-9) at that state against the oracle; then both advance step k
    from that state and the positions must agree within 1e-6·L_env."""
    x_all, xd_all, y_all, yd_all = (t.cpu().numpy() for t in b.get_state())
    b.set_targets(ykin_dev[k])
    checked = []
    rng = np.random.default_rng(k)
    for e in envs:
        x, v, y, yd = x_all[e], xd_all[e], y_all[e], yd_all[e]
        P = M.all_positions(mod, x, y)
        if not _guard_band_ok(sc, mod, P):            # reading R9: |s − d̂²| ≤ 1e-9 d̂² is a tie; skip
            continue
        pairs = C.active_pairs(mod, P)
        if require_contact:
            assert len(pairs) > 0, (k, e)
        assert np.array_equal(b.debug_active_pairs(e, x, y), pairs.keys()), (k, e)
        ctx = En.make_context(mod, x, v, y, yd, ei.ykin[k, e], sc.config.dt)
        vv = rng.normal(size=mod.n_dof)
        et, g, hv = b.debug_eval(e, x, y, ctx.lam_att, ctx.lam_kin, ctx.rho, vv, exact=True)
        terms = En.energy_terms(mod, ctx, x, y, pairs)
        for i, name in enumerate(En.TERMS):
            assert abs(et[i] - terms[name]) <= 1e-9 * max(abs(terms[name]), 1e-300) + 1e-300, (k, e, name, et[i], terms[name])
        go, H = En.assemble(mod, ctx, x, y, pairs, project=False)
        rel = lambda a, c: np.abs(a - c).max() / max(np.abs(a).max(), np.abs(c).max())
        assert rel(g, go) <= 1e-9, (k, e)
        assert rel(hv, H @ vv) <= 1e-9, (k, e)
        checked.append((e, (x, v, y, yd), len(pairs)))
    assert checked, "every sampled env hit the guard band"
    st = b.step(1)
    assert (st == 0).all()
    x1, _, y1, _ = (t.cpu().numpy() for t in b.get_state())
    for e, (x, v, y, yd), npairs in checked:
        L = M.env_scale(mod, ei.x0[e], ei.y0[e])
        ost, ostats = SO.step(mod, SO.State(x.copy(), v.copy(), y.copy(), yd.copy()), ei.ykin[k, e], L_env=L)
        assert ostats.status == 0
        P = M.all_positions(mod, x1[e], y1[e])
        Po = M.all_positions(mod, ost.x, ost.y)
        err = np.abs(P - Po).max() / L
        assert err <= 1e-6, (k, e, err)
        assert not SO.any_inverted(mod, x1[e])
        assert C.min_distance(mod, P) > 0
    return checked


def test_c2_contact_rich_single_steps_from_shared_states():
    """C2 × 1024 in the bench's lockstep configuration: at steps 20 (pads squeezing the peg while
    closing), 60 and 140 (oscillation phase: pad–peg and peg–hole contact), sampled envs 0, 517, 1023
    take one step on the GPU and in the oracle from the same state."""
    sc = S.make_scene("C2")
    E = 1024
    ei = S.env_inputs(sc, np.arange(E), n_steps=141)
    b = T.Batch(sc, E)
    assert (b.set_state(ei.x0, ei.y0) == 0).all()
    ykin = torch.tensor(ei.ykin, device=torch.device("cuda", 0))
    mod = M.prepare(sc)
    k = 0
    n_pairs = []
    for target in (20, 60, 140):
        _lockstep(b, ykin, k, target - k)
        n_pairs += [c[2] for c in _shared_state_step(sc, mod, ei, b, ykin, target, (0, 517, 1023))]
        k = target + 1
    assert max(n_pairs) >= 50                              # the dominant pad–peg squeeze is in the sample
    s = b.stats()
    assert min(d["min_dist"] for d in s) > 0


def test_c3_after_closing_single_step_and_sampled_derivatives():
    """C3 (high-res pads, 1,520 nodes / 5,400 tets each; the 1–8 GPU config) × 4096 envs, lockstep
    through the closing phase to step 42 (pads pressing the peg), every env converging; env 4095 then
    takes step 42 on the GPU and in the oracle from the shared state; sampled envs are inversion- and
    intersection-free.  In the same batch, the energy terms, gradient and HVP of a perturbed state of
    env 4094 match the oracle."""
    sc = S.make_scene("C3")
    E = 4096
    ei = S.env_inputs(sc, np.arange(E), n_steps=43)
    b = T.Batch(sc, E)
    assert (b.set_state(ei.x0, ei.y0) == 0).all()
    ykin = torch.tensor(ei.ykin, device=torch.device("cuda", 0))
    mod = M.prepare(sc)
    _lockstep(b, ykin, 0, 42)
    x_all, _, y_all, _ = (t.cpu().numpy() for t in b.get_state())
    for e in (0, 2047, 4095):
        assert not SO.any_inverted(mod, x_all[e])
        assert C.min_distance(mod, M.all_positions(mod, x_all[e], y_all[e])) > 0
    _shared_state_step(sc, mod, ei, b, ykin, 42, (4095,))
    # perturbed (contact-rich) state of env 4094 in the same 4096-env batch
    e = E - 2
    base, ctx, x, y = _perturbed_state(sc, mod, ei, e, seed=31)
    xn, v, yn, yd = base
    b.set_state(xn[None], yn[None], v[None], yd[None], env0=e)
    b.set_targets(ei.ykin[0, e][None], env0=e)
    P = M.all_positions(mod, x, y)
    assert _guard_band_ok(sc, mod, P)
    pairs = C.active_pairs(mod, P)
    assert len(pairs) > 0
    assert np.array_equal(b.debug_active_pairs(e, x, y), pairs.keys())
    rng = np.random.default_rng(7)
    vv = rng.normal(size=mod.n_dof)
    et, g, hv = b.debug_eval(e, x, y, ctx.lam_att, ctx.lam_kin, ctx.rho, vv, exact=True)
    terms = En.energy_terms(mod, ctx, x, y, pairs)
    for i, k in enumerate(En.TERMS):
        assert abs(et[i] - terms[k]) <= 1e-9 * max(abs(terms[k]), 1e-300) + 1e-300, (k, et[i], terms[k])
    go, H = En.assemble(mod, ctx, x, y, pairs, project=False)
    rel = lambda a, c: np.abs(a - c).max() / max(np.abs(a).max(), np.abs(c).max())
    assert rel(g, go) <= 1e-9
    assert rel(hv, H @ vv) <= 1e-9


def test_c3_env_split_bitwise_equal():
    """Sharding equivalence: C3 envs [0, 2048) and [2048, 4096) run as two batches give
    bitwise the same states after 3 lockstep steps as one 4096-env batch (the strong split of the
    2-GPU run)."""
    import gc
    sc = S.make_scene("C3")
    E, K = 4096, 3
    ei = S.env_inputs(sc, np.arange(E), n_steps=K)
    dev = torch.device("cuda", 0)

    def run(lo, hi):
        b = T.Batch(sc, hi - lo)
        assert (b.set_state(ei.x0[lo:hi], ei.y0[lo:hi]) == 0).all()
        _lockstep(b, torch.tensor(ei.ykin[:, lo:hi], device=dev), 0, K)
        out = [t.cpu().numpy() for t in b.get_state()]
        del b
        gc.collect()
        torch.cuda.empty_cache()
        return out

    full = run(0, E)
    halves = [run(0, 2048), run(2048, E)]
    for j in range(4):
        assert np.array_equal(full[j], np.concatenate([halves[0][j], halves[1][j]]))


def test_c2_with_friction_single_steps_from_shared_states():
    """C2 with lagged friction (μ = 0.5, reading R20; NEXT 1) × 256 envs, lockstep to step 25 (pads
    squeezing the peg: friction pairs on every pad–peg contact); envs 0 and 255 take step 25 on the GPU and
    in the oracle from the shared state (friction frozen at that state on both sides)."""
    import dataclasses
    sc = S.make_scene("C2")
    sc.config = dataclasses.replace(sc.config, mu_friction=0.5, eps_v=1e-3)
    E = 256
    ei = S.env_inputs(sc, np.arange(E), n_steps=26)
    b = T.Batch(sc, E)
    assert (b.set_state(ei.x0, ei.y0) == 0).all()
    ykin = torch.tensor(ei.ykin, device=torch.device("cuda", 0))
    mod = M.prepare(sc)
    _lockstep(b, ykin, 0, 25)
    assert max(s["n_friction"] for s in b.stats()) > 0
    _shared_state_step(sc, mod, ei, b, ykin, 25, (0, 255))


def test_c2_relaxed_pcg_tolerance_single_steps():
    """Relaxed PCG tolerance (reading R24, "carefully relaxing convergence tolerances"; NEXT 4): C2 ×
    64 envs with the Eisenstat–Walker forcing in [η, 0.1]; the converged steps still agree with the oracle's
    exact Newton solves from shared states at steps 12 and 30 (positions within 1e-6·L_env, active sets
    bit-exact, derivatives 1e-9), and the forcing is live (a different PCG iteration count from the fixed η)."""
    import dataclasses
    E = 64
    pcg_tot = []
    for em in (0.0, 0.1):
        sc = S.make_scene("C2")
        sc.config = dataclasses.replace(sc.config, pcg_eta_max=em)
        ei = S.env_inputs(sc, np.arange(E), n_steps=31)
        b = T.Batch(sc, E)
        assert (b.set_state(ei.x0, ei.y0) == 0).all()
        ykin = torch.tensor(ei.ykin, device=torch.device("cuda", 0))
        _lockstep(b, ykin, 0, 12)
        pcg_tot.append(sum(s["pcg_iters_total"] for s in b.stats()))
        if em > 0:
            mod = M.prepare(sc)
            _shared_state_step(sc, mod, ei, b, ykin, 12, (0, 33, 63))
            _lockstep(b, ykin, 13, 17)
            _shared_state_step(sc, mod, ei, b, ykin, 30, (0, 33, 63))
    assert pcg_tot[1] != pcg_tot[0], pcg_tot
