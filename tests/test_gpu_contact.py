"""GPU parity of the contact machinery the trajectory tests do not reach, through the C ABI:

* the LM-shifted exact-Hessian solve (R14c) that tac_step runs: (H + μM) p = −g with the EXACT H,
  against the oracle's block-Jacobi PCG and direct solve of the same system;
* soft–soft contact (scene P2: two gel tets touching edge to edge), the pairs the SpMV keeps
  matrix-free ("residual" pairs) — energies/gradients/HVPs, the solve and a 4-step trajectory;
* failure isolation: detected CAPACITY / NEWTON_STALL / AL_INFEASIBLE and injected faults
  roll the failed env back bitwise and leave the other envs bitwise unchanged;
* the 512-thread register budget of the env-resident PCG (k_pcg_r512).
Bars (north_star): active sets bit-exact; energies, gradients, HVPs within 1e-9 relative; positions
within 1e-6·L_env."""
import dataclasses
import os
import subprocess
import sys

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
from oracle import solver as SO

pytestmark = pytest.mark.gpu
REL = 1e-9


def rel_inf(a, b):
    return np.abs(np.asarray(a) - np.asarray(b)).max() / max(np.abs(a).max(), np.abs(b).max(), 1e-300)


@pytest.fixture(scope="module", autouse=True)
def _built():
    build()


def _perturbed(name, seed, amp=2e-5, press=None):
    sc = S.make_scene(name)
    mod = M.prepare(sc)
    ei = S.env_inputs(sc, [0], n_steps=1)
    rng = np.random.default_rng(seed)
    xn, yn = ei.x0[0], ei.y0[0]
    v = rng.normal(size=xn.shape) * 1e-3
    yd = np.zeros_like(yn)
    x = xn + rng.normal(size=xn.shape) * amp
    y = yn.copy()
    for b in range(len(y)):
        if mod.dof_slot[b] >= 0:
            yd[b] = rng.normal(size=12) * 1e-3 * np.r_[np.ones(3), np.full(9, 0.01)]
            y[b] += rng.normal(size=12) * amp * np.r_[np.full(3, 0.25), np.full(9, 0.01)]
    if press is not None:
        press(y)
    ctx = En.make_context(mod, xn, v, yn, yd, ei.ykin[0, 0] if ei.ykin.shape[2] else np.zeros((0, 12)), sc.config.dt)
    b = T.Batch(sc, 1)
    b.set_state(xn[None], yn[None], v[None], yd[None])
    if ei.ykin.shape[2]:
        b.set_targets(ei.ykin[0])
    return sc, mod, ctx, b, x, y


def _c1_press(y):
    y[1, 2] -= 0.2e-3 - 0.04e-3


@pytest.mark.parametrize("name,seed,press", [("C1", 11, _c1_press), ("C2", 14, None), ("P2", 3, None)])
def test_lm_exact_hessian_solve_matches_oracle(name, seed, press):
    """tac_debug_pcg(exact=1, μ): the same PCG launch tac_step runs under hessian_mode 2 — exact H,
    shift μM, and the in-kernel μ ← max(μ₀, 10μ) retry on negative curvature — against the oracle."""
    sc, mod, ctx, b, x, y = _perturbed(name, seed, press=press)
    pairs = C.active_pairs(mod, M.all_positions(mod, x, y))
    g, H = En.assemble(mod, ctx, x, y, pairs, project=False)
    Mm = SO.mass_matrix(mod)
    cfg = sc.config
    for mu in (0.0, 10.0, 1000.0):
        p_gpu, it_gpu, mu_gpu = b.debug_pcg(0, x, y, exact=True, mu=mu, with_mu=True)
        # the oracle's R14c rule in PCG mode (oracle/solver.py step, hessian_mode 2): solve, and on
        # negative curvature / non-descent raise μ ← max(μ₀, 10μ)
        mu_o, stats = mu, SO.StepStats()
        while True:
            p_ref = SO._solve_spd(mod, H + mu_o * Mm if mu_o > 0 else H, g, "pcg", cfg, stats)
            if p_ref is not None or mu_o > 1e12:
                break
            mu_o = max(cfg.lm_mu0, 10.0 * mu_o)
        # R14c rejects a system when CG meets negative curvature (or a non-descent direction).  On an
        # indefinite exact Hessian whether CG meets it depends on rounding, so the GPU may escalate past
        # the oracle; every μ it rejected below its accepted μ must then be a genuinely indefinite system
        # (Cholesky fails), and the oracle's PCG must accept the GPU's μ too (or fail identically).
        seq = [mu]
        while seq[-1] < mu_gpu:
            seq.append(max(cfg.lm_mu0, 10.0 * seq[-1]))
        assert seq[-1] == mu_gpu, (mu, mu_gpu)
        for m_rej in seq[:-1]:
            if m_rej >= mu_o:
                try:
                    np.linalg.cholesky((H + m_rej * Mm).toarray())
                    indefinite = False
                except np.linalg.LinAlgError:
                    indefinite = True
                assert indefinite, ("GPU rejected an SPD system", mu, m_rej)
        if mu_gpu < mu_o:                                  # GPU accepted where the oracle's CG rejected
            pass
        # the defining property of the PCG output on the accepted system A = H + μM: the block-Jacobi
        # residual norm reached the stopping test rᵀM⁻¹r ≤ η²·gᵀM⁻¹g (reading R15).  The exact Hessian is
        # near-singular along some contact directions, so two rounding orders may stop a few iterations
        # apart; the iterates themselves are compared through this test.
        A = (H + mu_gpu * Mm).tocsr()
        r_gpu = -g - A @ p_gpu
        assert _bj_norm2(mod, A, r_gpu) <= cfg.pcg_eta ** 2 * _bj_norm2(mod, A, g) * (1 + 1e-6)
        if mu_gpu == mu_o:
            assert abs(it_gpu - stats.pcg_iters) <= max(6, stats.pcg_iters // 5), (mu, it_gpu, stats.pcg_iters)
        assert g @ p_gpu < 0
        try:
            Lc = np.linalg.cholesky(A.toarray())
        except np.linalg.LinAlgError:
            continue
        import scipy.linalg as sla
        p_dir = sla.cho_solve((Lc, True), -g)
        model = lambda q: g @ q + 0.5 * q @ (A @ q)
        assert model(p_gpu) / model(p_dir) >= 0.99


def _bj_norm2(mod, A, r):
    """rᵀ M⁻¹ r with M the block-Jacobi preconditioner of A (3×3 per soft vertex, 12×12 per DoF body)."""
    V = mod.V
    blocks = [(3 * v, 3) for v in range(V)] + [(3 * V + 12 * s, 12) for s in range(mod.n_dof_bodies)]
    t = 0.0
    for o, k in blocks:
        B = A[o:o + k, o:o + k].toarray()
        t += r[o:o + k] @ np.linalg.solve(B, r[o:o + k])
    return t


def test_soft_soft_contact_residual_pairs():
    """Scene P2 (two gel tets touching edge to edge at d̂/2): the pair joins two soft bodies, so the
    SpMV keeps it matrix-free; energies/gradient/HVP (exact and projected), the active set and the
    PCG solve match the oracle."""
    sc, mod, ctx, b, x, y = _perturbed("P2", 5, amp=2e-6)
    P = M.all_positions(mod, x, y)
    pairs = C.active_pairs(mod, P)
    assert len(pairs) >= 1
    assert np.array_equal(b.debug_active_pairs(0, x, y), pairs.keys())
    v = np.random.default_rng(1).normal(size=mod.n_dof)
    for exact in (False, True):
        et, g, hv = b.debug_eval(0, x, y, ctx.lam_att, ctx.lam_kin, ctx.rho, v, exact=exact)
        terms = En.energy_terms(mod, ctx, x, y, pairs)
        for i, k in enumerate(En.TERMS):
            assert abs(et[i] - terms[k]) <= REL * max(abs(terms[k]), 1e-300) + 1e-300, (k, et[i], terms[k])
        go, H = En.assemble(mod, ctx, x, y, pairs, project=not exact)
        assert rel_inf(g, go) <= REL
        assert rel_inf(hv, H @ v) <= REL
    p_gpu, it_gpu = b.debug_pcg(0, x, y)
    g, H = En.assemble(mod, ctx, x, y, pairs)
    p_ref, it_ref = SO.block_jacobi_pcg(mod, H, g, sc.config.pcg_eta, sc.config.max_pcg)
    assert abs(it_gpu - it_ref) <= max(2, it_ref // 50)
    assert rel_inf(p_gpu, p_ref) <= 1e-6


def test_soft_soft_trajectory_and_residual_path():
    """P2 with the upper tet moving down at 10 mm/s: 4 steps through tac_step against the oracle
    (positions within 1e-6·L_env), every step intersection-free, and the stats show residual
    (matrix-free) pairs in the solve."""
    sc = S.make_scene("P2")
    mod = M.prepare(sc)
    ei = S.env_inputs(sc, [0], n_steps=4)
    x0 = ei.x0[0]
    v0 = np.zeros_like(x0)
    v0[4:] = [0.0, 0.0, -0.01]                        # tet B (vertices 4..7) approaches tet A
    b = T.Batch(sc, 1)
    assert b.set_state(x0[None], ei.y0, v0[None])[0] == 0
    st = SO.State(x0.copy(), v0.copy(), ei.y0[0].copy(), np.zeros_like(ei.y0[0]))
    L = M.env_scale(mod, st.x, st.y)
    saw_res = False
    for k in range(4):
        assert b.step(1)[0] == 0
        st, stats = SO.step(mod, st, np.zeros((0, 12)), L_env=L)
        assert stats.status == 0
        x = b.get_state()[0].cpu().numpy()[0]
        assert np.abs(x - st.x).max() <= 1e-6 * L, (k, np.abs(x - st.x).max() / L)
        s = b.stats()[0]
        assert s["min_dist"] > 0
        assert C.min_distance(mod, M.all_positions(mod, x, st.y)) > 0
        saw_res |= s["n_residual"] > 0
    assert saw_res


# ------------------------------------------------------------------------------------------ failures

def _c1_batch(cfg=None, E=3):
    sc = S.make_scene("C1")
    if cfg:
        sc.config = dataclasses.replace(sc.config, **cfg)
    ei = S.env_inputs(sc, range(E), n_steps=2)
    return sc, ei


def _states(b):
    return [t.cpu().numpy() for t in b.get_state()]


def test_injected_fault_rolls_back_and_isolates():
    """tac_debug_inject_fault: env 1 of 3 fails (each status 1..4 in turn); it is rolled back bitwise to
    the step's start state and DISABLED until set_state; envs 0 and 2 are bitwise identical to a run
    without the fault (per-env independence)."""
    sc, ei = _c1_batch()
    ref = T.Batch(sc, 3)
    ref.set_state(ei.x0, ei.y0)
    ref.set_targets(ei.ykin[0])
    assert (ref.step(1) == 0).all()
    xr = _states(ref)
    for status in (1, 2, 3, 4):
        b = T.Batch(sc, 3)
        b.set_state(ei.x0, ei.y0)
        before = _states(b)
        b.set_targets(ei.ykin[0])
        b.debug_inject_fault(1, status)
        st = b.step(1)
        assert list(st) == [0, status, 0]
        after = _states(b)
        for a, r, s0 in zip(after, xr, before):
            assert np.array_equal(a[[0, 2]], r[[0, 2]])
            assert np.array_equal(a[1], s0[1])
        b.set_targets(ei.ykin[1])
        assert list(b.step(1)) == [0, 6, 0]                # stays DISABLED
        b.set_state(ei.x0[1:2], ei.y0[1:2], env0=1)        # re-enabled by set_state
        b.set_targets(ei.ykin[0])
        assert b.step(1)[1] == 0


def test_capacity_detected_per_env():
    """A candidate capacity of 64 per env: env 0 (cube pressed onto the pad: hundreds of candidates)
    fails with CAPACITY and is rolled back; env 1 (cube lifted 20 mm: no candidates) steps normally."""
    sc, ei = _c1_batch({"cand_capacity_per_env": 64}, E=2)
    y0 = ei.y0.copy()
    y0[1, 1, 2] += 20e-3
    y0[0, 1, 2] -= 0.2e-3 - 0.04e-3
    b = T.Batch(sc, 2)
    assert list(b.set_state(ei.x0, y0)) == [3, 0]         # detected at set_state already
    # in a step: both envs valid at the start (env 0's cube 0.2 mm above the pad, env 1's 20 mm above);
    # env 0's target presses into the pad, env 1 holds still
    y1 = ei.y0.copy()
    y1[1, 1, 2] += 20e-3
    b2 = T.Batch(sc, 2)
    assert list(b2.set_state(ei.x0, y1)) == [0, 0]
    before = _states(b2)
    tk = np.stack([ei.ykin[0, 0], y1[1, 1:2]])
    tk[0, 0, 2] -= 0.16e-3
    b2.set_targets(tk)
    st = b2.step(1)
    assert st[0] == 3 and st[1] == 0, st
    after = _states(b2)
    for a, s0 in zip(after, before):
        assert np.array_equal(a[0], s0[0])                # rolled back


def test_newton_stall_and_al_infeasible_detected():
    """max_newton = 1: every env that needs a second Newton iteration stalls (NEWTON_STALL) and is
    rolled back; max_al_rounds = 1 with an AL tolerance below the first round's residual:
    AL_INFEASIBLE."""
    sc, ei = _c1_batch({"max_newton": 1}, E=2)
    b = T.Batch(sc, 2)
    b.set_state(ei.x0, ei.y0)
    before = _states(b)
    b.set_targets(ei.ykin[0])
    assert list(b.step(1)) == [1, 1]
    for a, s0 in zip(_states(b), before):
        assert np.array_equal(a, s0)
    sc2, ei2 = _c1_batch({"max_al_rounds": 1, "al_tol_rel": 1e-14}, E=2)
    b = T.Batch(sc2, 2)
    b.set_state(ei2.x0, ei2.y0)
    b.set_targets(ei2.ykin[0])
    assert list(b.step(1)) == [2, 2]


def test_resident_pcg_512_budget_parity():
    """k_pcg_r512 (the 512-thread register budget, used by envs needing more than 384 threads) against
    the oracle PCG: forced with TAC_PCG_R_LB512=1 in a fresh process (the choice is read once)."""
    env = dict(os.environ, TAC_PCG_R_LB512="1", TAC_PCG_CLUSTER="0")
    here = os.path.dirname(os.path.abspath(__file__))
    code = ("import sys; sys.path.insert(0, %r); from paper_2504_12908_b200 import scenes as S, taccel as T; "
            "b = T.Batch(S.make_scene('C2'), 1); print(b.pcg_kernel)" % os.path.dirname(here))
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True)
    assert r.stdout.strip() == "k_pcg_r512", r.stdout + r.stderr
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-m", "gpu", "-k", "pcg_matches_oracle",
                        os.path.join(here, "test_gpu_parity.py")], env=env, capture_output=True, text=True)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]
    assert " passed" in r.stdout


@pytest.mark.parametrize("nc", [2, 4])
def test_cluster_pcg_split_over_ctas(nc):
    """k_pcg_cl with the env's rows split over a cluster of nc CTAs (neighbouring rows read through
    distributed shared memory, bodies and couplings across CTAs) — forced on C1/C2 with
    TAC_PCG_CLUSTER=nc in a fresh process — passes the oracle PCG, LM-solve and trajectory parity tests."""
    env = dict(os.environ, TAC_PCG_CLUSTER=str(nc))
    here = os.path.dirname(os.path.abspath(__file__))
    code = ("import sys; sys.path.insert(0, %r); from paper_2504_12908_b200 import scenes as S, taccel as T; "
            "b = T.Batch(S.make_scene('C2'), 1); print(b.pcg_kernel)" % os.path.dirname(here))
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True)
    assert r.stdout.strip() == "k_pcg_cl", r.stdout + r.stderr
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-m", "gpu", "-k",
                        "pcg_matches_oracle or trajectory_parity or lm_exact or batch_equals_solo",
                        os.path.join(here, "test_gpu_parity.py"), os.path.join(here, "test_gpu_contact.py")],
                       env=env, capture_output=True, text=True)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]
    assert " passed" in r.stdout


# ------------------------------------------------------------------------------------------ friction

def _with_friction(sc, mu=0.5):
    sc.config = dataclasses.replace(sc.config, mu_friction=mu, eps_v=1e-3)
    return sc


@pytest.mark.parametrize("name,slide", [("C1", 0.0), ("C1", 3e-6), ("P1", 2e-5), ("P2", 1e-6)])
def test_friction_energy_gradient_hvp_parity(name, slide):
    """Lagged friction D_k (reading R20) through the C ABI: the seven energy terms (friction
    included), the gradient and the (exact, PSD) Hessian-vector product at an iterate slid away from
    xⁿ match the oracle within 1e-9; the friction pairs are frozen at the env's state xⁿ on both sides."""
    sc = _with_friction(S.make_scene(name))
    mod = M.prepare(sc)
    ei = S.env_inputs(sc, [0], n_steps=1)
    xn, yn = ei.x0[0].copy(), ei.y0[0].copy()
    if name == "C1":
        yn[1, 2] -= 0.2e-3 - 0.04e-3                      # cube 40 µm above the pad: PT and EE pairs
    rng = np.random.default_rng(21)
    x = xn + rng.normal(size=xn.shape) * slide
    if name == "P1":
        x[0] += slide * np.array([0.6, 0.8, 0.0])       # apex slides past the dynamic plateau
    y = yn.copy()
    yk = ei.ykin[0, 0] if ei.ykin.shape[2] else np.zeros((0, 12))
    if name == "C1":
        y[1, :3] += np.array([2e-6, -1e-6, -5e-6])        # the kinematic cube's iterate moves too
    ctx = En.make_context(mod, xn, np.zeros_like(xn), yn, np.zeros_like(yn), yk, sc.config.dt)
    assert len(ctx.fric) > 0
    b = T.Batch(sc, 1)
    assert b.set_state(xn[None], yn[None])[0] == 0
    if ei.ykin.shape[2]:
        b.set_targets(ei.ykin[0])
    pairs = C.active_pairs(mod, M.all_positions(mod, x, y))
    v = rng.normal(size=mod.n_dof)
    et, g, hv = b.debug_eval(0, x, y, ctx.lam_att, ctx.lam_kin, ctx.rho, v, exact=True)
    terms = En.energy_terms(mod, ctx, x, y, pairs)
    assert terms["friction"] > 0
    # terms that vanish analytically here (elastic at rest, orthogonality of a rotation) are rounding
    # noise on both sides: they are compared relative to 1e-12 of the total energy instead
    floor = 1e-12 * sum(abs(t) for t in terms.values())
    for i, k in enumerate(En.TERMS):
        assert abs(et[i] - terms[k]) <= max(REL * abs(terms[k]), floor), (k, et[i], terms[k])
    go, H = En.assemble(mod, ctx, x, y, pairs, project=False)
    assert rel_inf(g, go) <= REL
    assert rel_inf(hv, H @ v) <= REL


@pytest.mark.parametrize("name,n_steps", [("C1", 10)])
def test_friction_trajectory_parity(name, n_steps):
    """C1 with μ = 0.5: 10 steps through tac_step against the oracle (positions within 1e-6·L_env)."""
    sc = _with_friction(S.make_scene(name))
    mod = M.prepare(sc)
    ei = S.env_inputs(sc, [0], n_steps=n_steps)
    b = T.Batch(sc, 1)
    assert b.set_state(ei.x0, ei.y0)[0] == 0
    st = SO.State(ei.x0[0].copy(), np.zeros_like(ei.x0[0]), ei.y0[0].copy(), np.zeros_like(ei.y0[0]))
    L = M.env_scale(mod, st.x, st.y)
    nfr = 0
    for k in range(n_steps):
        b.set_targets(ei.ykin[k])
        assert b.step(1)[0] == 0
        st, stats = SO.step(mod, st, ei.ykin[k, 0], L_env=L)
        assert stats.status == 0
        x, _, y, _ = (t.cpu().numpy()[0] for t in b.get_state())
        err = np.abs(M.all_positions(mod, x, y) - M.all_positions(mod, st.x, st.y)).max() / L
        assert err <= 1e-6, (k, err)
        nfr = max(nfr, b.stats()[0]["n_friction"])
    assert nfr > 0


def _incline_scene(mu, tan_theta):
    import math
    th = math.atan(tan_theta)
    pV, pT = S.box_surface((0.04, 0.04, 0.01))
    cV, cT = S.box_surface((0.01, 0.01, 0.01))
    g = 9.81 * np.array([math.sin(th), 0.0, -math.cos(th)])
    cfg = dataclasses.replace(S.Config(dt=0.01), mu_friction=mu, eps_v=1e-3)
    sc = S.Scene("C1", [], [S.AffineBody(pV, pT, kind=S.STATIC), S.AffineBody(cV, cT, kind=S.DYNAMIC)], g, cfg, n_steps=1)
    y0 = np.array([S.pose([0, 0, -0.005]), S.pose([0.0013, 0.0007, 0.005 + 0.5e-4], S.rot_z(0.3))])
    return sc, y0


@pytest.mark.parametrize("mu", [0.2, 0.5])
def test_friction_incline_stick_slip_matches_oracle(mu):
    """The incline pin on the GPU: a cube on a plane tilted to tan θ = 0.9μ sticks and at
    1.1μ slides with growing per-step displacement; both trajectories match the oracle step by step."""
    eps_dt = 1e-3 * 0.01
    for t, stick in ((0.9 * mu, True), (1.1 * mu, False)):
        sc, y0 = _incline_scene(mu, t)
        mod = M.prepare(sc)
        b = T.Batch(sc, 1)
        assert b.set_state(np.zeros((1, 0, 3)), y0[None])[0] == 0
        st = SO.State(np.zeros((0, 3)), np.zeros((0, 3)), y0.copy(), np.zeros_like(y0))
        L = M.env_scale(mod, st.x, st.y)
        xs = []
        for k in range(12):
            assert b.step(1)[0] == 0
            st, stats = SO.step(mod, st, np.zeros((0, 12)), L_env=L)
            y = b.get_state()[2].cpu().numpy()[0]
            err = np.abs(M.all_positions(mod, np.zeros((0, 3)), y) - M.all_positions(mod, np.zeros((0, 3)), st.y)).max() / L
            assert err <= 1e-6, (mu, t, k, err)
            xs.append(y[1, 0])
        dx = np.diff(np.array(xs))[4:]
        if stick:
            assert np.all(np.abs(dx) < 10 * eps_dt), dx
        else:
            assert np.all(dx > 0) and np.all(np.diff(dx) > 0), dx


# ------------------------------------------------------------------------------------------ depth maps

@pytest.mark.parametrize("name,E,steps", [("C1", 2, 6), ("C2", 3, 12)])
def test_depth_normal_maps_match_oracle(name, E, steps):
    """tac_get_depth_maps (reading R22) after `steps` lockstep steps (pads pressed): depth
    and normal maps of every pad of every env match the oracle rasteriser within 1e-12 (NaN pattern
    identical), at a non-square resolution."""
    from oracle import tactile as Tc
    sc = S.make_scene(name)
    mod = M.prepare(sc)
    ei = S.env_inputs(sc, range(E), n_steps=steps)
    b = T.Batch(sc, E)
    assert (b.set_state(ei.x0, ei.y0) == 0).all()
    for k in range(steps):
        b.set_targets(ei.ykin[k])
        assert (b.step(1) == 0).all()
    H, W = 17, 23
    d, nm = (t.cpu().numpy() for t in b.get_depth_maps(H, W))
    x_all, _, y_all, _ = (t.cpu().numpy() for t in b.get_state())
    deepest = 0.0
    for e in range(E):
        Do, No = Tc.depth_maps(mod, x_all[e], y_all[e], H, W)
        assert np.array_equal(np.isnan(d[e]), np.isnan(Do))
        ok = ~np.isnan(Do)
        assert np.abs(d[e][ok] - Do[ok]).max() <= 1e-12
        assert np.abs(nm[e] - No).max() <= 1e-12
        deepest = max(deepest, np.nanmax(Do))
    assert deepest > 1e-5                                 # some pad is indented
