"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle on the same seeded inputs.

Bars (BASELINE.json north_star): contact-pair sets bit-exact; energies, gradients and
Hessian-vector products within 1e-9 relative (fp64); positions after each converged step within
1e-6·L_env."""
import dataclasses

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

REL = 1e-9


def rel_inf(a, b):
    return np.abs(np.asarray(a) - np.asarray(b)).max() / max(np.abs(a).max(), np.abs(b).max(), 1e-300)


@pytest.fixture(scope="module", autouse=True)
def _built():
    build()


def _perturbed(name, seed, amp=2e-5, press=None):
    # frictionless operator: these cases check the projected and exact barrier/elastic Hessians and the
    # PCG on them (friction batches use the exact Hessian only; friction parity: test_gpu_contact.py)
    sc = S.make_scene(name)
    sc.config = dataclasses.replace(sc.config, mu_friction=0.0)
    mod = M.prepare(sc)
    ei = S.env_inputs(sc, [0], n_steps=1)
    rng = np.random.default_rng(seed)
    xn, yn = ei.x0[0], ei.y0[0]
    v = rng.normal(size=xn.shape) * 1e-3
    yd = np.zeros_like(yn)
    for b in range(len(yn)):
        if mod.dof_slot[b] >= 0:
            yd[b] = rng.normal(size=12) * 1e-3 * np.r_[np.ones(3), np.full(9, 0.01)]
    x = xn + rng.normal(size=xn.shape) * amp
    y = yn.copy()
    for b in range(len(y)):
        if mod.dof_slot[b] >= 0:
            y[b] += rng.normal(size=12) * amp * np.r_[np.full(3, 0.25), np.full(9, 0.01)]
    if press is not None:
        press(y)
    ctx = En.make_context(mod, xn, v, yn, yd, ei.ykin[0, 0], sc.config.dt)
    ctx.lam_att = rng.normal(size=ctx.lam_att.shape) * 1e-6
    ctx.lam_kin = rng.normal(size=ctx.lam_kin.shape) * 1e-6
    ctx.rho = sc.config.al_rho0 * 2.0
    return sc, mod, ei, (xn, v, yn, yd), ctx, x, y


def _c1_press(y):
    y[1, 2] -= 0.2e-3 - 0.04e-3          # cube bottom 40 µm above the pad top → PT + EE pairs


def _batch_for(sc, base, ei, n_envs=1):
    b = T.Batch(sc, n_envs)
    xn, v, yn, yd = base
    b.set_state(np.repeat(xn[None], n_envs, 0), np.repeat(yn[None], n_envs, 0),
                np.repeat(v[None], n_envs, 0), np.repeat(yd[None], n_envs, 0))
    if ei.ykin.shape[2]:
        b.set_targets(np.repeat(ei.ykin[0, 0][None], n_envs, 0))
    return b


CASES = [("C1", 11, _c1_press), ("C1", 12, _c1_press), ("C1b", 13, None), ("C2", 14, None)]


@pytest.mark.parametrize("name,seed,press", CASES)
def test_energy_gradient_hvp_parity(name, seed, press):
    sc, mod, ei, base, ctx, x, y = _perturbed(name, seed, press=press)
    b = _batch_for(sc, base, ei)
    pairs = C.active_pairs(mod, M.all_positions(mod, x, y))
    if name in ("C1", "C2"):
        assert len(pairs) > 0
    rng = np.random.default_rng(seed + 100)
    v = rng.normal(size=mod.n_dof)
    et, g, hv = b.debug_eval(0, x, y, ctx.lam_att, ctx.lam_kin, ctx.rho, v)
    terms = En.energy_terms(mod, ctx, x, y, pairs)
    for i, k in enumerate(En.TERMS):
        ref = terms[k]
        assert abs(et[i] - ref) <= REL * max(abs(ref), 1e-300) + 1e-300, (k, et[i], ref)
    go, H = En.assemble(mod, ctx, x, y, pairs)
    assert rel_inf(g, go) <= REL
    assert rel_inf(hv, H @ v) <= REL
    # unprojected (exact) Hessian, used first by hessian_mode 1 (reading R14b)
    _, _, hv_x = b.debug_eval(0, x, y, ctx.lam_att, ctx.lam_kin, ctx.rho, v, exact=True)
    _, Hx = En.assemble(mod, ctx, x, y, pairs, project=False)
    assert rel_inf(hv_x, Hx @ v) <= REL


@pytest.mark.parametrize("name,seed,press", CASES)
def test_active_set_bit_exact(name, seed, press):
    sc, mod, ei, base, ctx, x, y = _perturbed(name, seed, press=press)
    b = _batch_for(sc, base, ei)
    P = M.all_positions(mod, x, y)
    cand = C.candidate_pairs(mod, P)
    _, d2 = C.classify(mod, P, cand)
    dh2 = sc.config.dhat ** 2
    assert np.all(np.abs(d2 - dh2) > 1e-9 * dh2)          # generator guard band (reading R9)
    ref = C.active_pairs(mod, P).keys()
    got = b.debug_active_pairs(0, x, y)
    assert np.array_equal(got, ref)
    # static candidate set = brute-force AABB-overlap set (same predicate, canonical order)
    assert np.array_equal(b.debug_candidates(0, x, y), cand)


@pytest.mark.parametrize("name,seed,press", CASES[:2] + CASES[3:])
def test_swept_candidates_and_accd(name, seed, press):
    sc, mod, ei, base, ctx, x, y = _perturbed(name, seed, press=press)
    b = _batch_for(sc, base, ei)
    rng = np.random.default_rng(seed + 7)
    p = rng.normal(size=mod.n_dof) * (3e-6 if seed % 2 else 1e-4)      # K_eff = 8 / 1
    p[3 * mod.V:] *= 0.05
    P = M.all_positions(mod, x, y)
    dx, dy = En.unpack(mod, p, np.zeros_like(y))
    Pd = SO._disp_positions(mod, dx, dy)
    K = SO.sweep_factor(sc.config, SO.embedded_inf_norm(mod, p))
    cand = C.candidate_pairs(mod, P, P + K * Pd)
    got = b.debug_candidates(0, x, y, p)
    assert np.array_equal(got, cand)
    a_ref = K * C.accd_bound(mod, P, K * Pd, cand)
    a_gpu = b.debug_accd(0, x, y, p)
    assert a_gpu == pytest.approx(a_ref, rel=1e-9)


@pytest.mark.parametrize("name,seed,press", CASES[:1] + CASES[3:])
def test_pcg_matches_oracle_pcg_and_direct(name, seed, press):
    sc, mod, ei, base, ctx, x, y = _perturbed(name, seed, press=press)
    ctx.lam_att[:] = 0
    ctx.lam_kin[:] = 0
    ctx.rho = sc.config.al_rho0
    b = _batch_for(sc, base, ei)
    p_gpu, it_gpu = b.debug_pcg(0, x, y)
    pairs = C.active_pairs(mod, M.all_positions(mod, x, y))
    g, H = En.assemble(mod, ctx, x, y, pairs)
    p_ref, it_ref = SO.block_jacobi_pcg(mod, H, g, sc.config.pcg_eta, sc.config.max_pcg)
    assert abs(it_gpu - it_ref) <= max(2, it_ref // 50)
    assert rel_inf(p_gpu, p_ref) <= 1e-6
    import scipy.sparse.linalg as spla
    p_dir = spla.spsolve(H.tocsc(), -g)
    assert g @ p_gpu < 0
    # CG minimises the quadratic model m(p) = gᵀp + ½pᵀHp; the truncated iterate reaches ≥ 99% of
    # the exact Newton model decrease
    model = lambda q: g @ q + 0.5 * q @ (H @ q)
    assert model(p_gpu) / model(p_dir) >= 0.99


def _oracle_run(sc, mod, ei, n_steps):
    st = SO.State(ei.x0[0].copy(), np.zeros_like(ei.x0[0]), ei.y0[0].copy(), np.zeros_like(ei.y0[0]))
    L = M.env_scale(mod, st.x, st.y)
    out = []
    for k in range(n_steps):
        st, stats = SO.step(mod, st, ei.ykin[k, 0] if ei.ykin.shape[2] else np.zeros((0, 12)), L_env=L)
        out.append((st, stats))
    return out, L


@pytest.mark.parametrize("name,n_steps", [("C1", 10), ("C1b", 6)])
def test_trajectory_parity_and_invariants(name, n_steps):
    sc = S.make_scene(name)
    mod = M.prepare(sc)
    ei = S.env_inputs(sc, [0], n_steps=n_steps)
    b = T.Batch(sc, 1)
    assert b.set_state(ei.x0, ei.y0)[0] == 0
    ref, L = _oracle_run(sc, mod, ei, n_steps)
    for k in range(n_steps):
        if ei.ykin.shape[2]:
            b.set_targets(ei.ykin[k])
        st = b.step(1)
        assert st[0] == 0, T.ENV_STATUS[int(st[0])]
        x, xd, y, yd = (t.cpu().numpy()[0] for t in b.get_state())
        ost, ostats = ref[k]
        assert ostats.status == 0
        P = M.all_positions(mod, x, y)
        Po = M.all_positions(mod, ost.x, ost.y)
        assert np.abs(P - Po).max() <= 1e-6 * L, (k, np.abs(P - Po).max() / L)
        # invariants on the GPU state: inversion- and intersection-free
        assert not SO.any_inverted(mod, x)
        assert C.min_distance(mod, P) > 0
    # readout parity on the final state
    coat, mpos, mflow = (t.cpu().numpy()[0] for t in b.get_gel_deformation())
    o = R.gel_deformation(mod, x, y)
    oc = np.concatenate([a[0] for a in o])
    om = np.concatenate([a[1] for a in o])
    of = np.concatenate([a[2] for a in o])
    assert np.abs(coat - oc).max() <= 1e-12 and np.abs(mpos - om).max() <= 1e-15 and np.abs(mflow - of).max() <= 1e-12
    s = b.stats()[0]
    assert s["status"] == 0 and s["newton_iters"] > 0 and s["pcg_iters"] > 0


def test_batch_equals_solo_bitwise():
    """Per-env results are independent of the batch size and of the env's position (S:L589-590,
    SURVEY §8(e) sharding equivalence)."""
    sc = S.make_scene("C1")
    ei = S.env_inputs(sc, [0, 1, 2], n_steps=3)
    big = T.Batch(sc, 3)
    big.set_state(ei.x0, ei.y0)
    solo = T.Batch(sc, 1)
    solo.set_state(ei.x0[2:3], ei.y0[2:3])
    for k in range(3):
        big.set_targets(ei.ykin[k])
        solo.set_targets(ei.ykin[k, 2:3])
        assert (big.step(1) == 0).all() and solo.step(1)[0] == 0
    xb = big.get_state()[0].cpu().numpy()[2]
    xs = solo.get_state()[0].cpu().numpy()[0]
    assert np.array_equal(xb, xs)
    # repeat run: bitwise deterministic
    again = T.Batch(sc, 1)
    again.set_state(ei.x0[2:3], ei.y0[2:3])
    for k in range(3):
        again.set_targets(ei.ykin[k, 2:3])
        again.step(1)
    assert np.array_equal(again.get_state()[0].cpu().numpy()[0], xs)


def test_bad_state_detected_and_isolated():
    sc = S.make_scene("C1")
    ei = S.env_inputs(sc, [0, 1], n_steps=1)
    x0 = ei.x0.copy()
    t = sc.soft[0].tets[0]
    x0[1, t[0]] = x0[1, t[1]] + (x0[1, t[1]] - x0[1, t[0]])     # invert one tet of env 1
    b = T.Batch(sc, 2)
    st = b.set_state(x0, ei.y0)
    assert st[0] == 0 and st[1] == 5
    b.set_targets(ei.ykin[0])
    st = b.step(1)
    assert st[0] == 0 and st[1] == 6                     # DISABLED until the next set_state


def _free_body_scene(gravity):
    V, Tr = S.box_surface((0.01, 0.01, 0.01))
    body = S.AffineBody(V, Tr, kind=S.DYNAMIC)
    return S.Scene("C1", [], [body], np.array(gravity, float), S.Config(dt=0.01), n_steps=1)


def test_free_fall_and_fixed_point_through_abi():
    """Closed forms through the C ABI: a free affine body moves by Δt v⁰ + Δt² g in one Newton
    step; with no forces the state is a fixed point."""
    sc = _free_body_scene((0, 0, -9.81))
    b = T.Batch(sc, 2)
    y0 = np.array([[[0.1, 0.2, 0.3, *S.rot_z(0.4).ravel()]], [[0.0, 0.0, 1.0, *np.eye(3).ravel()]]])
    yd0 = np.array([[[0.5, -0.2, 0.1, *np.zeros(9)]], [[0.0] * 12]])
    b.set_state(np.zeros((2, 0, 3)), y0, None, yd0)
    assert (b.step(1) == 0).all()
    y = b.get_state()[2].cpu().numpy()
    dt = sc.config.dt
    for e in range(2):
        expect = y0[e, 0, :3] + dt * yd0[e, 0, :3] + dt * dt * sc.gravity
        assert np.abs(y[e, 0, :3] - expect).max() <= 1e-15
        assert np.abs(y[e, 0, 3:] - y0[e, 0, 3:]).max() <= 1e-15
    sc0 = _free_body_scene((0, 0, 0))
    b0 = T.Batch(sc0, 1)
    b0.set_state(np.zeros((1, 0, 3)), y0[:1])
    assert b0.step(1)[0] == 0
    assert np.array_equal(b0.get_state()[2].cpu().numpy(), y0[:1])
    assert b0.stats()[0]["newton_iters"] == 1


@pytest.mark.parametrize("name,E,K", [("C1", 3, 4), ("C2", 6, 5)])
def test_schedule_matches_lockstep_bitwise(name, E, K):
    """tac_step_schedule (envs advance independently) == tac_set_targets + tac_step per step, bitwise,
    including the per-step gel readout."""
    sc = S.make_scene(name)
    ei = S.env_inputs(sc, range(E), n_steps=K)
    a = T.Batch(sc, E)
    a.set_state(ei.x0, ei.y0)
    ref = []
    for k in range(K):
        a.set_targets(ei.ykin[k])
        assert (a.step(1) == 0).all()
        ref.append([t.cpu().numpy() for t in a.get_gel_deformation()])
    xa = a.get_state()[0].cpu().numpy()
    b = T.Batch(sc, E)
    b.set_state(ei.x0, ei.y0)
    out = (np.zeros((K, E, b.n_coated, 3)), np.zeros((K, E, b.n_markers, 3)), np.zeros((K, E, b.n_markers, 3)))
    st = b.step_schedule(ei.ykin, out=out)
    assert (st == 0).all()
    assert np.array_equal(b.get_state()[0].cpu().numpy(), xa)
    for k in range(K):
        for j in range(3):
            assert np.array_equal(out[j][k], ref[k][j])


def test_streamed_pcg_path_parity():
    """The streamed-operator PCG (k_pcg, used when an env's operator does not fit one SM, e.g. C3)
    against the oracle PCG and direct solve on the same cases, forced with TAC_PCG_RESIDENT=0 in a
    fresh process (the launch choice is read once per process)."""
    import os
    import subprocess
    import sys
    env = dict(os.environ, TAC_PCG_RESIDENT="0")
    here = os.path.dirname(os.path.abspath(__file__))
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-m", "gpu", "-k", "pcg_matches_oracle",
                        os.path.join(here, "test_gpu_parity.py")], env=env, capture_output=True, text=True)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]
    assert " passed" in r.stdout


def test_chunked_assembly_scratch_bitwise():
    """The assembly scratch (per-tet and per-pair records) is sized for one chunk of envs and the Newton loop
    runs tets → pairs → assemble chunk by chunk (TAC_ASM_CHUNK).  C2 with 7 envs, 4 lockstep steps: chunks of
    3 envs (3 launches per phase, compacted env lists split across chunks) must give bitwise the states of
    the default single chunk."""
    import os
    import subprocess
    import sys
    here = os.path.dirname(os.path.abspath(__file__))
    code = ("import sys, hashlib, numpy as np, torch; sys.path.insert(0, %r)\n"
            "from paper_2504_12908_b200 import scenes as S, taccel as T\n"
            "sc = S.make_scene('C2'); ei = S.env_inputs(sc, np.arange(7), n_steps=4)\n"
            "b = T.Batch(sc, 7); b.set_state(ei.x0, ei.y0)\n"
            "for k in range(4):\n"
            "    b.set_targets(ei.ykin[k]); assert (b.step(1) == 0).all()\n"
            "h = hashlib.sha256(b''.join(t.cpu().numpy().tobytes() for t in b.get_state())).hexdigest()\n"
            "print(h, sum(s['n_friction'] for s in b.stats()))\n" % os.path.dirname(here))
    out = []
    for chunk in ("1024", "3"):
        r = subprocess.run([sys.executable, "-c", code], env=dict(os.environ, TAC_ASM_CHUNK=chunk),
                           capture_output=True, text=True)
        assert r.returncode == 0, r.stdout + r.stderr[-3000:]
        out.append(r.stdout.split())
    assert out[0][0] == out[1][0], out
    assert int(out[0][1]) > 0            # the default C2 workload carries frozen friction pairs
