"""GPU parity on the grasping workloads (BASELINE configs[3], configs[4]) and the
on-device forward kinematics:

* C4 (parallel gripper, star object k of 8, 256 envs per shape): lockstep through the closing phase,
  single steps from shared GPU states against the oracle on sampled envs, invariants on every sampled
  env;
* C5 (Allegro-like hand, 4 pads, 17 kinematic links, engraved tile): the link targets compiled on the
  device from joint targets (tac_set_joint_targets) against the oracle's homogeneous products (1e-12),
  and single steps from shared states in the grasp phase.
Bars (north_star): active sets bit-exact; energies/gradients/HVPs within 1e-9; positions within
1e-6·L_env."""
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
from oracle import kinematics as K
from oracle import mesh as M
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


def _lockstep(b, ykin_dev, k0, n):
    for k in range(k0, k0 + n):
        b.set_targets(ykin_dev[k])
        st = b.step(1)
        assert (st == 0).all(), (k, np.unique(st, return_counts=True))
        b.get_gel_deformation()


def _single_step(sc, mod, ei, b, ykin_dev, k, envs):
    """Shared-state single step: active set, energy terms, gradient, HVP at the GPU
    state after k steps; then both sides advance step k and positions must agree within 1e-6·L_env."""
    x_all, xd_all, y_all, yd_all = (t.cpu().numpy() for t in b.get_state())
    b.set_targets(ykin_dev[k])
    rng = np.random.default_rng(k)
    done = []
    for e in envs:
        x, v, y, yd = x_all[e], xd_all[e], y_all[e], yd_all[e]
        P = M.all_positions(mod, x, y)
        _, d2 = C.classify(mod, P, C.candidate_pairs(mod, P))
        dh2 = sc.config.dhat ** 2
        if not np.all(np.abs(d2 - dh2) > 1e-9 * dh2):       # reading R9 tie guard band
            continue
        pairs = C.active_pairs(mod, P)
        assert np.array_equal(b.debug_active_pairs(e, x, y), pairs.keys())
        ctx = En.make_context(mod, x, v, y, yd, ei.ykin[k, e], sc.config.dt)
        vv = rng.normal(size=mod.n_dof)
        et, g, hv = b.debug_eval(e, x, y, ctx.lam_att, ctx.lam_kin, ctx.rho, vv, exact=True)
        terms = En.energy_terms(mod, ctx, x, y, pairs)
        floor = 1e-12 * sum(abs(t) for t in terms.values())
        for i, name in enumerate(En.TERMS):
            assert abs(et[i] - terms[name]) <= max(1e-9 * abs(terms[name]), floor), (k, e, name)
        go, H = En.assemble(mod, ctx, x, y, pairs, project=False)
        rel = lambda a, c: np.abs(a - c).max() / max(np.abs(a).max(), np.abs(c).max())
        assert rel(g, go) <= 1e-9 and rel(hv, H @ vv) <= 1e-9, (k, e)
        done.append((e, (x, v, y, yd), len(pairs)))
    assert done
    assert (b.step(1) == 0).all()
    x1, _, y1, _ = (t.cpu().numpy() for t in b.get_state())
    for e, (x, v, y, yd), _ in done:
        L = M.env_scale(mod, ei.x0[e], ei.y0[e])
        ost, ostats = SO.step(mod, SO.State(x.copy(), v.copy(), y.copy(), yd.copy()), ei.ykin[k, e], L_env=L)
        assert ostats.status == 0
        err = np.abs(M.all_positions(mod, x1[e], y1[e]) - M.all_positions(mod, ost.x, ost.y)).max() / L
        assert err <= 1e-6, (k, e, err)
        assert not SO.any_inverted(mod, x1[e])
        assert C.min_distance(mod, M.all_positions(mod, x1[e], y1[e])) > 0
    return done


@pytest.mark.parametrize("shape", [0, 5])
def test_c4_grasp_single_steps_from_shared_states(shape):
    """C4 star object `shape`, 256 envs (one homogeneous batch of the 2048-env workload): lockstep to
    step 30 (closing) and 61 (object squeezed), sampled envs 0 and 255 step once on the GPU and in the
    oracle from the shared state."""
    sc = S.make_scene(f"C4:{shape}")
    E = 256
    ei = S.env_inputs(sc, np.arange(E), n_steps=62)
    b = T.Batch(sc, E)
    assert (b.set_state(ei.x0, ei.y0) == 0).all()
    ykin = torch.tensor(ei.ykin, device=torch.device("cuda", 0))
    mod = M.prepare(sc)
    _lockstep(b, ykin, 0, 30)
    _single_step(sc, mod, ei, b, ykin, 30, (0, 255))
    _lockstep(b, ykin, 31, 30)
    n = [c[2] for c in _single_step(sc, mod, ei, b, ykin, 61, (0, 255))]
    assert max(n) > 0                                      # the pads squeeze the object


def test_c5_device_fk_matches_homogeneous_products():
    """tac_set_joint_targets (on-device action compilation) on a 64-env C5 batch: the 17 link
    targets of every env match the oracle's 4×4 homogeneous products (oracle/kinematics.py) to 1e-12 and
    the scene generator's targets (fk_hand) to 1e-12."""
    sc = S.make_scene("C5")
    E = 64
    ei = S.env_inputs(sc, np.arange(E), n_steps=100)
    b = T.Batch(sc, E)
    ch = S.hand_chain()
    b.set_chain(ch)
    yp = S.hand_palm_pose()
    for k in (0, 50, 99):
        q = np.stack([S.hand_script(e, 100)[k].reshape(-1) for e in range(E)])
        b.set_joint_targets(q, base=np.repeat(yp[None], E, 0))
        got = b.get_targets()
        for e in (0, 17, 63):
            ref = K.forward(ch, yp, q[e])
            assert np.abs(got[e] - ref).max() <= 1e-12
            assert np.abs(got[e] - ei.ykin[k, e]).max() <= 1e-12


def test_c5_hand_grasp_single_steps():
    """C5 (4 pads, 17 kinematic links, engraved tile), 128 envs (the per-GPU share of 1024 on 8 GPUs):
    targets compiled on the device from the joint script each step; lockstep to step 60 (pads pressing the
    tile faces, env 0) and 85 (oscillation, env 127) one env steps once on the GPU and in the oracle (the
    oracle step of an engraved-tile env takes minutes: ~12k active pairs through autograd)."""
    sc = S.make_scene("C5")
    E = 128
    ei = S.env_inputs(sc, np.arange(E), n_steps=86)
    b = T.Batch(sc, E)
    assert (b.set_state(ei.x0, ei.y0) == 0).all()
    b.set_chain(S.hand_chain())
    yp = np.repeat(S.hand_palm_pose()[None], E, 0)
    scripts = np.stack([S.hand_script(e, 86).reshape(86, -1) for e in range(E)], 1)   # (S, E, 16)
    qdev = torch.tensor(scripts, device=torch.device("cuda", 0))
    mod = M.prepare(sc)
    ykin = torch.tensor(ei.ykin, device=torch.device("cuda", 0))
    for k in range(60):
        b.set_joint_targets(qdev[k], base=yp)
        assert (b.step(1) == 0).all(), k
    n = [c[2] for c in _single_step(sc, mod, ei, b, ykin, 60, (0,))]
    assert max(n) > 0
    for k in range(61, 85):
        b.set_joint_targets(qdev[k], base=yp)
        assert (b.step(1) == 0).all(), k
    _single_step(sc, mod, ei, b, ykin, 85, (127,))
