"""Pins for the CPU oracle: each test ties an oracle function to something other than itself —
values the paper fixes (tests/golden/closed_forms.json), closed forms, invariants, special cases
that reduce to a textbook result, and brute force on tiny inputs."""
import json
import math
import os

import numpy as np
import pytest
import torch

from paper_2504_12908_b200 import scenes as S
from oracle import contact as C
from oracle import distance as D
from oracle import energy as En
from oracle import mesh as M
from oracle import readout as R
from oracle import solver as SO

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "closed_forms.json")))
T = torch.as_tensor


def unit_tet():
    return np.array([[0, 0, 0], [1, 0, 0], [0, 1, 0], [0, 0, 1]], float), np.array([[0, 1, 2, 3]])


# ------------------------------------------------------------------------------------ mesh

def test_unit_simplex_volume_and_mass():
    X, tets = unit_tet()
    Dinv, vol = M.tet_rest(X, tets)
    assert vol[0] == pytest.approx(1 / 6, rel=1e-15)
    g = GOLD["lumped_mass_unit_simplex"]
    m = M.lumped_mass(4, tets, vol, g["density"])
    assert np.allclose(m, g["mass_per_vertex"], rtol=1e-14)


def test_orientation_fix_and_degenerate_reject():
    X, tets = unit_tet()
    flipped = tets[:, [0, 2, 1, 3]]
    assert np.array_equal(M.orient_tets(X, flipped)[0][[0, 3]], [0, 3])
    assert M.tet_rest(X, M.orient_tets(X, flipped))[1][0] > 0
    Xd = X.copy()
    Xd[3] = [0.5, 0.5, 0.0]
    with pytest.raises(ValueError):
        M.orient_tets(Xd, tets)


def test_single_tet_surface_outward():
    X, tets = unit_tet()
    F = M.boundary_faces(tets)
    assert len(F) == 4
    c = X.mean(0)
    for f in F:
        n = np.cross(X[f[1]] - X[f[0]], X[f[2]] - X[f[0]])
        assert np.dot(n, X[f].mean(0) - c) > 0


def test_lattice_surface_area_and_mass():
    pos, tets = S.lattice_tets(3, 3, 3, (1.0, 1.0, 1.0))
    tets = M.orient_tets(pos, tets)
    F = M.boundary_faces(tets)
    assert M.tri_area(pos, F).sum() == pytest.approx(6.0, rel=1e-13)
    Dinv, vol = M.tet_rest(pos, tets)
    assert vol.sum() == pytest.approx(1.0, rel=1e-13)
    m = M.lumped_mass(len(pos), tets, vol, 7.0)
    assert m.sum() == pytest.approx(7.0, rel=1e-12)
    # divergence-theorem volume of the extracted surface == Σ V_e (S:L52 property)
    v = np.einsum("ij,ij->i", pos[F[:, 0]], np.cross(pos[F[:, 1]], pos[F[:, 2]])).sum() / 6
    assert v == pytest.approx(1.0, rel=1e-12)


@pytest.mark.parametrize("offset", [(0, 0, 0), (0.3, -0.7, 1.1)])
def test_reduced_mass_box_closed_form(offset):
    a, b, c, rho = 0.3, 0.5, 0.7, 900.0
    V, Tr = S.box_surface((a, b, c), spacing=0.2)
    V = V + np.array(offset)
    vol, m, s1, My = M.body_moments(V, Tr, rho)
    mm = rho * a * b * c
    o = np.array(offset)
    S2 = mm * (np.outer(o, o) + np.diag([a * a, b * b, c * c]) / 12)
    assert vol == pytest.approx(a * b * c, rel=1e-12)
    assert np.allclose(s1, mm * o, rtol=1e-12, atol=1e-15)
    # M^y = I₃⊗[[m, s1ᵀ],[s1, S2]] in (t, A row-major) ordering (P:L113-116 JᵀMJ)
    for i in range(3):
        assert My[i, i] == pytest.approx(mm, rel=1e-12)
        for j in range(3):
            assert My[i, 3 + 3 * i + j] == pytest.approx(mm * o[j], rel=1e-12, abs=1e-15)
            for k in range(3):
                assert My[3 + 3 * i + j, 3 + 3 * i + k] == pytest.approx(S2[j, k], rel=1e-11, abs=1e-15)
    assert np.allclose(My, My.T)
    assert np.linalg.eigvalsh(My).min() > 0


def test_reduced_mass_L_shape_equals_sum_of_boxes():
    """Union of two boxes: moments add (linearity of ∫ over disjoint cells)."""
    xl, yl, zl = np.array([0, 1, 2.0]), np.array([0, 1.0]), np.array([0, 1, 2.0])
    solid = np.zeros((2, 1, 2), bool)
    solid[0, 0, 0] = solid[1, 0, 0] = solid[0, 0, 1] = True
    V, Tr = S.cell_union_surface(xl, yl, zl, solid)
    vol, m, s1, My = M.body_moments(V, Tr, 1.0)
    tot = np.zeros((12, 12))
    for c in ([0.5, 0.5, 0.5], [1.5, 0.5, 0.5], [0.5, 0.5, 1.5]):
        Vb, Tb = S.box_surface((1, 1, 1))
        tot += M.body_moments(Vb + np.array(c), Tb, 1.0)[3]
    assert vol == pytest.approx(3.0, rel=1e-12)
    assert np.allclose(My, tot, rtol=1e-12, atol=1e-14)


def test_reduced_kinetic_energy_equals_full_space():
    """½ẏᵀM^yẏ = ½∫ρ‖J ẏ‖² (P:L113 chain of equalities), checked by Monte-Carlo-free exact
    sampling: for a box the full-space integral of ‖v(x)‖² with v = ṫ + Ȧx is a quadratic
    polynomial integrated exactly by the box closed form."""
    a, b, c, rho = 0.2, 0.3, 0.4, 1000.0
    V, Tr = S.box_surface((a, b, c), spacing=0.1)
    My = M.body_moments(V, Tr, rho)[3]
    rng = np.random.default_rng(0)
    yd = rng.normal(size=12)
    td, Ad = yd[:3], yd[3:].reshape(3, 3)
    m = rho * a * b * c
    S2 = m * np.diag([a * a, b * b, c * c]) / 12
    full = 0.5 * (m * td @ td + np.trace(Ad @ S2 @ Ad.T))
    assert 0.5 * yd @ My @ yd == pytest.approx(full, rel=1e-11)


def test_rest_areas_partition_surface():
    sc = S.make_scene("C1")
    mod = M.prepare(sc)
    total = M.tri_area(mod.vert_xbar, mod.tris).sum()
    assert mod.A_v.sum() == pytest.approx(total, rel=1e-12)
    assert mod.A_e.sum() == pytest.approx(total, rel=1e-12)


def test_affine_jacobian_matches_fd_of_embedding():
    rng = np.random.default_rng(1)
    xb = rng.normal(size=3)
    y = rng.normal(size=12)
    J = M.affine_jacobian(xb)
    h = 1e-6
    for k in range(12):
        e = np.zeros(12)
        e[k] = h
        fd = (M.embed(y + e, xb[None])[0] - M.embed(y - e, xb[None])[0]) / (2 * h)
        assert np.allclose(fd, J[:, k], atol=1e-8)
    assert np.allclose(M.embed(np.r_[0, 0, 0, np.eye(3).ravel()], xb[None])[0], xb)


# ------------------------------------------------------------------------------------ energies

def test_barrier_closed_forms():
    g = GOLD["barrier"]
    dh = g["dhat"]
    d = T(np.array([dh, 0.5 * dh]), dtype=torch.float64).requires_grad_(True)
    b = En.barrier(d, dh)
    (gb,) = torch.autograd.grad(b.sum(), d, create_graph=True)
    (hb,) = torch.autograd.grad(gb.sum(), d)
    assert float(b[0]) == 0.0 and float(gb[0]) == 0.0 and float(hb[0]) == 0.0
    assert float(b[1]) / dh ** 2 == pytest.approx(g["b_at_half_over_dhat2"], rel=1e-14)
    assert float(gb[1]) / dh == pytest.approx(g["db_at_half_over_dhat"], rel=1e-14)
    assert float(hb[1]) == pytest.approx(g["d2b_at_half"], rel=1e-13)
    # support: zero beyond d̂, monotone decreasing inside
    dd = T(np.linspace(0.05, 2.0, 60) * dh)
    bb = En.barrier(dd, dh).numpy()
    assert np.all(bb[dd.numpy() >= dh] == 0)
    inside = bb[dd.numpy() < dh]
    assert np.all(np.diff(inside) < 0)


def test_neo_hookean_rest_and_rotation_invariance():
    mu, lam = M.lame(1e5, 0.4)
    F = torch.eye(3, dtype=torch.float64, requires_grad=True)
    psi = En.neo_hookean_psi(F, mu, lam)
    (P,) = torch.autograd.grad(psi, F)
    assert abs(float(psi)) < 1e-12 and float(P.abs().max()) < 1e-9
    rng = np.random.default_rng(2)
    Q, _ = np.linalg.qr(rng.normal(size=(3, 3)))
    Q *= np.sign(np.linalg.det(Q))
    Fr = rng.normal(size=(3, 3)) * 0.1 + np.eye(3)
    a = float(En.neo_hookean_psi(T(Fr), mu, lam))
    b = float(En.neo_hookean_psi(T(Q @ Fr), mu, lam))
    assert abs(a - b) < 1e-12 * max(1.0, abs(a))
    assert abs(float(En.neo_hookean_psi(T(Q), mu, lam))) < 1e-9


def test_neo_hookean_uniaxial_closed_form_and_rest_spectrum():
    mu, lam = 3.0, 5.0
    for s in (0.7, 1.0, 1.3):
        Fs = np.diag([s, 1.0, 1.0])
        closed = mu / 2 * (s * s - 1) - mu * math.log(s) + lam / 2 * math.log(s) ** 2
        assert float(En.neo_hookean_psi(T(Fs), mu, lam)) == pytest.approx(closed, rel=1e-13, abs=1e-14)
    H = torch.func.hessian(En.neo_hookean_psi)(torch.eye(3, dtype=torch.float64), mu, lam).reshape(9, 9).numpy()
    w = np.sort(np.linalg.eigvalsh(H))
    m = GOLD["neo_hookean_rest_spectrum"]["multiplicities"]
    assert np.allclose(w[:m["zero"]], 0, atol=1e-12)
    assert np.allclose(w[3:8], 2 * mu, rtol=1e-12)
    assert w[8] == pytest.approx(2 * mu + 3 * lam, rel=1e-12)


def test_ortho_energy_closed_forms():
    kap, vol = 1e8, 2e-6
    assert float(En.ortho_energy(torch.eye(3, dtype=torch.float64), kap, vol)) == 0.0
    R = S.rot_z(math.radians(30)) @ S.rot_y(0.3)
    assert abs(float(En.ortho_energy(T(R), kap, vol))) < 1e-12 * kap * vol
    e = 1e-3
    A = np.diag([1 + e, 1, 1])
    assert float(En.ortho_energy(T(A), kap, vol)) == pytest.approx(kap * vol * (2 * e + e * e) ** 2, rel=1e-12)


def test_mollifier_continuity():
    eps = 2.0
    c = T(np.array([eps * (1 - 1e-9), eps]), dtype=torch.float64).requires_grad_(True)
    m = En.ee_mollifier(c, eps)
    (dm,) = torch.autograd.grad(m.sum(), c)
    assert float(m[0]) == pytest.approx(1.0, abs=1e-12) and float(m[1]) == 1.0
    assert abs(float(dm[0])) < 1e-8 and float(dm[1]) == 0.0
    assert float(En.ee_mollifier(T(0.0), eps)) == 0.0


# ------------------------------------------------------------------------------------ distances

def _random_tri(rng):
    while True:
        t = rng.normal(size=(3, 3))
        if np.linalg.norm(np.cross(t[1] - t[0], t[2] - t[0])) > 0.3:
            return t


def _seg_dist2_dense(p, a, b, n=20001):
    s = np.linspace(0, 1, n)[:, None]
    return (((a + s * (b - a)) - p) ** 2).sum(1).min()


def test_pt_centroid_normal_distance():
    rng = np.random.default_rng(3)
    for _ in range(20):
        t = _random_tri(rng)
        n = np.cross(t[1] - t[0], t[2] - t[0])
        n /= np.linalg.norm(n)
        h = rng.uniform(0.01, 1)
        typ, d2 = D.pt_type(t.mean(0) + h * n, t[0], t[1], t[2])
        assert int(typ) == D.PT_T and math.sqrt(d2) == pytest.approx(h, rel=1e-12)


def test_pt_distance_vs_dense_sampling():
    """Brute force: min over a dense barycentric grid of the closed triangle."""
    rng = np.random.default_rng(4)
    nn = 400
    u, v = np.meshgrid(np.linspace(0, 1, nn), np.linspace(0, 1, nn))
    keep = (u + v) <= 1
    u, v = u[keep], v[keep]
    for _ in range(30):
        t = _random_tri(rng)
        p = rng.normal(size=3) * 1.5
        pts = t[0] + u[:, None] * (t[1] - t[0]) + v[:, None] * (t[2] - t[0])
        bf = ((pts - p) ** 2).sum(1).min()
        typ, d2 = D.pt_type(p, t[0], t[1], t[2])
        # the grid min is an upper bound within grid resolution of the exact min
        assert d2 <= bf + 1e-12
        assert math.sqrt(bf) - math.sqrt(d2) < 5e-3
        # classified sub-distance equals the exact closest-point distance on its sub-primitive
        if typ == D.PT_T:
            pass
        elif typ <= D.PT_E2:
            i = typ - D.PT_E0
            assert d2 == pytest.approx(_seg_dist2_dense(p, t[i], t[(i + 1) % 3]), rel=1e-6, abs=1e-12)
        else:
            assert d2 == pytest.approx(((p - t[typ - D.PT_V0]) ** 2).sum(), rel=1e-14)


def test_ee_closed_forms_and_grid():
    h = 0.37
    typ, d2 = D.ee_type([0, 0, 0], [1, 0, 0], [0.5, -0.5, h], [0.5, 0.5, h])
    assert int(typ) == D.EE_LL and math.sqrt(d2) == pytest.approx(h, rel=1e-13)
    typ, d2 = D.ee_type([0, 0, 0], [1, 0, 0], [0, h, 0], [1, h, 0])       # parallel
    assert math.sqrt(d2) == pytest.approx(h, rel=1e-13)
    rng = np.random.default_rng(5)
    s = np.linspace(0, 1, 200)
    for _ in range(30):
        a0, a1, b0, b1 = rng.normal(size=(4, 3))
        P = a0 + s[:, None, None] * (a1 - a0)
        Q = b0 + s[None, :, None] * (b1 - b0)
        bf = ((P - Q) ** 2).sum(-1).min()
        typ, d2 = D.ee_type(a0, a1, b0, b1)
        assert d2 <= bf + 1e-12
        assert math.sqrt(bf) - math.sqrt(d2) < 2e-2
        typ2, d2s = D.ee_type(b0, b1, a0, a1)                          # symmetry under swap
        assert d2s == pytest.approx(d2, rel=1e-9, abs=1e-14)


def test_distance_rigid_invariance():
    rng = np.random.default_rng(6)
    R = S.rot_z(0.7) @ S.rot_y(-0.4)
    t = rng.normal(size=3) * 10
    for _ in range(20):
        X = rng.normal(size=(4, 3))
        Y = X @ R.T + t
        assert D.pt_type(*X)[1] == pytest.approx(D.pt_type(*Y)[1], rel=1e-9, abs=1e-12)
        assert D.ee_type(*X)[1] == pytest.approx(D.ee_type(*Y)[1], rel=1e-9, abs=1e-12)


# ------------------------------------------------------------------------------------ gradients

def _perturbed_state(name, seed, amp=2e-5):
    sc = S.make_scene(name)
    mod = M.prepare(sc)
    ei = S.env_inputs(sc, [0], n_steps=1)
    rng = np.random.default_rng(seed)
    x = ei.x0[0] + rng.normal(size=ei.x0[0].shape) * amp
    y = ei.y0[0].copy()
    for b in range(len(y)):
        if mod.dof_slot[b] >= 0:
            y[b] += rng.normal(size=12) * amp * np.r_[np.ones(3), np.ones(9) * 0.01]
    v = rng.normal(size=x.shape) * 1e-3
    yd = rng.normal(size=y.shape) * 1e-3
    ctx = En.make_context(mod, ei.x0[0], v, ei.y0[0], yd, ei.ykin[0, 0], sc.config.dt)
    ctx.lam_att = rng.normal(size=ctx.lam_att.shape) * 1e-6
    ctx.lam_kin = rng.normal(size=ctx.lam_kin.shape) * 1e-6
    return sc, mod, ctx, x, y


def _press_state():
    """C1 with the cube pushed into the barrier zone (active PT and EE pairs)."""
    sc, mod, ctx, x, y = _perturbed_state("C1", 7)
    y[1, 2] -= 0.2e-3 - 0.04e-3          # cube bottom 40 µm above the pad top
    return sc, mod, ctx, x, y


def test_total_gradient_and_hvp_vs_finite_differences():
    """Unprojected gradient/HVP against central differences of the energy."""
    sc, mod, ctx, x, y = _press_state()
    pairs = C.active_pairs(mod, M.all_positions(mod, x, y))
    assert len(pairs) > 0 and (pairs.kind == 1).any() and (pairs.kind == 0).any()
    g, H = En.assemble(mod, ctx, x, y, pairs, project=False)
    q0 = En.pack(mod, x, y)
    rng = np.random.default_rng(8)
    v = rng.normal(size=q0.shape)
    h = 1e-9

    def E(q):
        xx, yy = En.unpack(mod, q, y)
        return En.total_energy(mod, ctx, xx, yy, pairs)
    fd = (E(q0 + h * v) - E(q0 - h * v)) / (2 * h)
    assert fd == pytest.approx(g @ v, rel=2e-5)

    def G(q):
        xx, yy = En.unpack(mod, q, y)
        return En.assemble(mod, ctx, xx, yy, pairs, project=False)[0]
    fdh = (G(q0 + h * v) - G(q0 - h * v)) / (2 * h)
    hv = H @ v
    assert np.abs(fdh - hv).max() <= 1e-4 * np.abs(hv).max()


def test_projected_hessian_is_psd_and_exact_at_rest():
    sc, mod, ctx, x, y = _press_state()
    pairs = C.active_pairs(mod, M.all_positions(mod, x, y))
    g, H = En.assemble(mod, ctx, x, y, pairs, project=True)
    Hd = H.toarray()
    assert np.allclose(Hd, Hd.T, atol=1e-12 * np.abs(Hd).max())
    assert np.linalg.eigvalsh(Hd).min() > 0
    # at the rest state no element clamp occurs: projected == unprojected (elastic part)
    sc2 = S.make_scene("C1")
    m2 = M.prepare(sc2)
    ei = S.env_inputs(sc2, [0], 1)
    ctx2 = En.make_context(m2, ei.x0[0], 0 * ei.x0[0], ei.y0[0], 0 * ei.y0[0], ei.ykin[0, 0], sc2.config.dt)
    e = En.Pairs(*(np.zeros(0, np.int64),) * 4, np.zeros(0))
    Hp = En.assemble(m2, ctx2, ei.x0[0], ei.y0[0], e, True)[1]
    Hu = En.assemble(m2, ctx2, ei.x0[0], ei.y0[0], e, False)[1]
    assert abs(Hp - Hu).max() <= 1e-12 * abs(Hu).max()


def test_affine_gravity_is_jacobian_pullback():
    """Affine gravity gradient equals Jᵀ of the full-space gradient −m g."""
    a, rho = 0.1, 1000.0
    V, Tr = S.box_surface((a, a, a), spacing=0.05)
    V = V + np.array([0.02, -0.01, 0.03])
    vol, m, s1, My = M.body_moments(V, Tr, rho)
    g = T([0.0, 0.0, -9.81])
    y = T(np.r_[0.1, 0.2, 0.3, (np.eye(3) + 0.01).ravel()]).requires_grad_(True)
    E = -(g * (m * y[:3] + y[3:].reshape(3, 3) @ T(s1))).sum()
    (gy,) = torch.autograd.grad(E, y)
    # ∫ρ J(x̄)ᵀ(−g) dV = [−m g ; −g ⊗ s1]
    expect = np.r_[-m * g.numpy(), np.outer(-g.numpy(), s1).ravel()]
    assert np.allclose(gy.numpy(), expect, rtol=1e-12, atol=1e-15)


# ------------------------------------------------------------------------------------ contact / CCD

def test_active_set_equals_naive_all_pairs():
    sc, mod, ctx, x, y = _press_state()
    P = M.all_positions(mod, x, y)
    act = C.active_pairs(mod, P)
    dhat2 = sc.config.dhat ** 2
    naive = []
    for v in mod.surf_verts:
        for t in range(len(mod.tris)):
            if mod.allowed[mod.vert_body[v], mod.tri_body[t]]:
                tt = mod.tris[t]
                if D.pt_type(P[v], P[tt[0]], P[tt[1]], P[tt[2]])[1] < dhat2:
                    naive.append((0, v, t))
    E = mod.edges
    for a in range(len(E)):
        for b in range(a + 1, len(E)):
            if mod.allowed[mod.edge_body[a], mod.edge_body[b]]:
                if D.ee_type(P[E[a, 0]], P[E[a, 1]], P[E[b, 0]], P[E[b, 1]])[1] < dhat2:
                    naive.append((1, a, b))
    assert np.array_equal(act.keys(), np.asarray(naive).reshape(-1, 3))


def test_far_cubes_empty_and_filter_rules():
    sc = S.make_scene("C1")
    mod = M.prepare(sc)
    ei = S.env_inputs(sc, [0], 1)
    P = M.all_positions(mod, ei.x0[0], ei.y0[0])      # cube 0.2 mm > d̂ above the pad
    assert len(C.active_pairs(mod, P)) == 0
    # the pad touches its mount (base) at distance 0 but that body pair is excluded
    assert not mod.allowed[0, 1] and mod.allowed[0, 2] and not mod.allowed[1, 2]


def test_accd_closed_forms():
    g = GOLD["accd_normal_approach"]
    tri = np.array([[-1, -1, 0], [2, -1, 0], [-1, 2, 0.0]])
    X = np.vstack([[0, 0, g["d0"]], tri])
    Pd = np.zeros((4, 3))
    Pd[0, 2] = -g["speed"]
    assert C.accd(0, X, Pd) == pytest.approx(g["alpha"], rel=1e-12)
    assert C.accd(0, X, np.zeros((4, 3))) == 1.0
    assert C.accd(0, X, np.tile([0.3, 0.2, 0.1], (4, 1))) == 1.0      # common translation


def test_accd_conservative_audit():
    """100 random trials: returned α ≤ exact TOI (dense bisection) and distance > 0 after the move
    (S:L138)."""
    rng = np.random.default_rng(9)
    for trial in range(100):
        kind = trial % 2
        X = rng.normal(size=(4, 3))
        Pd = rng.normal(size=(4, 3)) * 2.0
        t = C.accd(kind, X, Pd)
        ts = np.linspace(0, 1, 4001)
        d2 = np.array([C._pair_d2(kind, X + s * Pd) for s in ts])
        hit = np.nonzero(d2 < 1e-14)[0]
        toi = ts[hit[0]] if len(hit) else 1.0
        assert t <= toi + 1e-9
        assert C._pair_d2(kind, X + min(t, 1.0) * Pd) > 0


# ------------------------------------------------------------------------------------ solver

def _free_body_scene(gravity=(0, 0, -9.81)):
    V, Tr = S.box_surface((0.01, 0.01, 0.01))
    body = S.AffineBody(V, Tr, kind=S.DYNAMIC)
    sc = S.Scene("C1", [], [body], np.array(gravity, float), S.Config(dt=0.01), n_steps=1)
    return sc, M.prepare(sc)


def test_free_fall_exact_at_scene_scale():
    """Free affine body under gravity: the step's minimiser is t¹ = t⁰ + Δt v⁰ + Δt² g,
    A¹ = A⁰ (a quadratic problem).  L_env is the cube's own scale (bounding-box diagonal), so the
    R17c step cap (0.05·L_env) splits the ≈5 mm move into several capped Newton steps; the converged
    position must still be the closed form."""
    sc, mod = _free_body_scene()
    y0 = np.array([[0.1, 0.2, 0.3, *S.rot_z(0.4).ravel()]])
    yd0 = np.array([[0.5, -0.2, 0.1, *np.zeros(9)]])
    st = SO.State(np.zeros((0, 3)), np.zeros((0, 3)), y0, yd0)
    L = M.env_scale(mod, st.x, st.y)
    w = 0.01 * (math.cos(0.4) + math.sin(0.4))                       # 10 mm cube yawed 0.4 rad: bbox
    assert L == pytest.approx(math.sqrt(2 * w * w + 0.01 ** 2), rel=1e-12)
    new, stats = SO.step(mod, st, np.zeros((0, 12)), L_env=L)
    dt = sc.config.dt
    expect = y0[0, :3] + dt * yd0[0, :3] + dt * dt * sc.gravity
    assert stats.status == SO.ENV_OK
    assert np.allclose(new.y[0, :3], expect, rtol=0, atol=1e-14)
    assert np.allclose(new.y[0, 3:], y0[0, 3:], atol=1e-14)


def test_step_cap_limits_newton_step_length():
    """Reading R17c: a Newton step longer than max_step_rel·L_env (embedded ∞-norm) is scaled to
    exactly that length — the free-fall move (≈5 mm ≫ 0.05·17.3 mm) takes ⌈5 mm / 0.87 mm⌉ capped
    steps, each of length 0.05·L_env, then one full step and the convergence check."""
    sc, mod = _free_body_scene()
    y0 = np.array([[0.1, 0.2, 0.3, *S.rot_z(0.4).ravel()]])
    yd0 = np.array([[0.5, -0.2, 0.1, *np.zeros(9)]])
    st = SO.State(np.zeros((0, 3)), np.zeros((0, 3)), y0, yd0)
    L = M.env_scale(mod, st.x, st.y)
    trace = []
    new, stats = SO.step(mod, st, np.zeros((0, 12)), L_env=L, trace=trace)
    steps = [t for t in trace if "p_inf" in t]
    cap = sc.config.max_step_rel * L
    move = np.abs(sc.config.dt * yd0[0, :3] + sc.config.dt ** 2 * sc.gravity).max()   # translation only
    n_cap = int(math.floor(move / cap))
    assert len(steps) >= n_cap + 1
    for t in steps[:n_cap]:
        assert t["p_inf"] == pytest.approx(cap, rel=1e-12) and t["alpha"] == 1.0
    assert steps[-1]["p_inf"] < cap
    assert stats.newton_iters == len(steps) + 1


def test_fixed_point_without_forces():
    sc, mod = _free_body_scene(gravity=(0, 0, 0))
    y0 = np.array([[0.1, 0.2, 0.3, *np.eye(3).ravel()]])
    st = SO.State(np.zeros((0, 3)), np.zeros((0, 3)), y0, np.zeros_like(y0))
    new, stats = SO.step(mod, st, np.zeros((0, 12)), L_env=0.02)
    assert np.array_equal(new.y, y0) and stats.newton_iters == 1


def test_descent_direction_and_pcg_agrees_with_direct():
    sc, mod, ctx, x, y = _press_state()
    pairs = C.active_pairs(mod, M.all_positions(mod, x, y))
    g, H = En.assemble(mod, ctx, x, y, pairs)
    import scipy.sparse.linalg as spla
    p = spla.spsolve(H.tocsc(), -g)
    assert g @ p < 0
    pp, it = SO.block_jacobi_pcg(mod, H, g, 1e-8, 5000)
    assert it > 1
    assert np.abs(pp - p).max() <= 1e-5 * np.abs(p).max()
    assert g @ pp < 0


def test_al_fixed_vertex_single_tet():
    """A tet with one vertex constrained to a moved target converges within ≤5 AL rounds
    (S:L387)."""
    X, tets = unit_tet()
    X = X * 0.01
    base_V, base_T = S.box_surface((0.05, 0.05, 0.01))
    base = S.AffineBody(base_V, base_T, kind=S.KINEMATIC)
    pad = S.SoftPad(rest_pos=X, tets=tets, mount_body=0, mount_T=S.pose([0, 0, 0.1]),
                    attached=np.array([0], np.int32))
    sc = S.Scene("C1", [pad], [base], np.array([0, 0, -9.81]), S.Config(dt=0.01), n_steps=1)
    mod = M.prepare(sc)
    y0 = np.array([S.pose([0, 0, 0])])
    x0 = X + np.array([0, 0, 0.1])
    st = SO.State(x0, np.zeros_like(x0), y0, np.zeros_like(y0))
    target = S.pose([0.001, -0.0005, 0.0002])
    new, stats = SO.step(mod, st, target[None], L_env=0.1)
    assert stats.status == SO.ENV_OK and stats.al_rounds <= 5
    assert np.linalg.norm(new.x[0] - (np.array([0.001, -0.0005, 0.1002]))) <= sc.config.al_tol_rel * 0.1


# ------------------------------------------------------------------------------------ readout

def test_readout_rigid_motion_and_bary():
    sc = S.make_scene("C1")
    mod = M.prepare(sc)
    ei = S.env_inputs(sc, [0], 1)
    x, y = ei.x0[0].copy(), ei.y0[0].copy()
    # undeformed → zero displacement and flow
    coated, mpos, mflow = R.gel_deformation(mod, x, y)[0]
    assert np.abs(coated).max() < 1e-15 and np.abs(mflow).max() < 1e-15
    # rigid motion of the base (mount) together with the pad → zero flow
    Rz = S.rot_z(0.3)
    y2 = y.copy()
    y2[0] = S.pose([0.01, 0.02, -0.03], Rz)
    x2 = x @ Rz.T + np.array([0.01, 0.02, -0.03])
    coated, mpos, mflow = R.gel_deformation(mod, x2, y2)[0]
    assert np.abs(coated).max() < 1e-15 and np.abs(mflow).max() < 1e-15
    # barycentric weights (1,0,0) → exactly that vertex
    pad = sc.soft[0]
    pad.marker_bary = np.array([[1.0, 0.0, 0.0]])
    pad.marker_tri = pad.marker_tri[:1]
    c, mp, mf = R.gel_deformation(mod, x2, y2)[0]
    assert np.array_equal(mp[0], x2[pad.marker_tri[0, 0]])


def _naive_candidates(mod, P0, P1):
    dhat = mod.scene.config.dhat
    out = []
    sv = mod.surf_verts
    vlo, vhi = np.minimum(P0[sv], P1[sv]), np.maximum(P0[sv], P1[sv])
    T = mod.tris
    tlo = np.minimum(P0[T].min(1), P1[T].min(1)) - dhat
    thi = np.maximum(P0[T].max(1), P1[T].max(1)) + dhat
    for i, v in enumerate(sv):
        for t in range(len(T)):
            if mod.allowed[mod.vert_body[v], mod.tri_body[t]] and np.all(vlo[i] <= thi[t]) and np.all(tlo[t] <= vhi[i]):
                out.append((0, v, t))
    E = mod.edges
    elo, ehi = np.minimum(P0[E].min(1), P1[E].min(1)), np.maximum(P0[E].max(1), P1[E].max(1))
    for a in range(len(E)):
        for b in range(a + 1, len(E)):
            if mod.allowed[mod.edge_body[a], mod.edge_body[b]] and np.all(elo[a] <= ehi[b] + dhat) \
                    and np.all(elo[b] - dhat <= ehi[a]):
                out.append((1, a, b))
    return np.asarray(out).reshape(-1, 3)


@pytest.mark.parametrize("swept", [False, True])
def test_candidates_equal_naive_loops(swept):
    """The body-pruned brute force returns exactly the naive all-pairs AABB set (same predicate)."""
    sc, mod, ctx, x, y = _press_state()
    P = M.all_positions(mod, x, y)
    rng = np.random.default_rng(10)
    P1 = P + (rng.normal(size=P.shape) * 1e-4 if swept else 0.0)
    got = C.candidate_pairs(mod, P, P1)
    assert len(got) > 0
    assert np.array_equal(got, _naive_candidates(mod, P, P1))


# ------------------------------------------------------------------------------------ single pairs

def _pair_state(name):
    sc = S.make_scene(name)
    mod = M.prepare(sc)
    ei = S.env_inputs(sc, [0], n_steps=1)
    x, y = ei.x0[0], ei.y0[0]
    ctx = En.make_context(mod, x, np.zeros_like(x), y, np.zeros_like(y), np.zeros((0, 12)), sc.config.dt)
    return sc, mod, ctx, x, y


def _area(P, tri):
    i, j, k = tri
    return 0.5 * np.linalg.norm(np.cross(P[j] - P[i], P[k] - P[i]))


def _b_half():
    """b(d̂/2) from the golden closed form: (d̂²/4) ln 2."""
    g = GOLD["barrier"]
    return g["b_at_half_over_dhat2"] * g["dhat"] ** 2


def test_single_pt_pair_barrier_value():
    """One point–triangle pair (scene P1: a tet apex d̂/2 above a static box face): the barrier term
    equals Δt²·κ·A_k·b(d) with A_k = A_v(apex) = ⅓ of the rest areas of the apex's three incident
    faces (reading R12, P:L106 Eq. fullspace_ipc weight A_k; S:L213 'a single pair gives κA_k b')."""
    sc, mod, ctx, x, y = _pair_state("P1")
    pairs = C.active_pairs(mod, M.all_positions(mod, x, y))
    assert len(pairs) == 1 and pairs.kind[0] == 0 and pairs.a[0] == 0 and pairs.typ[0] == 0   # interior
    X = sc.soft[0].rest_pos
    A_v = (_area(X, (0, 1, 3)) + _area(X, (0, 1, 2)) + _area(X, (0, 2, 3))) / 3.0
    cfg = sc.config
    expect = cfg.dt ** 2 * cfg.kappa * A_v * _b_half()
    assert En.energy_terms(mod, ctx, x, y, pairs)["barrier"] == pytest.approx(expect, rel=1e-12)


def test_single_ee_pair_barrier_value():
    """One edge–edge pair (scene P2: two edges crossing at right angles at gap d̂/2): barrier =
    Δt²·κ·½(A_e(a)+A_e(b))·b(d), A_e = ⅓ of the two incident rest face areas; the mollifier is 1
    (c = ‖e₁×e₂‖² = 1000·ε×) (reading R12, R7)."""
    sc, mod, ctx, x, y = _pair_state("P2")
    pairs = C.active_pairs(mod, M.all_positions(mod, x, y))
    assert len(pairs) == 1 and pairs.kind[0] == 1
    XA, XB = sc.soft[0].rest_pos, sc.soft[1].rest_pos
    A_ea = (_area(XA, (0, 1, 2)) + _area(XA, (0, 1, 3))) / 3.0     # faces incident to the ridge edge (0,1)
    A_eb = (_area(XB, (0, 1, 2)) + _area(XB, (0, 1, 3))) / 3.0     # faces incident to the valley edge (0,1)
    assert A_ea == pytest.approx(2 * math.sqrt(2) / 3 * 1e-6, rel=1e-12)   # a = 1 mm: √2 a² per face
    cfg = sc.config
    expect = cfg.dt ** 2 * cfg.kappa * 0.5 * (A_ea + A_eb) * _b_half()
    assert En.energy_terms(mod, ctx, x, y, pairs)["barrier"] == pytest.approx(expect, rel=1e-12)


def test_single_ee_pair_mollifier_value():
    """Nearly parallel edges (scene P2m, sin θ = 0.02, unstretched): c/ε× = ‖e₁×e₂‖² /
    (1e-3‖ē₁‖²‖ē₂‖²) = 1000 sin²θ = 0.4, so m = (2 − 0.4)·0.4 = 0.64 multiplies the pair's barrier
    (reading R7: ε× = 1e-3 of the rest squared lengths' product)."""
    sc, mod, ctx, x, y = _pair_state("P2m")
    pairs = C.active_pairs(mod, M.all_positions(mod, x, y))
    assert len(pairs) == 1 and pairs.kind[0] == 1
    assert math.sqrt(pairs.d2[0]) == pytest.approx(0.5 * sc.config.dhat, rel=1e-12)
    XA, XB = sc.soft[0].rest_pos, sc.soft[1].rest_pos
    A_ea = (_area(XA, (0, 1, 2)) + _area(XA, (0, 1, 3))) / 3.0
    A_eb = (_area(XB, (0, 1, 2)) + _area(XB, (0, 1, 3))) / 3.0
    ratio = 1000 * 0.02 ** 2
    m = (2 - ratio) * ratio
    cfg = sc.config
    expect = cfg.dt ** 2 * cfg.kappa * 0.5 * (A_ea + A_eb) * m * _b_half()
    assert En.energy_terms(mod, ctx, x, y, pairs)["barrier"] == pytest.approx(expect, rel=1e-10)


# ------------------------------------------------------------------------------------ whole-step pins

def test_statics_contact_force_equals_weight():
    """Statics: a soft 8 mm cube (C1c, ρ = 1e3) dropped 50 µm onto a static plate
    settles with an upward contact force equal to its weight ρ·(8 mm)³·g within 3%.  The contact
    force is measured independently of the solver: −∂E_barrier/∂z of a rigid vertical translation of
    all cube vertices (central differences of the barrier term), divided by Δt² (E carries Δt²·κ·Σ…)."""
    sc = S.make_scene("C1c")
    mod = M.prepare(sc)
    ei = S.env_inputs(sc, [0], n_steps=1)
    st = SO.State(ei.x0[0].copy(), np.zeros_like(ei.x0[0]), ei.y0[0].copy(), np.zeros_like(ei.y0[0]))
    L = M.env_scale(mod, st.x, st.y)
    for _ in range(6):
        st, stats = SO.step(mod, st, np.zeros((0, 12)), L_env=L)
        assert stats.status == SO.ENV_OK
    ctx = En.make_context(mod, st.x, st.v, st.y, st.ydot, np.zeros((0, 12)), sc.config.dt)

    def e_barrier(dz):
        x = st.x.copy()
        x[:, 2] += dz
        return En.energy_terms(mod, ctx, x, st.y, C.active_pairs(mod, M.all_positions(mod, x, st.y)))["barrier"]

    h = 1e-9
    force_z = -(e_barrier(h) - e_barrier(-h)) / (2 * h) / sc.config.dt ** 2
    weight = 1e3 * (8e-3) ** 3 * 9.81
    assert abs(force_z / weight - 1.0) <= 0.03, force_z / weight


def test_energy_monotone_within_step():
    """Every accepted Newton iterate lowers E (Armijo, S:L391 'monotone energy within a step'), and
    the next iteration starts from the accepted energy (same AL round: λ, ρ fixed)."""
    sc = S.make_scene("C1")
    mod = M.prepare(sc)
    ei = S.env_inputs(sc, [0], n_steps=3)
    st = SO.State(ei.x0[0].copy(), np.zeros_like(ei.x0[0]), ei.y0[0].copy(), np.zeros_like(ei.y0[0]))
    L = M.env_scale(mod, st.x, st.y)
    n_checked = 0
    for k in range(3):
        trace = []
        st, stats = SO.step(mod, st, ei.ykin[k, 0], L_env=L, trace=trace)
        assert stats.status == SO.ENV_OK
        prev = None
        for t in trace:
            if "al_round" in t:
                prev = None
                continue
            assert t["E1"] <= t["E0"]
            if prev is not None:
                assert t["E0"] == pytest.approx(prev, rel=1e-12, abs=1e-18)
            prev = t["E1"]
            n_checked += 1
    assert n_checked >= 3


# ------------------------------------------------------------------------------------ lagged friction

from oracle import friction as Fr


def test_friction_f0_f1_closed_forms():
    """f1 continuous at ε_vΔt (left limit −1 + 2 = 1), f1(0⁺) = 0, f0(0) = ε/3 and
    f0(ε) = ε (the paper's f0(x) = ∫_ε^x f1 + ε at x = 0 and x = ε), and df0/dx = f1 (the written-out
    antiderivative against the paper's f1)."""
    eps = 1e-3 * 0.01
    e = T(np.array([eps]))
    assert float(Fr.f1(e * (1 - 1e-12), eps)) == pytest.approx(1.0, abs=1e-11) and float(Fr.f1(e, eps)) == 1.0
    assert float(Fr.f1(T(np.array([1e-30])), eps)) == pytest.approx(0.0, abs=1e-20)
    assert float(Fr.f0(T(np.array([0.0])), eps)) == pytest.approx(eps / 3, rel=1e-14)
    assert float(Fr.f0(e, eps)) == pytest.approx(eps, rel=1e-14)
    xs = T(np.array([0.1, 0.5, 0.99, 1.5, 3.0]) * eps).requires_grad_(True)
    (d,) = torch.autograd.grad(Fr.f0(xs, eps).sum(), xs)
    assert np.allclose(d.numpy(), Fr.f1(xs.detach(), eps).numpy(), rtol=1e-12, atol=1e-15)


def test_closest_point_weights_give_the_pair_distance():
    """Γ_k X is the separation of the closest points: ‖Γ_k X‖² equals the classified squared distance
    for PT and EE pairs of every type (random configurations)."""
    rng = np.random.default_rng(5)
    seen_pt, seen_ee = set(), set()
    for _ in range(3000):
        X = rng.normal(size=(4, 3))
        for kind in (0, 1):
            if kind == 0:
                typ, d2 = D.pt_type(X[0], X[1], X[2], X[3])
                seen_pt.add(int(typ))
            else:
                typ, d2 = D.ee_type(X[0], X[1], X[2], X[3])
                seen_ee.add(int(typ))
            g = Fr.closest_weights(kind, int(typ), X)
            sep = g @ X
            assert abs(sep @ sep - float(d2)) <= 1e-10 * float(d2), (kind, typ)
            assert abs(g.sum()) < 1e-12                       # a difference of two points
    assert seen_pt == set(range(7)) and {0, 1, 2, 3, 4, 5, 6, 7, 8} >= seen_ee >= {1, 3, 4, 5, 7}


def _fric_pair_state(mu=0.5):
    import dataclasses
    sc = S.make_scene("P1")
    sc.config = dataclasses.replace(sc.config, mu_friction=mu)
    mod = M.prepare(sc)
    ei = S.env_inputs(sc, [0], n_steps=1)
    return sc, mod, ei.x0[0], ei.y0[0]


def test_friction_lagged_force_and_plateau():
    """Single PT pair (scene P1, apex d̂/2 above a static face): λⁿ = κ A_v |b′(d̂/2)| with b′(d̂/2) from
    the golden closed form; sliding the apex tangentially by 2ε_vΔt, the friction force has
    magnitude μλⁿ exactly (dynamic plateau) and opposes the slide; with no slide it is 0."""
    sc, mod, x, y = _fric_pair_state(0.5)
    cfg = sc.config
    ctx = En.make_context(mod, x, np.zeros_like(x), y, np.zeros_like(y), np.zeros((0, 12)), cfg.dt)
    fr = ctx.fric
    assert len(fr) == 1
    X = sc.soft[0].rest_pos
    A_v = (_area(X, (0, 1, 3)) + _area(X, (0, 1, 2)) + _area(X, (0, 2, 3))) / 3.0
    lam = cfg.kappa * A_v * abs(GOLD["barrier"]["db_at_half_over_dhat"] * cfg.dhat)
    assert fr.mu_lam[0] == pytest.approx(0.5 * lam, rel=1e-12)
    assert np.allclose(np.abs(fr.nhat[0]), [0, 0, 1], atol=1e-12)
    eps = cfg.eps_v * cfg.dt
    for slide, expect in ((0.0, 0.0), (2 * eps, 0.5 * lam)):
        xs = x.copy()
        xs[0] += slide * np.array([0.6, 0.8, 0.0])            # apex only, in the tangent plane
        pairs = C.active_pairs(mod, M.all_positions(mod, xs, y))
        g, _ = En.assemble(mod, ctx, xs, y, pairs, project=False)
        ctx0 = dataclasses_replace(ctx, fric=None)
        g0, _ = En.assemble(mod, ctx0, xs, y, pairs, project=False)
        f = -(g - g0)[:3] / cfg.dt ** 2                       # friction force on the apex (E carries Δt²·D)
        assert np.linalg.norm(f) == pytest.approx(expect, rel=1e-12, abs=1e-30)
        if slide:
            assert f @ np.array([0.6, 0.8, 0.0]) < 0


def dataclasses_replace(obj, **kw):
    import dataclasses
    return dataclasses.replace(obj, **kw)


def test_friction_gradient_and_hvp_vs_finite_differences():
    """Total energy with friction (C1 press, μ = 0.5, lagged at xⁿ, iterate slid away from xⁿ):
    gradient and exact-Hessian HVP against central differences."""
    import dataclasses
    sc, mod, ctx, x, y = _press_state()
    sc.config = dataclasses.replace(sc.config, mu_friction=0.5)
    mod = M.prepare(sc)
    ei = S.env_inputs(sc, [0], n_steps=1)
    yn = ei.y0[0].copy()
    yn[1, 2] -= 0.2e-3 - 0.04e-3
    ctx = En.make_context(mod, ei.x0[0], np.zeros_like(ei.x0[0]), yn, np.zeros_like(yn), ei.ykin[0, 0], sc.config.dt)
    assert len(ctx.fric) > 10
    rng = np.random.default_rng(3)
    x = ei.x0[0] + rng.normal(size=ei.x0[0].shape) * 3e-6
    y = yn.copy()
    pairs = C.active_pairs(mod, M.all_positions(mod, x, y))
    g, H = En.assemble(mod, ctx, x, y, pairs, project=False)
    q = En.pack(mod, x, y)

    def E(qq):
        xx, yy = En.unpack(mod, qq, y)
        return En.energy_terms(mod, ctx, xx, yy, C.active_pairs(mod, M.all_positions(mod, xx, yy)))["friction"]

    gf, _ = En.assemble(mod, dataclasses.replace(ctx, fric=None), x, y, pairs, project=False)
    gfr = g - gf
    idx = rng.choice(3 * mod.V, 12, replace=False)
    h = 1e-9
    for i in idx:
        e = np.zeros_like(q)
        e[i] = h
        fd = (E(q + e) - E(q - e)) / (2 * h)
        assert fd == pytest.approx(gfr[i], rel=1e-5, abs=1e-6 * np.abs(gfr).max())


def _incline(mu, tan_theta):
    import dataclasses
    th = math.atan(tan_theta)
    pV, pT = S.box_surface((0.04, 0.04, 0.01))
    cV, cT = S.box_surface((0.01, 0.01, 0.01))
    plate = S.AffineBody(pV, pT, kind=S.STATIC)
    cube = S.AffineBody(cV, cT, kind=S.DYNAMIC)
    g = 9.81 * np.array([math.sin(th), 0.0, -math.cos(th)])      # plane inclined by θ about y
    cfg = dataclasses.replace(S.Config(dt=0.01), mu_friction=mu, eps_v=1e-3)
    sc = S.Scene("C1", [], [plate, cube], g, cfg, n_steps=1)
    y0 = np.array([S.pose([0, 0, -0.005]), S.pose([0.0013, 0.0007, 0.005 + 0.5e-4], S.rot_z(0.3))])
    return sc, M.prepare(sc), y0


@pytest.mark.parametrize("mu", [0.2, 0.5])
def test_friction_incline_stick_and_slip(mu):
    """A stiff cube on a plane inclined by θ (gravity tilted): with tan θ = 0.9μ it sticks (per-step
    slide < 10·ε_vΔt after settling), with tan θ = 1.1μ it slides with growing per-step displacement
    (Coulomb threshold tan θ = μ)."""
    out = {}
    for label, t in (("stick", 0.9 * mu), ("slip", 1.1 * mu)):
        sc, mod, y0 = _incline(mu, t)
        st = SO.State(np.zeros((0, 3)), np.zeros((0, 3)), y0.copy(), np.zeros_like(y0))
        L = M.env_scale(mod, st.x, st.y)
        xs = []
        for k in range(12):
            st, stats = SO.step(mod, st, np.zeros((0, 12)), L_env=L)
            assert stats.status == SO.ENV_OK, (label, k)
            xs.append(st.y[1, 0])
        out[label] = np.diff(np.array(xs))
    eps_dt = 1e-3 * 0.01
    assert np.all(np.abs(out["stick"][4:]) < 10 * eps_dt), out["stick"]
    assert np.all(out["slip"][4:] > 0) and np.all(np.diff(out["slip"][4:]) > 0), out["slip"]


# ------------------------------------------------------------------------------------ forward kinematics

from oracle import kinematics as K


def test_fk_planar_three_link_closed_form():
    """3-joint planar arm: joint axes z, link lengths along x; the tip is at
    Σ_i L_i (cos Σ_{j≤i} θ_j, sin Σ_{j≤i} θ_j) and its frame is rotated by Σθ — closed form to 1e-12."""
    L = [0.3, 0.2, 0.1]
    th = [0.4, -1.1, 0.7]
    ident = np.r_[np.zeros(3), np.eye(3).ravel()]
    chain = {"parent": [-1, 0, 1, 2], "joint": [0, 1, 2, -1], "axis": [[0, 0, 1]] * 4,
             "origin": [ident, np.r_[L[0], 0, 0, np.eye(3).ravel()], np.r_[L[1], 0, 0, np.eye(3).ravel()],
                        np.r_[L[2], 0, 0, np.eye(3).ravel()]],
             "body": [ident] * 4}
    out = K.forward(chain, ident, np.array(th))
    c = np.cumsum(th)
    tip = np.array([sum(L[i] * math.cos(c[i]) for i in range(3)), sum(L[i] * math.sin(c[i]) for i in range(3)), 0.0])
    assert np.allclose(out[3, :3], tip, atol=1e-12)
    assert np.allclose(out[3, 3:].reshape(3, 3), S.rot_z(c[-1]), atol=1e-12)


def test_fk_hand_chain_matches_scene_generator():
    """The C5 chain description (input to tac_set_chain) reproduces the scene generator's link targets
    (12-vector compositions) through the oracle's 4×4 homogeneous products, to 1e-12."""
    ch = S.hand_chain()
    qs = S.hand_script(3, 120)
    yp = S.hand_palm_pose()
    for k in (0, 40, 79, 119):
        ref = S.fk_hand(yp, qs[k])
        q = qs[k].reshape(-1)
        out = K.forward(ch, yp, q)
        assert np.abs(out[1:] - ref).max() <= 1e-12
        assert np.abs(out[0] - yp).max() <= 1e-15


# ------------------------------------------------------------------------------------ depth maps

from oracle import tactile as Tc


def _c1_pad_state():
    sc = S.make_scene("C1")
    mod = M.prepare(sc)
    ei = S.env_inputs(sc, [0], n_steps=1)
    return sc, mod, ei.x0[0].copy(), ei.y0[0].copy()


def test_depth_map_undeformed_and_rigid_motion():
    """Undeformed pad → depth 0 and normal +z at every pixel (S:L532 'zero depth without contact');
    moving the pad rigidly with its mount link leaves the maps unchanged (sensor frame)."""
    sc, mod, x, y = _c1_pad_state()
    D0, N0 = Tc.depth_maps(mod, x, y, 9, 11)
    assert np.all(np.abs(D0) <= 1e-15) and np.allclose(N0, [0, 0, 1], atol=1e-15)
    R = S.rot_z(0.7) @ S.rot_y(0.2)
    t = np.array([0.01, -0.02, 0.03])
    y2 = y.copy()
    y2[0] = np.r_[t + R @ y[0, :3], (R @ y[0, 3:].reshape(3, 3)).ravel()]
    x2 = x @ R.T + t
    D1, N1 = Tc.depth_maps(mod, x2, y2, 9, 11)
    assert np.all(np.abs(D1) <= 1e-12) and np.allclose(N1, [0, 0, 1], atol=1e-12)


def test_depth_map_sphere_cap_closed_form():
    """A sphere of radius R pressed h into the coated face (constructed state: every coated vertex
    lowered to the cap): pixels on lattice vertices read the analytic cap depth
    d(r) = h − (R − √(R² − r²)) and pixels on lattice edges the average of the edge's vertex depths
    (the surface is piecewise linear), to 1e-12; flat regions keep normal +z."""
    sc, mod, x, y = _c1_pad_state()
    pad = sc.soft[0]
    Rs, h = 10e-3, 0.6e-3
    off = 0
    cap = lambda r: np.maximum(0.0, h - (Rs - np.sqrt(np.maximum(Rs * Rs - r * r, 0.0))))
    xs = x.copy()
    X = pad.rest_pos
    for v in pad.coated:
        xs[off + v, 2] -= cap(np.hypot(X[v, 0], X[v, 1]))
    H = W = 15                                           # 8x8 vertex lattice → vertices at even pixels
    D, N = Tc.depth_maps(mod, xs, y, H, W)
    xv = np.linspace(X[pad.coated, 0].min(), X[pad.coated, 0].max(), W)
    yv = np.linspace(X[pad.coated, 1].min(), X[pad.coated, 1].max(), H)
    for i in range(0, H, 2):
        for j in range(0, W, 2):
            assert D[0, i, j] == pytest.approx(cap(np.hypot(xv[j], yv[i])), abs=1e-12)
    for i in range(0, H, 2):                             # midpoints of lattice edges along x
        for j in range(1, W, 2):
            expect = 0.5 * (cap(np.hypot(xv[j - 1], yv[i])) + cap(np.hypot(xv[j + 1], yv[i])))
            assert D[0, i, j] == pytest.approx(expect, abs=1e-12)
    assert np.allclose(N[0, 0, 0], [0, 0, 1], atol=1e-12)
    assert np.nanmax(D) <= h                              # the interpolant never exceeds the cap depth


def test_relaxed_pcg_tolerance_reaches_the_same_step():
    """Reading R24 ("carefully relaxing convergence tolerances"): the Eisenstat–Walker forcing only
    changes how accurately each Newton direction is solved, not the minimiser — a C1 press step with the PCG
    solver at η ∈ [1e-4, 0.1] lands on the direct-solve step within 1e-7·L_env (the Newton tolerance), the
    forcing is live (a different PCG iteration count from the fixed η), and the first solve of a step uses
    η_max."""
    import dataclasses
    sc0 = S.make_scene("C1")
    ei = S.env_inputs(sc0, [0], n_steps=3)
    out = {}
    for key, (solver, em) in {"direct": ("direct", 0.0), "fixed": ("pcg", 0.0), "relaxed": ("pcg", 0.1)}.items():
        sc = S.make_scene("C1")
        sc.config = dataclasses.replace(sc.config, pcg_eta_max=em)
        mod = M.prepare(sc)
        L = M.env_scale(mod, ei.x0[0], ei.y0[0])
        st = SO.State(ei.x0[0].copy(), np.zeros_like(ei.x0[0]), ei.y0[0].copy(), np.zeros_like(ei.y0[0]))
        pcg = 0
        for k in range(3):
            st, stats = SO.step(mod, st, ei.ykin[k, 0], solver=solver, L_env=L)
            assert stats.status == SO.ENV_OK
            pcg += stats.pcg_iters
        out[key] = (M.all_positions(mod, st.x, st.y), pcg, L)
    P0, _, L = out["direct"]
    for key in ("fixed", "relaxed"):
        assert np.abs(out[key][0] - P0).max() <= 1e-7 * L, key
    assert out["relaxed"][1] != out["fixed"][1], (out["relaxed"][1], out["fixed"][1])
    assert SO.forcing_eta(dataclasses.replace(sc0.config, pcg_eta_max=0.1), 1.0, None) == 0.1
