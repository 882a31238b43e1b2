"""Oracle energies, gradients and projected Hessians (test infrastructure only — see oracle/__init__.py).

The per-env objective (assembled from P:L92 Eq. IP, P:L102 Eq. fullspace_ipc,
P:L121-122 Eq. unified_ipc, P:L137 Eq. unified_ipc_AL with reading R13):

  E(x,y) = ½‖x−x̃‖²_M + Σ_b ½‖y_b−ỹ_b‖²_{M^y_b}
         + Δt²·[ Σ_e V_e Ψ(F_e) + Σ_b κ_s V_b ‖A_bA_bᵀ−I‖²_F − Σ_v m_v gᵀx_v − Σ_b gᵀ(m_b t_b + A_b s₁_b)
                 + κ Σ_{k∈𝒜} A_k m_k b(d_k) ]
         + E_AL,   E_AL = Σ_c (ρ/2) r_cᵀW_c r_c − λ_cᵀW_c r_c

Every term is written once as a plain energy of its element's local coordinates; gradients and
Hessians come from automatic differentiation (torch.func.grad / torch.func.hessian) of that
definition, and PSD projections from numpy.linalg.eigh with eigenvalues clamped to 0 (the
per-element clamp of S:L242; Neo-Hookean projected in F-space, barrier on the full 12×12,
orthogonality on the 9×9 A-block: readings R4, R12, R6 in DESIGN.md).
"""
from __future__ import annotations

import dataclasses

import numpy as np
import scipy.sparse as sp
import torch
from torch.func import grad, hessian, jacrev, vmap

from . import distance as D
from .mesh import Model, affine_jacobian

torch.set_default_dtype(torch.float64)

TERMS = ("inertia", "elastic", "ortho", "gravity", "barrier", "al", "friction")


# ---------------------------------------------------------------------------------------------
# scalar definitions
# ---------------------------------------------------------------------------------------------

def barrier(d, dhat):
    """b(d) = −(d−d̂)² log(d/d̂) on (0, d̂), 0 otherwise (Eq. ipc_energy)."""
    inside = (d < dhat)
    dd = torch.where(inside, d, torch.as_tensor(dhat, dtype=d.dtype) * 0.5)
    return torch.where(inside, -(dd - dhat) ** 2 * torch.log(dd / dhat), torch.zeros_like(d))


def det3(F):
    """Determinant of a 3×3 matrix by cofactor expansion along the first row."""
    return (F[0, 0] * (F[1, 1] * F[2, 2] - F[1, 2] * F[2, 1])
            - F[0, 1] * (F[1, 0] * F[2, 2] - F[1, 2] * F[2, 0])
            + F[0, 2] * (F[1, 0] * F[2, 1] - F[1, 1] * F[2, 0]))


def neo_hookean_psi(F, mu, lam):
    """Ψ(F) = μ/2 (tr FᵀF − 3) − μ ln J + λ/2 (ln J)², J = det F (reading R3 of P:L86/P:L358)."""
    J = det3(F)
    lnJ = torch.log(J)
    return 0.5 * mu * ((F * F).sum() - 3.0) - mu * lnJ + 0.5 * lam * lnJ * lnJ


def deformation_gradient(x4, Dm_inv):
    """F = D_s D_m⁻¹ with D_s = [x1−x0, x2−x0, x3−x0] (columns)."""
    Ds = torch.stack([x4[1] - x4[0], x4[2] - x4[0], x4[3] - x4[0]], 1)
    return Ds @ Dm_inv


def ortho_energy(A, kappa_s, vol):
    """κ_s V_b ‖AAᵀ − I‖²_F (reading R9/R6 of the garbled 'ARAP' term)."""
    G = A @ A.T - torch.eye(3, dtype=A.dtype)
    return kappa_s * vol * (G * G).sum()


def ee_mollifier(c, eps):
    """m(c) = (2 − c/ε×)(c/ε×) for c < ε×, else 1 (IPC convention; reading R7)."""
    r = c / eps
    return torch.where(c < eps, (2.0 - r) * r, torch.ones_like(c))


# ---------------------------------------------------------------------------------------------
# per-env context
# ---------------------------------------------------------------------------------------------

@dataclasses.dataclass
class Context:
    """Per-step constants of one env: x̃, ỹ, static poses, targets, AL multipliers and ρ."""
    x_tilde: np.ndarray       # (V,3)
    y_tilde: np.ndarray       # (NA,12) (static rows unused)
    y_static: np.ndarray      # (NA,12) poses used for static bodies
    s_att: np.ndarray         # (NC,3) targets of ∂⁻G vertices
    s_kin: np.ndarray         # (NK,12) targets of kinematic bodies
    lam_att: np.ndarray       # (NC,3)
    lam_kin: np.ndarray       # (NK,12)
    rho: float
    fric: object = None       # oracle.friction.FrictionData (lagged at xⁿ) when μ > 0


def attached_targets(model: Model, y_pose: np.ndarray) -> np.ndarray:
    """s^x for ∂⁻G: the mount link's affine target applied to the vertex's link-frame rest
    position ('node position targets for gel pad attached surfaces')."""
    out = np.zeros((len(model.att_vert), 3))
    for i, (b, xl) in enumerate(zip(model.att_body, model.att_local)):
        out[i] = y_pose[b, :3] + y_pose[b, 3:].reshape(3, 3) @ xl
    return out


def make_context(model: Model, x_n, v_n, y_n, ydot_n, y_targets_kin, dt, lam_att=None, lam_kin=None, rho=None):
    """x̃ = xⁿ + Δt ẋⁿ, ỹ = yⁿ + Δt ẏⁿ; s^y from the kinematic targets; s^x derived from
    the mount links' targets (static mounts use their current pose)."""
    cfg = model.scene.config
    y_pose = np.array(y_n, np.float64, copy=True)
    for i, b in enumerate(model.kin_bodies):
        y_pose[b] = y_targets_kin[i]
    fric = None
    if getattr(cfg, "mu_friction", 0.0) > 0.0:
        from . import friction as Fr
        fric = Fr.lagged(model, x_n, y_n)
    return Context(x_tilde=x_n + dt * v_n, y_tilde=y_n + dt * ydot_n, y_static=np.array(y_n, copy=True),
                   s_att=attached_targets(model, y_pose),
                   s_kin=np.array(y_targets_kin, np.float64).reshape(-1, 12),
                   lam_att=np.zeros((len(model.att_vert), 3)) if lam_att is None else lam_att,
                   lam_kin=np.zeros((len(model.kin_bodies), 12)) if lam_kin is None else lam_kin,
                   rho=cfg.al_rho0 if rho is None else rho, fric=fric)


# ---------------------------------------------------------------------------------------------
# element energies (torch, local coordinates)
# ---------------------------------------------------------------------------------------------

def _vertex_energy(x, m, xt, g, dt2, s, lam, c, rho):
    """½ m‖x − x̃‖² − Δt² m gᵀx + c·[(ρ/2) m‖x − s‖² − m λᵀ(x − s)] for one soft vertex."""
    r = x - s
    return (0.5 * m * ((x - xt) ** 2).sum() - dt2 * m * (g * x).sum()
            + c * (0.5 * rho * m * (r * r).sum() - m * (lam * r).sum()))


def _tet_energy(x12, Dm_inv, vol, mu, lam, dt2):
    F = deformation_gradient(x12.reshape(4, 3), Dm_inv)
    return dt2 * vol * neo_hookean_psi(F, mu, lam)


def _body_energy_quadratic(y, M, yt, g, m, s1, dt2, s, lam, c, rho):
    """Inertia ½(y−ỹ)ᵀM^y(y−ỹ), gravity −Δt² gᵀ(m t + A s₁), AL c·[(ρ/2) rᵀM^y r − λᵀM^y r]."""
    d = y - yt
    A = y[3:].reshape(3, 3)
    r = y - s
    return (0.5 * d @ (M @ d) - dt2 * (g * (m * y[:3] + A @ s1)).sum()
            + c * (0.5 * rho * r @ (M @ r) - lam @ (M @ r)))


def _body_ortho(y, kappa, vol, dt2):
    return dt2 * ortho_energy(y[3:].reshape(3, 3), kappa, vol)


def _pair_energy_factory(kind, typ, dhat, kappa, dt2, mollify):
    """E_k(X) = Δt² κ A_k m_k b(√s_type(X)) for a fixed kind/type."""
    def f(X12, A_k, eps):
        P = X12.reshape(4, 3)
        if kind == 0:
            s = D.pt_d2_single(torch, typ, P[0], P[1], P[2], P[3])
            m = torch.ones((), dtype=X12.dtype)
        else:
            s = D.ee_d2_single(torch, typ, P[0], P[1], P[2], P[3])
            if mollify:
                n = D._cross(torch, P[1] - P[0], P[3] - P[2])
                m = ee_mollifier((n * n).sum(), eps)
            else:
                m = torch.ones((), dtype=X12.dtype)
        return dt2 * kappa * A_k * m * barrier(torch.sqrt(s), dhat)
    return f


def psd_project(H):
    """Clamp negative eigenvalues to 0 (numpy.linalg.eigh), batched over leading dims."""
    w, Q = np.linalg.eigh(H)
    w = np.maximum(w, 0.0)
    return np.einsum("...ij,...j,...kj->...ik", Q, w, Q)


# ---------------------------------------------------------------------------------------------
# active-pair data
# ---------------------------------------------------------------------------------------------

@dataclasses.dataclass
class Pairs:
    kind: np.ndarray    # 0 PT, 1 EE
    a: np.ndarray       # PT: vertex id; EE: edge id (a < b)
    b: np.ndarray       # PT: triangle id; EE: edge id
    typ: np.ndarray
    d2: np.ndarray

    def __len__(self):
        return len(self.kind)

    def keys(self):
        return np.stack([self.kind, self.a, self.b], 1) if len(self.kind) else np.zeros((0, 3), np.int64)


def pair_vertices(model: Model, kind, a, b):
    """The 4 global vertex ids of a pair: PT (p, t0, t1, t2), EE (a0, a1, b0, b1)."""
    if kind == 0:
        t = model.tris[b]
        return np.array([a, t[0], t[1], t[2]], np.int64)
    return np.array([model.edges[a, 0], model.edges[a, 1], model.edges[b, 0], model.edges[b, 1]], np.int64)


def pair_area(model: Model, kind, a, b):
    """A_PT = A_v(point); A_EE = ½(A_e(a) + A_e(b)) (reading R12 of the undefined A_k)."""
    if kind == 0:
        return model.A_v[a]
    return 0.5 * (model.A_e[a] + model.A_e[b])


def pair_eps(model: Model, kind, a, b):
    if kind == 0:
        return 1.0
    return 1e-3 * model.edge_rest_len2[a] * model.edge_rest_len2[b]


# ---------------------------------------------------------------------------------------------
# energies and assembly
# ---------------------------------------------------------------------------------------------

def _T(a):
    return torch.as_tensor(np.asarray(a, np.float64))


def energy_terms(model: Model, ctx: Context, x, y, pairs: Pairs):
    """The six terms of E at (x, y) as floats (elastic = +inf if any det F ≤ 0)."""
    cfg = model.scene.config
    dt2 = cfg.dt ** 2
    g = _T(model.scene.gravity)
    out = dict.fromkeys(TERMS, 0.0)
    # soft vertices
    xt, X = _T(ctx.x_tilde), _T(x)
    m = _T(model.mass)[:, None]
    out["inertia"] += float((0.5 * m * (X - xt) ** 2).sum())
    out["gravity"] += float(-dt2 * (m * (g * X)).sum())
    if len(model.att_vert):
        r = X[model.att_vert] - _T(ctx.s_att)
        ma = m[model.att_vert]
        out["al"] += float((0.5 * ctx.rho * ma * r * r).sum() - (ma * _T(ctx.lam_att) * r).sum())
    # tets
    if len(model.tets):
        x12 = X[model.tets].reshape(-1, 12)
        F = vmap(deformation_gradient)(x12.reshape(-1, 4, 3), _T(model.Dm_inv))
        J = vmap(det3)(F)
        if bool((J <= 0).any()):
            out["elastic"] = float("inf")
        else:
            e = vmap(_tet_energy, in_dims=(0, 0, 0, 0, 0, None))(
                x12, _T(model.Dm_inv), _T(model.vol), _T(model.mu), _T(model.lam), dt2)
            out["elastic"] = float(e.sum())
    # bodies
    kin_index = {int(b): i for i, b in enumerate(model.kin_bodies)}
    for bi in range(len(model.body_xbar)):
        if model.dof_slot[bi] < 0:
            continue
        yb = _T(y[bi])
        M = _T(model.body_My[bi])
        d = yb - _T(ctx.y_tilde[bi])
        out["inertia"] += float(0.5 * d @ (M @ d))
        A = yb[3:].reshape(3, 3)
        out["gravity"] += float(-dt2 * (g * (model.body_mass[bi] * yb[:3] + A @ _T(model.body_s1[bi]))).sum())
        out["ortho"] += float(_body_ortho(yb, model.body_kappa[bi], model.body_vol[bi], dt2))
        if bi in kin_index:
            k = kin_index[bi]
            r = yb - _T(ctx.s_kin[k])
            out["al"] += float(0.5 * ctx.rho * r @ (M @ r) - _T(ctx.lam_kin[k]) @ (M @ r))
    # barrier
    out["barrier"] = float(sum(_pair_values(model, x, y, pairs)))
    # lagged friction Δt² Σ_k D_k (oracle/friction.py)
    out["friction"] = float(sum(_friction_values(model, ctx, x, y)))
    return out


def _friction_values(model, ctx, x, y):
    fr = ctx.fric
    if fr is None or len(fr) == 0:
        return []
    from . import friction as Fr
    from .mesh import all_positions
    P = all_positions(model, x, y)
    dt2 = model.scene.config.dt ** 2
    out = []
    for k in range(len(fr)):
        X = P[fr.vids[k]]
        rest = Fr.tangential_sq(X, fr.Xn[k], fr.gamma[k], fr.nhat[k]) == 0.0
        out.append(dt2 * float(Fr.pair_energy(_T(X.ravel()), _T(fr.Xn[k].ravel()), _T(fr.gamma[k]), _T(fr.nhat[k]),
                                              float(fr.mu_lam[k]), fr.eps, rest)))
    return out


def total_energy(model, ctx, x, y, pairs):
    return float(sum(energy_terms(model, ctx, x, y, pairs).values()))


def _positions_of(model, x, y, vids):
    from .mesh import all_positions
    P = all_positions(model, x, y)
    return P[vids]


def _pair_groups(model, x, y, pairs: Pairs):
    """Group active pairs by (kind, type) with their stacked local coordinates."""
    from .mesh import all_positions
    P = all_positions(model, x, y)
    groups = {}
    for k in range(len(pairs)):
        key = (int(pairs.kind[k]), int(pairs.typ[k]))
        groups.setdefault(key, []).append(k)
    out = []
    for (kind, typ), ks in groups.items():
        vids = np.stack([pair_vertices(model, kind, pairs.a[k], pairs.b[k]) for k in ks])
        X = P[vids].reshape(len(ks), 12)
        Ak = np.array([pair_area(model, kind, pairs.a[k], pairs.b[k]) for k in ks])
        eps = np.array([pair_eps(model, kind, pairs.a[k], pairs.b[k]) for k in ks])
        out.append((kind, typ, np.asarray(ks), vids, X, Ak, eps))
    return out


def _pair_values(model, x, y, pairs):
    cfg = model.scene.config
    vals = []
    for kind, typ, ks, vids, X, Ak, eps in _pair_groups(model, x, y, pairs):
        f = _pair_energy_factory(kind, typ, cfg.dhat, cfg.kappa, cfg.dt ** 2, cfg.ee_mollifier)
        vals += list(vmap(f)(_T(X), _T(Ak), _T(eps)).numpy())
    return vals


def vertex_dof_map(model: Model, vid):
    """(dof indices, 3×k matrix) mapping a vertex displacement to DoFs: identity for soft
    vertices, J_v for non-static affine bodies, nothing for static bodies."""
    if vid < model.V:
        return np.arange(3 * vid, 3 * vid + 3), np.eye(3)
    b = model.vert_aff[vid]
    slot = model.dof_slot[b]
    if slot < 0:
        return np.zeros(0, np.int64), np.zeros((3, 0))
    base = 3 * model.V + 12 * slot
    return np.arange(base, base + 12), affine_jacobian(model.vert_xbar[vid])


def assemble(model: Model, ctx: Context, x, y, pairs: Pairs, project=True):
    """Gradient g and (projected) Hessian H (scipy CSR) of E over the DoFs q = [x; y_dof]."""
    cfg = model.scene.config
    dt2 = cfg.dt ** 2
    n = model.n_dof
    g = np.zeros(n)
    rows, cols, vals = [], [], []

    def add_block(idx_r, idx_c, B):
        if len(idx_r) == 0 or len(idx_c) == 0:
            return
        R, C = np.meshgrid(idx_r, idx_c, indexing="ij")
        rows.append(R.ravel()); cols.append(C.ravel()); vals.append(np.asarray(B).ravel())

    grav = _T(model.scene.gravity)
    # soft vertices: inertia + gravity + AL
    V = model.V
    c = np.zeros(V); s = np.zeros((V, 3)); lam = np.zeros((V, 3))
    c[model.att_vert] = 1.0
    s[model.att_vert] = ctx.s_att
    lam[model.att_vert] = ctx.lam_att
    if V:
        args = (_T(x), _T(model.mass), _T(ctx.x_tilde))
        gv = vmap(grad(_vertex_energy), in_dims=(0, 0, 0, None, None, 0, 0, 0, None))(
            *args, grav, dt2, _T(s), _T(lam), _T(c), ctx.rho).numpy()
        Hv = vmap(hessian(_vertex_energy), in_dims=(0, 0, 0, None, None, 0, 0, 0, None))(
            *args, grav, dt2, _T(s), _T(lam), _T(c), ctx.rho).numpy()
        g[:3 * V] += gv.ravel()
        for v in range(V):
            add_block(np.arange(3 * v, 3 * v + 3), np.arange(3 * v, 3 * v + 3), Hv[v])
    # tets: gradient by autograd, Hessian = Δt² V_e Bᵀ Π(∂²Ψ/∂F²) B with B = ∂vec F/∂x
    if len(model.tets):
        x12 = _T(x)[model.tets].reshape(-1, 12)
        Dmi = _T(model.Dm_inv)
        gt = vmap(grad(_tet_energy), in_dims=(0, 0, 0, 0, 0, None))(
            x12, Dmi, _T(model.vol), _T(model.mu), _T(model.lam), dt2).numpy()
        F = vmap(deformation_gradient)(x12.reshape(-1, 4, 3), Dmi)
        HF = vmap(hessian(neo_hookean_psi))(F, _T(model.mu), _T(model.lam)).reshape(-1, 9, 9).numpy()
        B = vmap(jacrev(lambda z, Dm: deformation_gradient(z.reshape(4, 3), Dm).reshape(9)))(x12, Dmi).numpy()
        if project:
            HF = psd_project(HF)
        Ht = dt2 * model.vol[:, None, None] * np.einsum("tai,tab,tbj->tij", B, HF, B)
        for e, tet in enumerate(model.tets):
            idx = (3 * tet[:, None] + np.arange(3)[None, :]).ravel()
            np.add.at(g, idx, gt[e])
            add_block(idx, idx, Ht[e])
    # affine bodies
    kin_index = {int(b): i for i, b in enumerate(model.kin_bodies)}
    for bi in range(len(model.body_xbar)):
        slot = model.dof_slot[bi]
        if slot < 0:
            continue
        idx = np.arange(3 * V + 12 * slot, 3 * V + 12 * slot + 12)
        yb = _T(y[bi])
        ck = 1.0 if bi in kin_index else 0.0
        sk = _T(ctx.s_kin[kin_index[bi]]) if ck else _T(np.zeros(12))
        lk = _T(ctx.lam_kin[kin_index[bi]]) if ck else _T(np.zeros(12))
        qargs = (yb, _T(model.body_My[bi]), _T(ctx.y_tilde[bi]), grav, float(model.body_mass[bi]),
                 _T(model.body_s1[bi]), dt2, sk, lk, ck, ctx.rho)
        gb = grad(_body_energy_quadratic)(*qargs).numpy()
        Hb = hessian(_body_energy_quadratic)(*qargs).numpy()
        oargs = (yb, float(model.body_kappa[bi]), float(model.body_vol[bi]), dt2)
        gb = gb + grad(_body_ortho)(*oargs).numpy()
        Ho = hessian(_body_ortho)(*oargs).numpy()
        if project:
            Ho[3:, 3:] = psd_project(Ho[3:, 3:])
        g[idx] += gb
        add_block(idx, idx, Hb + Ho)
    # barrier pairs: 12×12 in vertex coordinates, projected, pulled back through I₃ / J_v
    for kind, typ, ks, vids, X, Ak, eps in _pair_groups(model, x, y, pairs):
        f = _pair_energy_factory(kind, typ, cfg.dhat, cfg.kappa, dt2, cfg.ee_mollifier)
        gp = vmap(grad(f))(_T(X), _T(Ak), _T(eps)).numpy()
        Hp = vmap(hessian(f))(_T(X), _T(Ak), _T(eps)).numpy()
        if project:
            Hp = psd_project(Hp)
        for j in range(len(ks)):
            maps = [vertex_dof_map(model, v) for v in vids[j]]
            for si, (ri, Ji) in enumerate(maps):
                if len(ri) == 0:
                    continue
                g[ri] += Ji.T @ gp[j, 3 * si:3 * si + 3]
                for sj, (rj, Jj) in enumerate(maps):
                    if len(rj) == 0:
                        continue
                    add_block(ri, rj, Ji.T @ Hp[j, 3 * si:3 * si + 3, 3 * sj:3 * sj + 3] @ Jj)
    # lagged friction pairs: gradient and Hessian of Δt²·D_k by autograd on the 12 slot positions (the
    # Hessian of μλ f0(‖u‖) is PSD for the paper's f1, so no projection), pulled back like the barrier
    fr = ctx.fric
    if fr is not None and len(fr):
        from . import friction as Fr
        from .mesh import all_positions
        P = all_positions(model, x, y)
        for k in range(len(fr)):
            X = P[fr.vids[k]]
            rest = Fr.tangential_sq(X, fr.Xn[k], fr.gamma[k], fr.nhat[k]) == 0.0
            args = (_T(fr.Xn[k].ravel()), _T(fr.gamma[k]), _T(fr.nhat[k]), float(fr.mu_lam[k]), fr.eps, rest)
            fk = lambda z: dt2 * Fr.pair_energy(z, *args)
            Xt = _T(X.ravel())
            gk = torch.autograd.functional.jacobian(fk, Xt).numpy()
            Hk = torch.autograd.functional.hessian(fk, Xt).numpy()
            maps = [vertex_dof_map(model, v) for v in fr.vids[k]]
            for si, (ri, Ji) in enumerate(maps):
                if len(ri) == 0:
                    continue
                g[ri] += Ji.T @ gk[3 * si:3 * si + 3]
                for sj, (rj, Jj) in enumerate(maps):
                    if len(rj) == 0:
                        continue
                    add_block(ri, rj, Ji.T @ Hk[3 * si:3 * si + 3, 3 * sj:3 * sj + 3] @ Jj)
    if rows:
        H = sp.coo_matrix((np.concatenate(vals), (np.concatenate(rows), np.concatenate(cols))), shape=(n, n)).tocsr()
    else:
        H = sp.csr_matrix((n, n))
    return g, H


# ---------------------------------------------------------------------------------------------
# DoF vector helpers
# ---------------------------------------------------------------------------------------------

def pack(model: Model, x, y):
    q = np.zeros(model.n_dof)
    q[:3 * model.V] = np.asarray(x).ravel()
    for bi in range(len(model.body_xbar)):
        s = model.dof_slot[bi]
        if s >= 0:
            q[3 * model.V + 12 * s:3 * model.V + 12 * s + 12] = y[bi]
    return q


def unpack(model: Model, q, y_like):
    x = q[:3 * model.V].reshape(-1, 3).copy()
    y = np.array(y_like, np.float64, copy=True)
    for bi in range(len(model.body_xbar)):
        s = model.dof_slot[bi]
        if s >= 0:
            y[bi] = q[3 * model.V + 12 * s:3 * model.V + 12 * s + 12]
    return x, y
