"""Oracle lagged friction (test infrastructure only — see oracle/__init__.py).

P:L398-412 (App. A.3, Frictional Contact): each contact pair k adds the approximate friction potential
    D_k(x, xⁿ) = μ λ_kⁿ f0(‖u_k‖)
with λ_kⁿ "the magnitude of the lagged normal contact force", u_k ∈ ℝ² "the tangential relative
displacement in the local contact frame", and
    f0(x) = ∫_{ε_vΔt}^{x} f1(y) dy + ε_vΔt,
    f1(y) = −y²/(ε_v²Δt²) + 2y/(ε_vΔt)  for y ∈ (0, Δt ε_v),   f1(y) = 1  for y ≥ Δt ε_v;
the full objective adds Δt²·Σ_k D_k (P:L102 Eq. fullspace_ipc, P:L414 Eq. suppeq:fullspace_ipc).

Written out (ε = ε_vΔt), the integral of the paper's f1 gives
    f0(x) = −x³/(3ε²) + x²/ε + ε/3   for x < ε,        f0(x) = x   for x ≥ ε
(∫_ε^x (−y²/ε² + 2y/ε) dy + ε = [−y³/(3ε²) + y²/ε]_ε^x + ε = −x³/(3ε²) + x²/ε − 2ε/3 + ε; pinned in
tests by df0/dx = f1 and f0(0) = ε/3).

Readings of what the paper leaves open (R20):
  * lagging: the friction pairs, λ_kⁿ, the contact normal and the closest-point weights are frozen once
    per time step at xⁿ ("frozen from the previous time step", no friction outer loop); the pairs
    are the barrier's active set 𝒜(xⁿ);
  * λ_kⁿ = κ A_k m_k |b′(d_k)| at xⁿ — the magnitude of the force of pair k's barrier potential
    κ A_k m_k b(d_k) (m_k = 1 for PT, the EE mollifier otherwise);
  * Γ_k: the closest-point weights at xⁿ (PT: p − Σβ_i t_i with the closest point's barycentric β on
    the triangle; EE: (1−s)a₀ + s a₁ − (1−t)b₀ − t b₁ with the closest-point parameters), so Γ_k X is the
    separation vector of the closest points and n̂ = Γ_k Xⁿ / d_k;
  * u_k = T_kᵀ Γ_k (X − Xⁿ) for any orthonormal basis T_k of the plane ⊥ n̂, hence
    ‖u_k‖ = ‖(I − n̂n̂ᵀ) Γ_k (X − Xⁿ)‖ (the basis choice does not enter the energy).
"""
from __future__ import annotations

import dataclasses

import numpy as np
import torch

from . import distance as Dst
from .mesh import Model, all_positions

torch.set_default_dtype(torch.float64)


def f1(y, eps):
    """The paper's f1, eps = ε_vΔt."""
    return torch.where(y < eps, -y * y / (eps * eps) + 2.0 * y / eps, torch.ones_like(y))


def f0(x, eps):
    """f0(x) = ∫_ε^x f1 + ε, written out (module docstring)."""
    return torch.where(x < eps, -x ** 3 / (3.0 * eps * eps) + x * x / eps + eps / 3.0, x)


def closest_weights(kind, typ, X):
    """Γ weights (4,) of the closest points for a classified pair with positions X (4, 3), numpy.
    PT slots (p, t0, t1, t2); EE slots (a0, a1, b0, b1)."""
    X = np.asarray(X, np.float64)
    g = np.zeros(4)
    if kind == 0:
        p, t0, t1, t2 = X
        g[0] = 1.0
        if typ == Dst.PT_T:
            e1, e2, w = t1 - t0, t2 - t0, p - t0
            a11, a12, a22 = e1 @ e1, e1 @ e2, e2 @ e2
            b1, b2 = e1 @ w, e2 @ w
            det = a11 * a22 - a12 * a12
            be1 = (a22 * b1 - a12 * b2) / det
            be2 = (a11 * b2 - a12 * b1) / det
            g[1:] = [-(1.0 - be1 - be2), -be1, -be2]
        elif Dst.PT_E0 <= typ <= Dst.PT_E2:
            i = typ - Dst.PT_E0
            T = [t0, t1, t2]
            a, b = T[i], T[(i + 1) % 3]
            s = (p - a) @ (b - a) / ((b - a) @ (b - a))
            g[1 + i] -= 1.0 - s
            g[1 + (i + 1) % 3] -= s
        else:
            g[1 + typ - Dst.PT_V0] = -1.0
        return g
    a0, a1, b0, b1 = X
    ss, ts = divmod(int(typ), 3)
    d1, d2, r = a1 - a0, b1 - b0, a0 - b0
    if ss == 1 and ts == 1:                      # line-line: solve for both parameters
        A, B, E = d1 @ d1, d1 @ d2, d2 @ d2
        C, F = d1 @ r, d2 @ r
        den = A * E - B * B
        s = (B * F - C * E) / den
        t = (A * F - B * C) / den
    elif ss == 1:                                # endpoint of b against segment a
        t = 0.0 if ts == 0 else 1.0
        q = b0 if ts == 0 else b1
        s = (q - a0) @ d1 / (d1 @ d1)
    elif ts == 1:                                # endpoint of a against segment b
        s = 0.0 if ss == 0 else 1.0
        q = a0 if ss == 0 else a1
        t = (q - b0) @ d2 / (d2 @ d2)
    else:
        s = 0.0 if ss == 0 else 1.0
        t = 0.0 if ts == 0 else 1.0
    return np.array([1.0 - s, s, -(1.0 - t), -t])


@dataclasses.dataclass
class FrictionData:
    """Lagged friction pairs of one env for one time step (frozen at xⁿ)."""
    vids: np.ndarray     # (K, 4) global vertex ids of the pair slots
    gamma: np.ndarray    # (K, 4) closest-point weights Γ_k
    nhat: np.ndarray     # (K, 3) contact normal at xⁿ
    mu_lam: np.ndarray   # (K,) μ·λ_kⁿ
    Xn: np.ndarray       # (K, 4, 3) slot positions at xⁿ
    eps: float           # ε_vΔt

    def __len__(self):
        return len(self.mu_lam)


def barrier_d1(d, dhat):
    """b′(d) of the barrier b(d) = −(d − d̂)² ln(d/d̂), by torch autograd of the definition."""
    from .energy import barrier
    t = torch.as_tensor(np.atleast_1d(np.asarray(d, np.float64))).requires_grad_(True)
    (g,) = torch.autograd.grad(barrier(t, dhat).sum(), t)
    return g.numpy()


def lagged(model: Model, x_n, y_n) -> FrictionData:
    """Friction pairs and their frozen data at xⁿ (readings in the module docstring)."""
    from . import contact as Cn
    from . import energy as En
    cfg = model.scene.config
    eps = cfg.eps_v * cfg.dt
    P = all_positions(model, x_n, y_n)
    pairs = Cn.active_pairs(model, P)
    K = len(pairs)
    vids = np.zeros((K, 4), np.int64)
    gam = np.zeros((K, 4))
    nh = np.zeros((K, 3))
    lam = np.zeros(K)
    if K:
        d = np.sqrt(pairs.d2)
        b1 = barrier_d1(d, cfg.dhat)
    for k in range(K):
        kind, a, b = int(pairs.kind[k]), int(pairs.a[k]), int(pairs.b[k])
        vids[k] = En.pair_vertices(model, kind, a, b)
        X = P[vids[k]]
        gam[k] = closest_weights(kind, int(pairs.typ[k]), X)
        sep = gam[k] @ X
        nh[k] = sep / np.linalg.norm(sep)
        m = 1.0
        if kind == 1 and cfg.ee_mollifier:
            c = np.cross(X[1] - X[0], X[3] - X[2])
            c = float(c @ c)
            ex = En.pair_eps(model, kind, a, b)
            m = (2.0 - c / ex) * (c / ex) if c < ex else 1.0
        lam[k] = cfg.kappa * En.pair_area(model, kind, a, b) * m * abs(float(b1[k]))
    return FrictionData(vids=vids, gamma=gam, nhat=nh, mu_lam=cfg.mu_friction * lam, Xn=P[vids] if K else np.zeros((0, 4, 3)),
                        eps=eps)


def tangential_sq(X, Xn, gamma, nhat):
    """‖(I − n̂n̂ᵀ) Γ (X − Xⁿ)‖² (numpy), to pick the at-rest form of pair_energy."""
    w = gamma @ (np.asarray(X) - np.asarray(Xn))
    v = w - nhat * (nhat @ w)
    return float(v @ v)


def pair_energy(X12, Xn12, gamma, nhat, mu_lam, eps, at_rest=False):
    """D_k = μλ_k f0(‖(I − n̂n̂ᵀ) Γ_k (X − Xⁿ)‖) for one pair (torch, X12 = the 4 slot positions).
    at_rest (‖u‖ = 0 exactly, e.g. at the first Newton iterate x = xⁿ): f0(z) = z²/ε + ε/3 − z³/(3ε²)
    and the cubic term has zero value, slope and curvature at z = 0, so the energy is evaluated as
    μλ(z²/ε + ε/3) there — the same value, gradient and Hessian, without √0 in the derivatives."""
    dX = (X12 - Xn12).reshape(4, 3)
    w = (gamma[:, None] * dX).sum(0)
    v = w - nhat * (nhat * w).sum()
    z2 = (v * v).sum()
    if at_rest:
        return mu_lam * (z2 / eps + eps / 3.0)
    return mu_lam * f0(torch.sqrt(z2), eps)
