"""Oracle primitive distances (test infrastructure only — see oracle/__init__.py).

Contact pairs are point-triangle (PT) and edge-edge (EE) pairs of surface primitives (P:L391,
Eq. ipc_energy P:L393 acts on their distance d_k).  The paper does not define the closest-point
classification; this follows SURVEY §8(c)-10/11 (reading R6/R7 in DESIGN.md):

PT: interior iff the projected barycentric coordinates are all ≥ 0 (point-plane distance); else
    the minimum over the three edges e0=(t0,t1), e1=(t1,t2), e2=(t2,t0) of the clamped
    point-segment distance (parameter ≤0 → vertex a, ≥1 → vertex b, else point-line), ties to the
    lowest edge index.  Types: 0 P-T, 1..3 P-E0..2, 4..6 P-V0..2.
EE: Ericson's clamped closest-point order (solve s; t=(b·s+f)/e; clamp t, re-solve s); parallel
    iff a·e−b² ≤ 1e-14·a·e → s=0.  Type = 3·state(s) + state(t), state ∈ {0: endpoint 0,
    1: interior, 2: endpoint 1}; type 4 is line-line.

The squared distance of a pair is that of its active sub-primitive:
    point-point ‖p−q‖², point-line ‖(p−a)×(b−a)‖²/‖b−a‖², point-plane ((p−t0)·n)²/‖n‖²,
    line-line ((a0−b0)·n)²/‖n‖² with n=(a1−a0)×(b1−b0).
Functions are written once over an array module ``xp`` (numpy for classification, torch for the
autograd derivatives in energy.py).
"""
from __future__ import annotations

import numpy as np

PT_T, PT_E0, PT_E1, PT_E2, PT_V0, PT_V1, PT_V2 = range(7)
EE_LL = 4


def _cross(xp, a, b):
    return xp.stack([a[..., 1] * b[..., 2] - a[..., 2] * b[..., 1],
                     a[..., 2] * b[..., 0] - a[..., 0] * b[..., 2],
                     a[..., 0] * b[..., 1] - a[..., 1] * b[..., 0]], -1)


def _dot(a, b):
    return (a * b).sum(-1)


def d2_pp(xp, p, q):
    d = p - q
    return _dot(d, d)


def d2_pl(xp, p, a, b):
    e = b - a
    c = _cross(xp, p - a, e)
    return _dot(c, c) / _dot(e, e)


def d2_pt_plane(xp, p, t0, t1, t2):
    n = _cross(xp, t1 - t0, t2 - t0)
    u = _dot(p - t0, n)
    return u * u / _dot(n, n)


def d2_ll(xp, a0, a1, b0, b1):
    n = _cross(xp, a1 - a0, b1 - b0)
    u = _dot(a0 - b0, n)
    return u * u / _dot(n, n)


def pt_type(p, t0, t1, t2):
    """Vectorised PT classification (numpy, arrays (...,3)) → (type, squared distance)."""
    p, t0, t1, t2 = (np.asarray(a, np.float64) for a in (p, t0, t1, t2))
    e1, e2, w = t1 - t0, t2 - t0, p - t0
    a11, a12, a22 = _dot(e1, e1), _dot(e1, e2), _dot(e2, e2)
    b1, b2 = _dot(e1, w), _dot(e2, w)
    det = a11 * a22 - a12 * a12
    be1 = (a22 * b1 - a12 * b2) / det
    be2 = (a11 * b2 - a12 * b1) / det
    be0 = 1.0 - be1 - be2
    inside = (be0 >= 0) & (be1 >= 0) & (be2 >= 0)
    T = [t0, t1, t2]
    best_d = np.full(p.shape[:-1], np.inf)
    best_t = np.zeros(p.shape[:-1], np.int64)
    for i in range(3):
        a, b = T[i], T[(i + 1) % 3]
        e = b - a
        s = _dot(p - a, e) / _dot(e, e)
        d_a, d_b, d_l = d2_pp(np, p, a), d2_pp(np, p, b), d2_pl(np, p, a, b)
        d = np.where(s <= 0, d_a, np.where(s >= 1, d_b, d_l))
        typ = np.where(s <= 0, PT_V0 + i, np.where(s >= 1, PT_V0 + (i + 1) % 3, PT_E0 + i))
        better = d < best_d
        best_d = np.where(better, d, best_d)
        best_t = np.where(better, typ, best_t)
    d_plane = d2_pt_plane(np, p, t0, t1, t2)
    typ = np.where(inside, PT_T, best_t)
    d2 = np.where(inside, d_plane, best_d)
    return typ, d2


def ee_type(a0, a1, b0, b1):
    """Vectorised EE classification (numpy) → (type, squared distance)."""
    a0, a1, b0, b1 = (np.asarray(v, np.float64) for v in (a0, a1, b0, b1))
    d1, d2v, r = a1 - a0, b1 - b0, a0 - b0
    A, E, F = _dot(d1, d1), _dot(d2v, d2v), _dot(d2v, r)
    C, B = _dot(d1, r), _dot(d1, d2v)
    denom = A * E - B * B
    par = denom <= 1e-14 * A * E
    with np.errstate(divide="ignore", invalid="ignore"):
        s = np.where(par, 0.0, np.clip((B * F - C * E) / np.where(par, 1.0, denom), 0.0, 1.0))
    t = (B * s + F) / E
    lo, hi = t < 0, t > 1
    s = np.where(lo, np.clip(-C / A, 0.0, 1.0), np.where(hi, np.clip((B - C) / A, 0.0, 1.0), s))
    t = np.where(lo, 0.0, np.where(hi, 1.0, t))
    ss = np.where(s == 0, 0, np.where(s == 1, 2, 1))
    ts = np.where(t == 0, 0, np.where(t == 1, 2, 1))
    typ = 3 * ss + ts
    d2 = ee_d2_of_type(np, typ, a0, a1, b0, b1)
    return typ, d2


def ee_d2_of_type(xp, typ, a0, a1, b0, b1):
    """Squared distance of the EE sub-primitive selected by `typ` (vectorised)."""
    with np.errstate(divide="ignore", invalid="ignore"):
        out = d2_ll(xp, a0, a1, b0, b1)
        for k in range(9):
            if k != EE_LL:
                out = xp.where(typ == k, ee_d2_single(xp, k, a0, a1, b0, b1), out)
    return out


def pt_d2_of_type(xp, typ, p, t0, t1, t2):
    """Squared distance of the PT sub-primitive selected by `typ` (vectorised)."""
    T = [t0, t1, t2]
    out = d2_pt_plane(xp, p, t0, t1, t2)
    for i in range(3):
        out = xp.where(typ == PT_E0 + i, d2_pl(xp, p, T[i], T[(i + 1) % 3]), out)
        out = xp.where(typ == PT_V0 + i, d2_pp(xp, p, T[i]), out)
    return out


def pt_d2_single(xp, typ, p, t0, t1, t2):
    """Sub-distance for ONE fixed type (no masking) — used under autograd."""
    T = [t0, t1, t2]
    if typ == PT_T:
        return d2_pt_plane(xp, p, t0, t1, t2)
    if PT_E0 <= typ <= PT_E2:
        i = typ - PT_E0
        return d2_pl(xp, p, T[i], T[(i + 1) % 3])
    return d2_pp(xp, p, T[typ - PT_V0])


def ee_d2_single(xp, typ, a0, a1, b0, b1):
    ss, ts = divmod(int(typ), 3)
    pa, pb = [a0, None, a1], [b0, None, b1]
    if ss == 1 and ts == 1:
        return d2_ll(xp, a0, a1, b0, b1)
    if ss == 1:
        return d2_pl(xp, pb[ts], a0, a1)
    if ts == 1:
        return d2_pl(xp, pa[ss], b0, b1)
    return d2_pp(xp, pa[ss], pb[ts])
