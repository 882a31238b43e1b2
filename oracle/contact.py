"""Oracle contact sets and additive CCD (test infrastructure only — see oracle/__init__.py).

* Pair universe ("point-triangle and edge-edge pairs from the surface meshes of soft and
  affine objects"): PT = (surface vertex of body B₁, surface triangle of body B₂), EE = (edge a of
  B₁, edge b of B₂) with a < b, for body pairs allowed by the filter of reading R8.
* Candidate set C (static) / C′ (swept): every allowed pair whose axis-aligned boxes overlap when
  the target primitive's box (triangle for PT, edge b for EE) is inflated by d̂ — brute force over
  all pairs; for C′ each primitive's box spans its start and end positions (x and x+p).
* Active set 𝒜 = {k : s_k < d̂²}, strict (P:L393's indicator on the open interval (0, d̂)),
  canonically ordered by (kind PT<EE, a, b).
* ACCD (reading R16; P:L195 motivates linear-trajectory CCD for ABD): additive CCD with
  s = 0.1, t_c = 1 on the pair's four linear vertex trajectories.
"""
from __future__ import annotations

import numpy as np

from . import distance as D
from .energy import Pairs
from .mesh import Model


def _boxes(P0, P1, idx):
    """Box of primitives given their vertex ids idx (N,k), spanning both P0 and P1."""
    A, B = P0[idx], P1[idx]
    lo = np.minimum(A.min(1), B.min(1))
    hi = np.maximum(A.max(1), B.max(1))
    return lo, hi


def _overlap_matrix(qlo, qhi, tlo_i, thi_i):
    """M[i, j] = query box i (raw) overlaps target box j (inflated by d̂)."""
    return (np.all(qlo[:, None, :] <= thi_i[None, :, :], 2) & np.all(tlo_i[None, :, :] <= qhi[:, None, :], 2))


def candidate_pairs(model: Model, P0, P1=None):
    """Brute-force candidate set over all allowed pairs (reading R8/R11): returns (kind, a, b) rows
    in canonical order.  Query box raw, target box inflated by d̂:  lo_q ≤ hi_t + d̂ and
    lo_t − d̂ ≤ hi_q on every axis.  Evaluated body pair by body pair; primitives whose box misses
    the other body's (inflated) bounding box are skipped, which cannot change the result because
    the predicate is monotone in the boxes (fl(min lo − d̂) = min fl(lo − d̂))."""
    dhat = model.scene.config.dhat
    P1 = P0 if P1 is None else P1
    NB = model.allowed.shape[0]
    sv = model.surf_verts
    vlo, vhi = _boxes(P0, P1, sv[:, None])
    tlo, thi = _boxes(P0, P1, model.tris)
    elo, ehi = _boxes(P0, P1, model.edges)
    vb, tb, eb = model.vert_body[sv], model.tri_body, model.edge_body

    def body_box(lo, hi, mask):
        return lo[mask].min(0), hi[mask].max(0)

    out = []
    for bq in range(NB):
        for bt in range(NB):
            if not model.allowed[bq, bt]:
                continue
            # PT: vertices of bq against triangles of bt
            qm, tm = vb == bq, tb == bt
            if qm.any() and tm.any():
                Tlo, Thi = body_box(tlo, thi, tm)
                Qlo, Qhi = body_box(vlo, vhi, qm)
                qi = np.nonzero(qm & np.all(vlo <= Thi + dhat, 1) & np.all(Tlo - dhat <= vhi, 1))[0]
                ti = np.nonzero(tm & np.all(Qlo <= thi + dhat, 1) & np.all(tlo - dhat <= Qhi, 1))[0]
                if len(qi) and len(ti):
                    Mx = _overlap_matrix(vlo[qi], vhi[qi], tlo[ti] - dhat, thi[ti] + dhat)
                    ii, jj = np.nonzero(Mx)
                    out += [(0, int(sv[qi[i]]), int(ti[j])) for i, j in zip(ii, jj)]
            # EE: edges of bq (lower indices) against edges of bt, only for bq < bt
            if bq < bt:
                qm, tm = eb == bq, eb == bt
                if qm.any() and tm.any():
                    Tlo, Thi = body_box(elo, ehi, tm)
                    Qlo, Qhi = body_box(elo, ehi, qm)
                    qi = np.nonzero(qm & np.all(elo <= Thi + dhat, 1) & np.all(Tlo - dhat <= ehi, 1))[0]
                    ti = np.nonzero(tm & np.all(Qlo <= ehi + dhat, 1) & np.all(elo - dhat <= Qhi, 1))[0]
                    if len(qi) and len(ti):
                        Mx = _overlap_matrix(elo[qi], ehi[qi], elo[ti] - dhat, ehi[ti] + dhat)
                        ii, jj = np.nonzero(Mx)
                        out += [(1, int(qi[i]), int(ti[j])) for i, j in zip(ii, jj)]
    arr = np.asarray(out, np.int64).reshape(-1, 3)
    if len(arr):
        arr = arr[np.lexsort((arr[:, 2], arr[:, 1], arr[:, 0]))]
    return arr


def classify(model: Model, P, cand):
    """Type and squared distance of each candidate (kind, a, b) at positions P."""
    typ = np.zeros(len(cand), np.int64)
    d2 = np.zeros(len(cand))
    pt = cand[:, 0] == 0
    if pt.any():
        v, t = cand[pt, 1], model.tris[cand[pt, 2]]
        typ[pt], d2[pt] = D.pt_type(P[v], P[t[:, 0]], P[t[:, 1]], P[t[:, 2]])
    ee = ~pt
    if ee.any():
        ea, eb = model.edges[cand[ee, 1]], model.edges[cand[ee, 2]]
        typ[ee], d2[ee] = D.ee_type(P[ea[:, 0]], P[ea[:, 1]], P[eb[:, 0]], P[eb[:, 1]])
    return typ, d2


def active_pairs(model: Model, P, cand=None) -> Pairs:
    """𝒜 = {k : s_k < d̂²} (strict) in canonical order."""
    if cand is None:
        cand = candidate_pairs(model, P)
    typ, d2 = classify(model, P, cand)
    keep = d2 < model.scene.config.dhat ** 2
    c = cand[keep]
    return Pairs(kind=c[:, 0], a=c[:, 1], b=c[:, 2], typ=typ[keep], d2=d2[keep])


def min_distance(model: Model, P):
    """Smallest squared distance over all allowed pairs whose boxes overlap (for audits)."""
    cand = candidate_pairs(model, P)
    if len(cand) == 0:
        return np.inf
    _, d2 = classify(model, P, cand)
    return float(d2.min())


def _pair_d2(kind, X):
    if kind == 0:
        return float(D.pt_type(X[0], X[1], X[2], X[3])[1])
    return float(D.ee_type(X[0], X[1], X[2], X[3])[1])


def accd(kind, X, Pd, s=0.1, t_c=1.0, max_iters=10000):
    """Additive CCD (Li et al. 2021, reading R16) for one pair with positions X (4,3) and
    displacements Pd (4,3); returns the step bound t ∈ (0, 1].

      subtract the mean displacement; l_p = ‖p0‖ + max(‖p1‖,‖p2‖,‖p3‖) (PT) or
      max(‖p0‖,‖p1‖) + max(‖p2‖,‖p3‖) (EE); l_p = 0 → 1.  g = s·d₀.  t = 0,
      t_l = (1−s)·d/l_p.  loop: X += t_l·Pd; d = dist(X); if t > 0 and d < g: stop;
      t += t_l; if t > t_c: return 1;  t_l = (1−s)·d/l_p.  Return t (cap → current t)."""
    X = np.array(X, np.float64, copy=True)
    Pd = np.asarray(Pd, np.float64) - np.asarray(Pd, np.float64).mean(0)
    n = np.sqrt((Pd * Pd).sum(1))
    lp = n[0] + max(n[1], n[2], n[3]) if kind == 0 else max(n[0], n[1]) + max(n[2], n[3])
    if lp == 0.0:
        return 1.0
    d = np.sqrt(_pair_d2(kind, X))
    g = s * d
    t = 0.0
    tl = (1.0 - s) * d / lp
    it = 0
    while True:
        X = X + tl * Pd
        d = np.sqrt(_pair_d2(kind, X))
        if t > 0.0 and d < g:
            break
        t += tl
        if t > t_c:
            return 1.0
        tl = (1.0 - s) * d / lp
        it += 1
        if it >= max_iters:
            break
    return t


def accd_bound(model: Model, P0, Pdisp, cand):
    """α_max = min(1, min over C′ of ACCD)."""
    cfg = model.scene.config
    from .energy import pair_vertices
    alpha = 1.0
    for kind, a, b in cand:
        vids = pair_vertices(model, int(kind), int(a), int(b))
        t = accd(int(kind), P0[vids], Pdisp[vids], cfg.accd_s, 1.0, cfg.max_accd_iters)
        alpha = min(alpha, t)
    return alpha
