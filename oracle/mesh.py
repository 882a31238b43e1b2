"""Oracle mesh preparation (test infrastructure only — see oracle/__init__.py).

Rest quantities of the soft FEM bodies (stacked x, lumped M, Φ=∫Ψ), contact
surfaces and rest areas ("point-triangle and edge-edge pairs from the surface meshes"),
and the ABD reduced quantities J and M^y = JᵀMJ.
"""
from __future__ import annotations

import dataclasses
from typing import List

import numpy as np

from paper_2504_12908_b200.scenes import DYNAMIC, KINEMATIC, STATIC, Scene

SOFT = -1  # body kind tag for soft pads in the body-pair rules


@dataclasses.dataclass
class Model:
    scene: Scene
    # soft FEM
    V: int
    X: np.ndarray            # (V,3) rest positions (pad frames)
    tets: np.ndarray         # (T,4) positively oriented
    Dm_inv: np.ndarray       # (T,3,3)
    vol: np.ndarray          # (T,)
    mu: np.ndarray           # (T,)
    lam: np.ndarray          # (T,)
    mass: np.ndarray         # (V,)
    # affine bodies
    n_soft_bodies: int
    body_kind: np.ndarray    # (NA,)
    body_xbar: List[np.ndarray]
    body_mass: np.ndarray
    body_s1: np.ndarray      # (NA,3)  ∫ρ x̄
    body_vol: np.ndarray
    body_My: np.ndarray      # (NA,12,12)
    body_kappa: np.ndarray
    dof_slot: np.ndarray     # (NA,) index of the body's 12 DoFs among non-static bodies, -1 for static
    n_dof_bodies: int
    # contact primitives (global vertex numbering: soft 0..V-1, then affine bodies' vertices)
    NVall: int
    vert_body: np.ndarray    # (NVall,) global body id (soft pads first, then affine)
    vert_aff: np.ndarray     # (NVall,) affine body index or -1
    vert_xbar: np.ndarray    # (NVall,3) rest position in own frame
    surf_verts: np.ndarray   # sorted global ids of contact vertices
    tris: np.ndarray         # (NT,3) global vertex ids
    tri_body: np.ndarray
    edges: np.ndarray        # (NE,2)
    edge_body: np.ndarray
    A_v: np.ndarray          # (NVall,) rest vertex area weight
    A_e: np.ndarray          # (NE,)
    edge_rest_len2: np.ndarray
    allowed: np.ndarray      # (NB,NB) body-pair mask
    # kinematic constraints
    att_vert: np.ndarray     # (NC,) soft vertex ids in ∂⁻G
    att_body: np.ndarray     # (NC,) mount affine body index
    att_local: np.ndarray    # (NC,3) position in the mount body frame: mount_T(X_v)
    kin_bodies: np.ndarray   # (NK,) affine body indices with kinematic targets

    @property
    def n_dof(self) -> int:
        return 3 * self.V + 12 * self.n_dof_bodies


def lame(youngs: float, poisson: float):
    """Lamé parameters from (ℰ, ν) (P:L86 names the NH model by ℰ, ν)."""
    mu = youngs / (2.0 * (1.0 + poisson))
    lam = youngs * poisson / ((1.0 + poisson) * (1.0 - 2.0 * poisson))
    return mu, lam


def orient_tets(X, tets):
    """Swap two indices of any tet with negative signed volume (SPEC S:L46 orientation fix)."""
    tets = tets.copy()
    for i, t in enumerate(tets):
        D = np.stack([X[t[1]] - X[t[0]], X[t[2]] - X[t[0]], X[t[3]] - X[t[0]]], 1)
        v = np.linalg.det(D) / 6.0
        if abs(v) < 1e-15:
            raise ValueError(f"degenerate tet {i} (|volume| {abs(v):.3e} < 1e-15 m^3)")
        if v < 0:
            tets[i, [1, 2]] = tets[i, [2, 1]]
    return tets


def tet_rest(X, tets):
    """D_m (columns X1-X0, X2-X0, X3-X0), its inverse and V_e = det(D_m)/6 > 0."""
    Dm = np.stack([X[tets[:, 1]] - X[tets[:, 0]], X[tets[:, 2]] - X[tets[:, 0]],
                   X[tets[:, 3]] - X[tets[:, 0]]], 2)
    vol = np.linalg.det(Dm) / 6.0
    return np.linalg.inv(Dm), vol


def lumped_mass(nv, tets, vol, density):
    """Each tet gives ρV_e/4 to each of its vertices."""
    m = np.zeros(nv)
    for t, v in zip(tets, vol):
        for a in t:
            m[a] += density * v / 4.0
    return m


def canonical_tri(t):
    """Rotate an oriented triangle so its smallest vertex id comes first (orientation kept)."""
    t = list(t)
    k = int(np.argmin(t))
    return tuple(t[k:] + t[:k])


def boundary_faces(tets):
    """Faces appearing in exactly one tet, oriented outward for positively oriented tets
    (faces (a,c,b), (a,b,d), (a,d,c), (b,c,d)), in canonical order (sorted by sorted triple)."""
    count = {}
    oriented = {}
    for a, b, c, d in tets:
        for f in ((a, c, b), (a, b, d), (a, d, c), (b, c, d)):
            key = tuple(sorted(f))
            count[key] = count.get(key, 0) + 1
            oriented[key] = canonical_tri(f)
    keys = sorted(k for k, n in count.items() if n == 1)
    return np.asarray([oriented[k] for k in keys], np.int64).reshape(-1, 3)


def sorted_tris(tris):
    keys = [tuple(sorted(t)) for t in tris]
    order = sorted(range(len(tris)), key=lambda i: keys[i])
    return np.asarray([canonical_tri(tris[i]) for i in order], np.int64).reshape(-1, 3)


def tri_edges(tris):
    """Unique undirected edges (min,max) of a triangle list, sorted lexicographically."""
    s = set()
    for t in tris:
        for i in range(3):
            a, b = int(t[i]), int(t[(i + 1) % 3])
            s.add((min(a, b), max(a, b)))
    return np.asarray(sorted(s), np.int64).reshape(-1, 2)


def tri_area(P, tris):
    return 0.5 * np.linalg.norm(np.cross(P[tris[:, 1]] - P[tris[:, 0]], P[tris[:, 2]] - P[tris[:, 0]]), axis=1)


def affine_jacobian(xbar):
    """J_v = ∂(t + A x̄)/∂y for y = (t, A row-major): [I₃ | I₃ ⊗ x̄ᵀ]."""
    J = np.zeros((3, 12))
    J[:, :3] = np.eye(3)
    for i in range(3):
        J[i, 3 + 3 * i:6 + 3 * i] = xbar
    return J


_Q_A, _Q_B = 0.5854101966249685, 0.1381966011250105   # 4-point tet rule, exact for degree 2


def body_moments(xbar, tris, density):
    """Volume, mass, ∫ρx̄ and M^y = ∫_Ω ρ J(x̄)ᵀJ(x̄) dV (= JᵀMJ with M the body's volumetric mass,
    P:L113-116) by exact degree-2 quadrature over the signed tets (0, a, b, c) of the closed surface
    (divergence theorem)."""
    vol, s1, My = 0.0, np.zeros(3), np.zeros((12, 12))
    for t in tris:
        P = [np.zeros(3), xbar[t[0]], xbar[t[1]], xbar[t[2]]]
        v = np.dot(P[1], np.cross(P[2], P[3])) / 6.0
        vol += v
        for q in range(4):
            bary = np.full(4, _Q_B)
            bary[q] = _Q_A
            xq = sum(bary[i] * P[i] for i in range(4))
            w = v / 4.0
            s1 += density * w * xq
            J = affine_jacobian(xq)
            My += density * w * (J.T @ J)
    return vol, density * vol, s1, My


def body_pair_allowed(kind_a, kind_b, a, b, mount_of_soft):
    """Contact filter (proposal): different bodies; not a pad with its own mount
    link; not static/kinematic against static/kinematic (relative motion prescribed)."""
    if a == b:
        return False
    for s, o in ((a, b), (b, a)):
        if s in mount_of_soft and mount_of_soft[s] == o:
            return False
    if kind_a in (STATIC, KINEMATIC) and kind_b in (STATIC, KINEMATIC):
        return False
    return True


def prepare(scene: Scene) -> Model:
    # ---- soft bodies ----
    Xs, Ts, ms, mus, lams = [], [], [], [], []
    off = 0
    tris_soft, pad_bodies = [], []
    att_v, att_b, att_l = [], [], []
    for pi, pad in enumerate(scene.soft):
        X = np.asarray(pad.rest_pos, np.float64)
        tets = orient_tets(X, np.asarray(pad.tets, np.int64))
        Dinv, vol = tet_rest(X, tets)
        mu, lam = lame(pad.youngs, pad.poisson)
        Xs.append(X)
        Ts.append(tets + off)
        ms.append(lumped_mass(len(X), tets, vol, pad.density))
        mus.append(np.full(len(tets), mu))
        lams.append(np.full(len(tets), lam))
        tris_soft.append(boundary_faces(tets) + off)
        if pad.mount_body >= 0:
            R = np.asarray(pad.mount_T[3:], np.float64).reshape(3, 3)
            t = np.asarray(pad.mount_T[:3], np.float64)
            for v in pad.attached:
                att_v.append(off + int(v))
                att_b.append(pad.mount_body)
                att_l.append(t + R @ X[v])
        off += len(X)
    V = off
    X = np.concatenate(Xs) if Xs else np.zeros((0, 3))
    tets = np.concatenate(Ts) if Ts else np.zeros((0, 4), np.int64)
    Dm_inv, vol = tet_rest(X, tets)
    mass = np.concatenate(ms) if ms else np.zeros(0)

    # ---- affine bodies ----
    NA = len(scene.affine)
    ns = len(scene.soft)
    kind = np.array([b.kind for b in scene.affine], np.int64)
    dof_slot = np.full(NA, -1, np.int64)
    k = 0
    for i in range(NA):
        if kind[i] != STATIC:
            dof_slot[i] = k
            k += 1
    bvol, bmass, bs1, bMy = np.zeros(NA), np.zeros(NA), np.zeros((NA, 3)), np.zeros((NA, 12, 12))
    for i, b in enumerate(scene.affine):
        bvol[i], bmass[i], bs1[i], bMy[i] = body_moments(np.asarray(b.rest_pos, np.float64), b.tris, b.density)

    # ---- global contact primitives ----
    NVall = V + sum(len(b.rest_pos) for b in scene.affine)
    vert_body = np.zeros(NVall, np.int64)
    vert_aff = np.full(NVall, -1, np.int64)
    vert_xbar = np.zeros((NVall, 3))
    o = 0
    for pi, pad in enumerate(scene.soft):
        n = len(pad.rest_pos)
        vert_body[o:o + n] = pi
        vert_xbar[o:o + n] = pad.rest_pos
        o += n
    tri_list, tri_body, edge_list, edge_body = [], [], [], []
    for pi in range(ns):
        T = tris_soft[pi]
        tri_list.append(T)
        tri_body += [pi] * len(T)
        E = tri_edges(T)
        edge_list.append(E)
        edge_body += [pi] * len(E)
    for i, b in enumerate(scene.affine):
        n = len(b.rest_pos)
        vert_body[o:o + n] = ns + i
        vert_aff[o:o + n] = i
        vert_xbar[o:o + n] = b.rest_pos
        T = sorted_tris(np.asarray(b.tris, np.int64) + o)
        tri_list.append(T)
        tri_body += [ns + i] * len(T)
        E = tri_edges(T)
        edge_list.append(E)
        edge_body += [ns + i] * len(E)
        o += n
    tris = np.concatenate(tri_list).astype(np.int64)
    edges = np.concatenate(edge_list).astype(np.int64)
    surf_verts = np.unique(tris.ravel())

    # rest areas: A_v = 1/3 Σ_{f∋v} area(f̄), A_e = 1/3 Σ_{f∋e} area(f̄) (SURVEY §8(c)-12 proposal)
    areas = tri_area(vert_xbar, tris)
    A_v = np.zeros(NVall)
    for t, a in zip(tris, areas):
        for v in t:
            A_v[v] += a / 3.0
    eidx = {tuple(e): i for i, e in enumerate(edges)}
    A_e = np.zeros(len(edges))
    for t, a in zip(tris, areas):
        for j in range(3):
            u, w = int(t[j]), int(t[(j + 1) % 3])
            A_e[eidx[(min(u, w), max(u, w))]] += a / 3.0
    elen2 = ((vert_xbar[edges[:, 1]] - vert_xbar[edges[:, 0]]) ** 2).sum(1)

    # body-pair mask
    NB = ns + NA
    kinds = [DYNAMIC] * ns + list(kind)
    mount_of_soft = {pi: ns + pad.mount_body for pi, pad in enumerate(scene.soft) if pad.mount_body >= 0}
    allowed = np.zeros((NB, NB), bool)
    for a in range(NB):
        for b in range(NB):
            allowed[a, b] = body_pair_allowed(kinds[a], kinds[b], a, b, mount_of_soft)
    if scene.collide is not None:
        allowed &= np.asarray(scene.collide, bool)

    return Model(scene=scene, V=V, X=X, tets=tets, Dm_inv=Dm_inv, vol=vol,
                 mu=np.concatenate(mus) if mus else np.zeros(0),
                 lam=np.concatenate(lams) if lams else np.zeros(0), mass=mass,
                 n_soft_bodies=ns, body_kind=kind, body_xbar=[np.asarray(b.rest_pos, np.float64) for b in scene.affine],
                 body_mass=bmass, body_s1=bs1, body_vol=bvol, body_My=bMy,
                 body_kappa=np.array([b.kappa_s for b in scene.affine], np.float64),
                 dof_slot=dof_slot, n_dof_bodies=int(k),
                 NVall=NVall, vert_body=vert_body, vert_aff=vert_aff, vert_xbar=vert_xbar,
                 surf_verts=surf_verts, tris=tris, tri_body=np.asarray(tri_body, np.int64),
                 edges=edges, edge_body=np.asarray(edge_body, np.int64), A_v=A_v, A_e=A_e,
                 edge_rest_len2=elen2, allowed=allowed,
                 att_vert=np.asarray(att_v, np.int64), att_body=np.asarray(att_b, np.int64),
                 att_local=np.asarray(att_l, np.float64).reshape(-1, 3),
                 kin_bodies=np.asarray(scene.kinematic_bodies, np.int64))


# ---- state helpers -------------------------------------------------------------------------

def embed(y, xbar):
    """φ: vertex positions t + A x̄."""
    return xbar @ y[3:].reshape(3, 3).T + y[:3]


def all_positions(model: Model, x, y):
    """World positions of every contact vertex: soft x, then each affine body's φ(y_b)."""
    P = np.zeros((model.NVall, 3))
    P[:model.V] = x
    o = model.V
    for i, xb in enumerate(model.body_xbar):
        P[o:o + len(xb)] = embed(y[i], xb)
        o += len(xb)
    return P


def env_scale(model: Model, x, y):
    """L_env: bounding-box diagonal of all vertices at the given (initial) state (SURVEY §8 notation)."""
    P = all_positions(model, x, y)
    return float(np.linalg.norm(P.max(0) - P.min(0)))
