"""Seeded synthetic scene generator (shared INPUT module — holds none of the method's arithmetic).

This module only builds geometry and per-env scripted inputs: tet lattices, watertight box-union
surfaces, rest poses, initial states and kinematic targets.  It is imported by both the oracle
(``oracle/``) and the CUDA path's harness; it never computes energies, derivatives, masses,
distances, surfaces-for-contact or any other step of the method.  Mesh preparation (volumes,
D_m^-1, lumped masses, surface extraction, areas, reduced mass) is done independently by each side.

Workloads follow SURVEY.md §8(d) (the configs of BASELINE.json):
  C1   1 env: ~500-tet gel pad pressed 1 mm by one kinematic ABD cube, 10 steps at dt=1e-2
  C1b  free ABD cube dropped on the pad (variant used for parity)
  C1c  soft cube resting on a static plate (statics variant)
  C2   peg insertion, dual low-res pads (8x6x3 lattice), 1024 envs
  C3   as C2 with high-res pads (19x16x5 lattice), 4096 envs
  C4   parallel-gripper grasp: two 40x40x4 mm pads (14x14x3) squeeze one of 8 procedural star-shaped
       objects (perturbed level-3 icospheres, 642 v / 1280 t) resting on a static table; "C4:k" = shape k
       (homogeneous batch per shape, 256 envs each, 2048 envs in total)
  C5   Allegro-like hand: palm + 4 fingers x 4 kinematic link boxes (17 kinematic bodies), four 24x24x3 mm
       fingertip pads (9x9x4) in a four-sided precision grasp of a dynamic 16x30x22 mm tile whose two 30x22
       faces carry a seeded 0.3 mm engraving (48x36 cells), on a static table; link targets from the
       forward kinematics of a 16-joint script (fk_hand)
  P1   single point-triangle pair: a tet's lowest vertex d̂/2 above a static box (barrier pins)
  P2   single edge-edge pair: two tets' edges crossing at gap d̂/2 (perpendicular; P2m: nearly
       parallel, inside the mollifier range) — also the soft–soft (matrix-free) contact case
Per-env randomness uses numpy's Philox keyed by (250412908 + cfg index, global env id), so an
env's inputs never depend on how envs are sharded across GPUs.

Units are SI (m, kg, s).  Affine states y are 12-vectors (t[3], A[3x3] row-major): a body vertex
with rest position xbar (body frame) sits at t + A xbar (P:L110-116 embedding phi).
"""
from __future__ import annotations

import dataclasses
import math
from typing import List, Optional

import numpy as np

DYNAMIC, KINEMATIC, STATIC = 0, 1, 2
CFG_INDEX = {"C1": 1, "C1b": 11, "C1c": 12, "C2": 2, "C3": 3, "C4": 4, "C5": 5, "P1": 21, "P2": 22, "P2m": 23}
SEED_BASE = 250412908


@dataclasses.dataclass
class SoftPad:
    """A tetrahedral gel pad G_i. rest_pos is in the pad (sensor) frame."""
    rest_pos: np.ndarray            # (nv,3) f64
    tets: np.ndarray                # (nt,4) i32
    youngs: float = 1.0e5
    poisson: float = 0.40
    density: float = 1.0e3
    mount_body: int = -1            # index into Scene.affine, -1 = free soft body
    mount_T: np.ndarray = dataclasses.field(default_factory=lambda: np.r_[np.zeros(3), np.eye(3).ravel()])
    attached: np.ndarray = dataclasses.field(default_factory=lambda: np.zeros(0, np.int32))   # ∂⁻G
    coated: np.ndarray = dataclasses.field(default_factory=lambda: np.zeros(0, np.int32))     # ∂⁺G
    marker_tri: np.ndarray = dataclasses.field(default_factory=lambda: np.zeros((0, 3), np.int32))
    marker_bary: np.ndarray = dataclasses.field(default_factory=lambda: np.zeros((0, 3)))


@dataclasses.dataclass
class AffineBody:
    """An ABD body: closed outward-oriented triangle surface in its body frame."""
    rest_pos: np.ndarray            # (nv,3) f64, body frame
    tris: np.ndarray                # (nt,3) i32, outward
    kind: int = DYNAMIC
    density: float = 1.0e3
    kappa_s: float = 1.0e8


@dataclasses.dataclass
class Config:
    """Solver constants (proposals; the paper gives none)."""
    dt: float = 0.02
    dhat: float = 1.0e-4
    kappa: float = 1.0e8
    max_step_rel: float = 5.0e-2   # relative step cap (R17c)
    newton_tol_rel: float = 1.0e-7
    al_tol_rel: float = 1.0e-6
    pcg_eta: float = 1.0e-4
    armijo_c: float = 1.0e-4
    accd_s: float = 0.1
    al_rho0: float = 1.0e8
    max_newton: int = 400
    max_al_rounds: int = 8
    max_pcg: int = 2000
    max_accd_iters: int = 10000
    ee_mollifier: int = 1
    hessian_mode: int = 2          # 0: PSD-projected; 1: exact first + projected fallback (R14b); 2: exact + LM shift (R14c)
    ls_expand: int = 16            # line-search expansion bound K (R17b); 1 = plain backtracking
    hold_cap: int = 16             # max projected iterations between exact-Hessian attempts (R14b)
    lm_mu0: float = 10.0           # first mass-scaled shift of hessian_mode 2 (R14c); 10 measured best on C2
    bp_margin: float = 1.0e-4      # δ of the reusable candidate list (R11b); 0 = rebuild every iteration
    cand_capacity_per_env: int = 65536
    active_capacity_per_env: int = 4096
    pcg_eta_max: float = 0.0       # relaxed PCG tolerance (reading R24): 0 = fixed η; > 0 = Eisenstat–Walker forcing in [η, η_max]
    mu_friction: float = 0.0       # Coulomb coefficient μ of the lagged friction D_k; 0 = frictionless
    eps_v: float = 1.0e-3          # ε_v (m/s): static/dynamic friction transition of f1 (S:L244 default)


@dataclasses.dataclass
class Scene:
    name: str
    soft: List[SoftPad]
    affine: List[AffineBody]
    gravity: np.ndarray
    config: Config
    n_steps: int
    collide: Optional[np.ndarray] = None

    @property
    def n_soft_verts(self) -> int:
        return int(sum(p.rest_pos.shape[0] for p in self.soft))

    @property
    def kinematic_bodies(self) -> List[int]:
        return [i for i, b in enumerate(self.affine) if b.kind == KINEMATIC]


# ----------------------------------------------------------------------------------------------
# geometry builders (topology + coordinates only)
# ----------------------------------------------------------------------------------------------

def lattice_tets(nx: int, ny: int, nz: int, size):
    """Node lattice nx*ny*nz spanning [0,sx]x[0,sy]x[0,sz], each hex split into 5 tets with the
    alternating (parity) split so neighbouring hexes share face diagonals.  Node id = i + nx*(j + ny*k).
    Tets are returned with the index order of the split; orientation is NOT normalised here."""
    sx, sy, sz = size
    xs, ys, zs = np.linspace(0, sx, nx), np.linspace(0, sy, ny), np.linspace(0, sz, nz)
    X = np.stack(np.meshgrid(xs, ys, zs, indexing="ij"), -1)          # (nx,ny,nz,3)
    pos = X.transpose(2, 1, 0, 3).reshape(-1, 3).copy()                # id = i + nx*(j + ny*k)
    nid = lambda i, j, k: i + nx * (j + ny * k)
    even = [(1, 2, 4, 7), (0, 1, 2, 4), (3, 1, 2, 7), (5, 1, 4, 7), (6, 2, 4, 7)]
    odd = [(0, 3, 5, 6), (1, 0, 3, 5), (2, 0, 3, 6), (4, 0, 5, 6), (7, 3, 5, 6)]
    tets = []
    for k in range(nz - 1):
        for j in range(ny - 1):
            for i in range(nx - 1):
                c = [nid(i + (b & 1), j + ((b >> 1) & 1), k + ((b >> 2) & 1)) for b in range(8)]
                for t in (even if (i + j + k) % 2 == 0 else odd):
                    tets.append([c[t[0]], c[t[1]], c[t[2]], c[t[3]]])
    return pos, np.asarray(tets, np.int32)


def _axis_lines(breaks, spacing):
    """Grid lines covering the sorted break points with segments no longer than `spacing`."""
    out = [breaks[0]]
    for a, b in zip(breaks[:-1], breaks[1:]):
        n = max(1, int(math.ceil((b - a) / spacing - 1e-9)))
        out += list(a + (b - a) * np.arange(1, n + 1) / n)
    return np.asarray(out)


def cell_union_surface(xl, yl, zl, solid):
    """Watertight outward-oriented triangle surface of a union of cells of a rectilinear grid.
    solid[i,j,k] marks cell [xl[i],xl[i+1]]x[yl[j],yl[j+1]]x[zl[k],zl[k+1]].  Every face between
    a solid and an empty cell becomes a quad split into two triangles; vertices are grid nodes."""
    nx, ny, nz = solid.shape
    S = np.zeros((nx + 2, ny + 2, nz + 2), bool)
    S[1:-1, 1:-1, 1:-1] = solid
    vid = {}
    verts, tris = [], []

    def v(i, j, k):
        key = (i, j, k)
        if key not in vid:
            vid[key] = len(verts)
            verts.append((xl[i], yl[j], zl[k]))
        return vid[key]

    for ax in range(3):
        for i in range(nx + 1 if ax == 0 else nx):
            for j in range(ny + 1 if ax == 1 else ny):
                for k in range(nz + 1 if ax == 2 else nz):
                    lo = [i, j, k]
                    # cells on either side of the face at grid index lo along axis ax
                    c_lo = list(lo); c_lo[ax] -= 1
                    s_lo = S[c_lo[0] + 1, c_lo[1] + 1, c_lo[2] + 1]
                    s_hi = S[lo[0] + 1, lo[1] + 1, lo[2] + 1]
                    if s_lo == s_hi:
                        continue
                    u, w = [(1, 2), (2, 0), (0, 1)][ax]
                    p = []
                    for du, dw in ((0, 0), (1, 0), (1, 1), (0, 1)):
                        q = list(lo); q[u] += du; q[w] += dw
                        p.append(v(*q))
                    # (u,w,ax) is right-handed, so quad p0..p3 has normal +ax; flip if solid is on +ax side
                    if s_lo:       # solid below -> outward normal +ax
                        tris += [(p[0], p[1], p[2]), (p[0], p[2], p[3])]
                    else:
                        tris += [(p[0], p[2], p[1]), (p[0], p[3], p[2])]
    return np.asarray(verts, np.float64), np.asarray(tris, np.int32)


def box_surface(size, spacing=None, center=True):
    sx, sy, sz = size
    sp = spacing if spacing is not None else max(size) * 2
    xl, yl, zl = (_axis_lines([0.0, s], sp) for s in size)
    V, T = cell_union_surface(xl, yl, zl, np.ones((len(xl) - 1, len(yl) - 1, len(zl) - 1), bool))
    if center:
        V = V - np.array([sx, sy, sz]) / 2
    return V, T


def rot_z(theta):
    c, s = math.cos(theta), math.sin(theta)
    return np.array([[c, -s, 0.0], [s, c, 0.0], [0.0, 0.0, 1.0]])


def rot_y(theta):
    c, s = math.cos(theta), math.sin(theta)
    return np.array([[c, 0.0, s], [0.0, 1.0, 0.0], [-s, 0.0, c]])


def pose(t, R=None):
    R = np.eye(3) if R is None else np.asarray(R, np.float64)
    return np.r_[np.asarray(t, np.float64), R.ravel()]


def compose(y_parent, T_child):
    """Compose two 12-vector affine poses: x -> tp + Ap (tc + Ac x)."""
    tp, Ap = y_parent[:3], y_parent[3:].reshape(3, 3)
    tc, Ac = T_child[:3], T_child[3:].reshape(3, 3)
    return np.r_[tp + Ap @ tc, (Ap @ Ac).ravel()]


def apply_pose(y, X):
    return X @ y[3:].reshape(3, 3).T + y[:3]


def _pad_regions(nx, ny, nz):
    """Bottom face (k=0) is the attached region ∂⁻G, top face (k=nz-1) the coated region ∂⁺G."""
    ids = np.arange(nx * ny * nz).reshape(nz, ny, nx)
    return ids[0].ravel().astype(np.int32), ids[-1].ravel().astype(np.int32)


def _markers(nx, ny, nz, every=2):
    """Markers at the centroids-ish of top-face triangles on a regular sub-grid of ∂⁺G: each marker
    is a (tri of 3 top vertices, barycentric weights) with Σα=1, α∈[0,1]."""
    ids = np.arange(nx * ny * nz).reshape(nz, ny, nx)[-1]
    tri, bary = [], []
    for j in range(0, ny - 1, every):
        for i in range(0, nx - 1, every):
            tri.append([ids[j, i], ids[j, i + 1], ids[j + 1, i]])
            bary.append([0.5, 0.25, 0.25])
    return np.asarray(tri, np.int32), np.asarray(bary, np.float64)


def make_pad(nx, ny, nz, size, mount_body, mount_T, **mat):
    pos, tets = lattice_tets(nx, ny, nz, size)
    pos = pos - np.array([size[0] / 2, size[1] / 2, 0.0])      # pad frame: bottom face centred at 0
    att, coat = _pad_regions(nx, ny, nz)
    mt, mb = _markers(nx, ny, nz)
    return SoftPad(rest_pos=pos, tets=tets, mount_body=mount_body, mount_T=np.asarray(mount_T, np.float64),
                   attached=att, coated=coat, marker_tri=mt, marker_bary=mb, **mat)


# ----------------------------------------------------------------------------------------------
# configs
# ----------------------------------------------------------------------------------------------

MM = 1e-3


def scene_C1(variant="C1"):
    """C1: one 8x8x3 pad (21x21x4 mm) with its bottom attached to a static base;
    a kinematic 10 mm cube (8 v / 12 t) 0.2 mm above, yawed 7°, offset (0.37,-0.21) mm, whose
    target descends 0.12 mm/step for 10 steps (nominal press 1.0 mm).  dt = 0.01 s.
    C1b: the cube is dynamic and dropped from 1 mm.  C1c: a soft 5-tet-lattice cube on a static plate."""
    cfg = Config(dt=0.01)
    base_V, base_T = box_surface((30 * MM, 30 * MM, 5 * MM))
    base = AffineBody(base_V, base_T, kind=STATIC)
    if variant == "C1c":
        cube_pos, cube_tets = lattice_tets(4, 4, 4, (8 * MM, 8 * MM, 8 * MM))
        cube_pos = cube_pos - np.array([4 * MM, 4 * MM, 0.0])
        soft = SoftPad(rest_pos=cube_pos, tets=cube_tets, mount_body=-1,
                       mount_T=pose([0.3 * MM, -0.2 * MM, 2.5 * MM + 0.05 * MM]))
        return Scene("C1c", [soft], [base], np.array([0, 0, -9.81]), cfg, n_steps=10)
    pad = make_pad(8, 8, 3, (21 * MM, 21 * MM, 4 * MM), mount_body=0, mount_T=pose([0, 0, 2.5 * MM]))
    cube_V, cube_T = box_surface((10 * MM, 10 * MM, 10 * MM))
    kind = DYNAMIC if variant == "C1b" else KINEMATIC
    cube = AffineBody(cube_V, cube_T, kind=kind)
    return Scene(variant, [pad], [base, cube], np.array([0, 0, -9.81]), cfg, n_steps=10)


# Coulomb coefficient of the manipulation workloads C2-C5 (reading R23): the paper's E_IPC carries the lagged
# friction D_k and its peg insertion and grasps rely on it; μ itself is not given
# (P:L216 calibrates it per object), 0.5 is a typical gel-on-object value.  Without friction a squeezed peg or
# object has no tangential hold and slides out of the grasp within a step (measured: Newton tails of 100-400
# iterations on C2/C3).  C1 stays frictionless (its pins are the frictionless closed forms).
MU_MANIP = 0.5


def scene_C2(high_res=False):
    """C2/C3: two pads on two kinematic finger boxes (25x22x6 mm) squeezing a
    dynamic 12x12x60 mm square peg (~3 mm tessellation) that rests on the floor of a static blind
    hole (40x40x20 mm block, 12.6 mm square hole 15 mm deep, 0.3 mm clearance).  dt = 0.02 s, μ = MU_MANIP.
    Active-pair capacity (barrier + frozen friction pairs): C2 4096, C3 8192 (measured C3 maxima ≈ 2,800
    barrier pairs, about as many friction pairs)."""
    cfg = Config(dt=0.02, mu_friction=MU_MANIP, active_capacity_per_env=8192 if high_res else 4096)
    # static block with the hole; top face at z=0
    hw = 6.3 * MM
    xl = _axis_lines([-20 * MM, -hw, hw, 20 * MM], 3.5 * MM)
    yl = _axis_lines([-20 * MM, -hw, hw, 20 * MM], 3.5 * MM)
    zl = _axis_lines([-20 * MM, -15 * MM, 0.0], 5.0 * MM)
    solid = np.ones((len(xl) - 1, len(yl) - 1, len(zl) - 1), bool)
    xc, yc, zc = (xl[:-1] + xl[1:]) / 2, (yl[:-1] + yl[1:]) / 2, (zl[:-1] + zl[1:]) / 2
    solid &= ~((np.abs(xc)[:, None, None] < hw) & (np.abs(yc)[None, :, None] < hw) & (zc[None, None, :] > -15 * MM))
    hole_V, hole_T = cell_union_surface(xl, yl, zl, solid)
    hole = AffineBody(hole_V, hole_T, kind=STATIC)
    peg_V, peg_T = box_surface((12 * MM, 12 * MM, 60 * MM), spacing=3 * MM)
    peg = AffineBody(peg_V, peg_T, kind=DYNAMIC)
    fV, fT = box_surface((6 * MM, 22 * MM, 25 * MM))
    finger_l = AffineBody(fV, fT, kind=KINEMATIC)
    finger_r = AffineBody(fV.copy(), fT.copy(), kind=KINEMATIC)
    if high_res:
        lat, size = (19, 16, 5), (21 * MM, 17.5 * MM, 4 * MM)
    else:
        lat, size = (8, 6, 3), (21 * MM, 15 * MM, 4 * MM)
    # pad frame: z = thickness (bottom attached to finger inner face), x along world z, y along world y.
    # finger frame: centred box, inner face at +x (left finger) / -x (right finger).
    # left finger's inner face is at local x=+3 mm; pad frame maps pad-z -> +x, pad-x -> world z.
    R_l = np.array([[0.0, 0.0, 1.0], [0.0, 1.0, 0.0], [-1.0, 0.0, 0.0]])   # pad (x,y,z) -> finger (-z.. ) frame
    R_r = np.array([[0.0, 0.0, -1.0], [0.0, 1.0, 0.0], [1.0, 0.0, 0.0]])
    pad_l = make_pad(*lat, size, mount_body=2, mount_T=pose([3 * MM, 0, 0], R_l))
    pad_r = make_pad(*lat, size, mount_body=3, mount_T=pose([-3 * MM, 0, 0], R_r))
    name = "C3" if high_res else "C2"
    return Scene(name, [pad_l, pad_r], [hole, peg, finger_l, finger_r], np.array([0, 0, -9.81]), cfg,
                 n_steps=200)


def scene_pair(name: str) -> Scene:
    """Hand-placed single-pair scenes (geometry only; the expected values are derived by hand in
    tests/test_oracle_pins.py).  dt = 0.01 s, no gravity, gap h = d̂/2 (d̂ = 1e-4 m).
      P1: tet with vertices (0,0,0), (a,0,a), (−a/2, ±a√3/2, a), a = 2 mm (only the apex points down),
          above the top face of a static 30×30×5 mm box (box pose from env_inputs: the apex sits over
          box-frame point (7, 3) mm, away from the top face's diagonal) → one PT pair.
      P2: tet A with its ridge edge (±a,0,0) on top, tet B with its valley edge at angle θ at z = h
          on the bottom, a = b = 1 mm, θ = 90° → one EE pair (mollifier inactive).
      P2m: as P2 with a = b = 10 mm and sin θ = 0.02 → one EE pair with c/ε× = 1000 sin²θ = 0.4."""
    cfg = Config(dt=0.01)
    h = 0.5 * cfg.dhat
    tet = np.array([[0, 1, 2, 3]], np.int32)
    if name == "P1":
        a = 2 * MM
        X = np.array([[0, 0, 0], [a, 0, a], [-a / 2, a * math.sqrt(3) / 2, a], [-a / 2, -a * math.sqrt(3) / 2, a]])
        bV, bT = box_surface((30 * MM, 30 * MM, 5 * MM))
        return Scene(name, [SoftPad(rest_pos=X, tets=tet)], [AffineBody(bV, bT, kind=STATIC)], np.zeros(3), cfg, n_steps=1)
    if name in ("P2", "P2m"):
        a = b = (1 * MM if name == "P2" else 10 * MM)
        th = math.pi / 2 if name == "P2" else math.asin(0.02)
        c, s = math.cos(th), math.sin(th)
        XA = np.array([[-a, 0, 0], [a, 0, 0], [0, -a, -a], [0, a, -a]])
        XB = np.array([[-b * c, -b * s, h], [b * c, b * s, h], [b * s, -b * c, h + b], [-b * s, b * c, h + b]])
        return Scene(name, [SoftPad(rest_pos=XA, tets=tet), SoftPad(rest_pos=XB, tets=tet.copy())], [], np.zeros(3), cfg,
                     n_steps=1)
    raise ValueError(name)


def icosphere(level: int):
    """Unit icosphere: icosahedron subdivided `level` times, vertices projected to the sphere;
    outward-oriented triangles (level 3: 642 vertices / 1280 triangles)."""
    t = (1.0 + math.sqrt(5.0)) / 2.0
    V = [(-1, t, 0), (1, t, 0), (-1, -t, 0), (1, -t, 0), (0, -1, t), (0, 1, t), (0, -1, -t), (0, 1, -t),
         (t, 0, -1), (t, 0, 1), (-t, 0, -1), (-t, 0, 1)]
    V = [np.array(v, np.float64) / np.linalg.norm(v) for v in V]
    F = [(0, 11, 5), (0, 5, 1), (0, 1, 7), (0, 7, 10), (0, 10, 11), (1, 5, 9), (5, 11, 4), (11, 10, 2), (10, 7, 6),
         (7, 1, 8), (3, 9, 4), (3, 4, 2), (3, 2, 6), (3, 6, 8), (3, 8, 9), (4, 9, 5), (2, 4, 11), (6, 2, 10), (8, 6, 7),
         (9, 8, 1)]
    for _ in range(level):
        mid = {}

        def m(a, b):
            key = (min(a, b), max(a, b))
            if key not in mid:
                v = V[a] + V[b]
                V.append(v / np.linalg.norm(v))
                mid[key] = len(V) - 1
            return mid[key]
        F = [f for (a, b, c) in F for f in ((a, m(a, b), m(c, a)), (b, m(b, c), m(a, b)), (c, m(c, a), m(b, c)),
                                            (m(a, b), m(b, c), m(c, a)))]
    return np.array(V), np.array(F, np.int32)


def star_object(shape: int):
    """C4 object `shape` (0..7): a level-3 icosphere with radius R ~ U[20, 30] mm and a seeded low-order
    radial perturbation r(u) = R (1 + 0.15 h(u)), h a sum of quadratic/cubic ridge functions of u
    normalised to max |h| = 1 (star-shaped, smooth)."""
    rng = np.random.Generator(np.random.Philox(key=(SEED_BASE + CFG_INDEX["C4"]) * (1 << 32) + 1_000_000 + shape))
    U, F = icosphere(3)
    R = rng.uniform(20.0, 30.0) * MM
    h = np.zeros(len(U))
    for k in range(6):
        a = rng.normal(size=3)
        a /= np.linalg.norm(a)
        h += rng.uniform(-1, 1) * (U @ a) ** (2 + k % 2)
    h /= np.abs(h).max()
    return U * (R * (1.0 + 0.15 * h))[:, None], F


def scene_C4(shape: int = 0):
    """C4: parallel gripper — two 40x40x4 mm pads (14x14x3 lattice) on kinematic finger
    boxes (6x44x44 mm) squeeze star object `shape` (dynamic) standing on a static 200x200x20 mm table
    (top face at z = 0).  dt = 0.02 s, μ = MU_MANIP, active-pair capacity 8192."""
    cfg = Config(dt=0.02, mu_friction=MU_MANIP, active_capacity_per_env=8192)
    tV, tT = box_surface((200 * MM, 200 * MM, 20 * MM), spacing=25 * MM)
    table = AffineBody(tV, tT, kind=STATIC)
    oV, oT = star_object(shape)
    obj = AffineBody(oV, oT, kind=DYNAMIC)
    fV, fT = box_surface((6 * MM, 44 * MM, 44 * MM))
    R_l = np.array([[0.0, 0.0, 1.0], [0.0, 1.0, 0.0], [-1.0, 0.0, 0.0]])
    R_r = np.array([[0.0, 0.0, -1.0], [0.0, 1.0, 0.0], [1.0, 0.0, 0.0]])
    pad_l = make_pad(14, 14, 3, (40 * MM, 40 * MM, 4 * MM), mount_body=2, mount_T=pose([3 * MM, 0, 0], R_l))
    pad_r = make_pad(14, 14, 3, (40 * MM, 40 * MM, 4 * MM), mount_body=3, mount_T=pose([-3 * MM, 0, 0], R_r))
    return Scene(f"C4:{shape}", [pad_l, pad_r],
                 [table, obj, AffineBody(fV, fT, kind=KINEMATIC), AffineBody(fV.copy(), fT.copy(), kind=KINEMATIC)],
                 np.array([0, 0, -9.81]), cfg, n_steps=200)


# ---- C5: Allegro-like hand ------------------------------------------------------------------------
HAND_L = (20 * MM, 25 * MM, 20 * MM, 24 * MM)          # link lengths: proximal, 2 middle links, distal
HAND_FINGERS = ("thumb", "index", "middle", "ring")
HAND_APPROACH = {"thumb": (1.0, 0.0), "index": (-1.0, 0.0), "middle": (0.0, -1.0), "ring": (0.0, 1.0)}
TILE = (16 * MM, 30 * MM, 22 * MM)                     # x (between the engraved faces), y, z
HAND_PALM_HALF = 7.5 * MM                               # half the palm thickness (finger bases on its bottom face)
HAND_PAD_LIFT = 2.0 * MM                                # distal-link centre above the tile centre


def engraved_tile(seed_shape: int = 0):
    """The C5 tile: a 16x30x22 mm box whose two x-faces (30x22 mm) carry a seeded 0.3 mm-deep engraving
    on a 48x36 cell grid (random rectangles and a ring), as a watertight cell-union surface."""
    rng = np.random.Generator(np.random.Philox(key=(SEED_BASE + CFG_INDEX["C5"]) * (1 << 32) + 2_000_000 + seed_shape))
    hx, hy, hz = TILE[0] / 2, TILE[1] / 2, TILE[2] / 2
    d = 0.3 * MM
    xl = np.array([-hx, -hx + d, hx - d, hx])
    yl = np.linspace(-hy, hy, 49)
    zl = np.linspace(-hz, hz, 37)
    solid = np.ones((3, 48, 36), bool)
    yc, zc = (yl[:-1] + yl[1:]) / 2, (zl[:-1] + zl[1:]) / 2
    for side in (0, 2):
        eng = np.zeros((48, 36), bool)
        for _ in range(6):                              # random grooves/pockets, away from the rim
            j0, k0 = rng.integers(2, 40), rng.integers(2, 28)
            eng[j0:j0 + rng.integers(2, 7), k0:k0 + rng.integers(2, 7)] = True
        r = np.hypot(yc[:, None] - rng.uniform(-5, 5) * MM, zc[None, :] - rng.uniform(-3, 3) * MM)
        eng |= (r > 4.0 * MM) & (r < 5.2 * MM)         # a ring
        eng[:2, :] = eng[-2:, :] = False
        eng[:, :2] = eng[:, -2:] = False
        solid[side] = ~eng
    return cell_union_surface(xl, yl, zl, solid)


def _rx(t):
    c, s = math.cos(t), math.sin(t)
    return np.array([[1.0, 0, 0], [0, c, -s], [0, s, c]])


def hand_base_frames():
    """Per finger: the base frame of its chain in the palm frame (x = approach direction toward the
    tile, z = up), placed so that with zero joint angles the distal link hangs straight down with its
    pad's coated face 0.2 mm from the tile face, the pad centre level with the tile centre."""
    L0, L1, L2, L3 = HAND_L
    out = {}
    for f in HAND_FINGERS:
        ax, ay = HAND_APPROACH[f]
        R = np.array([[ax, -ay, 0.0], [ay, ax, 0.0], [0.0, 0.0, 1.0]])      # columns: x_l = a, y_l, z_l = up
        face = TILE[0] / 2 if ay == 0 else TILE[1] / 2
        dist = face + 0.2 * MM + 3 * MM + 4 * MM        # tile face, gap, pad thickness, half the distal link
        c_distal = -dist * np.array([ax, ay, 0.0])      # horizontal offset from the palm centre
        base = c_distal + np.array([0, 0, -HAND_PALM_HALF])   # on the palm's bottom face
        out[f] = (base, R)
    return out


def fk_hand(y_palm, q):
    """Forward kinematics (homogeneous products) of the 4 fingers: q (4, 4) joint angles per finger
    (abduction about the base's z, then three flexions about the local y; positive flexion moves the
    finger tip toward the tile).  Returns the 16 link body poses (12-vectors, world), finger-major:
    proximal, middle, middle-2, distal; each link's body frame is the centre of its segment."""
    L = HAND_L
    out = []
    for fi, f in enumerate(HAND_FINGERS):
        base, Rb = hand_base_frames()[f]
        T = compose(y_palm, pose(base, Rb))
        T = compose(T, pose([0, 0, 0], rot_z(q[fi, 0])))
        for j in range(4):
            if j > 0:
                T = compose(T, pose([0, 0, -L[j - 1]], rot_y(-q[fi, j])))
            out.append(compose(T, pose([0, 0, -L[j] / 2])))
    return np.stack(out)


def hand_chain():
    """The C5 hand as a kinematic tree (input description for tac_set_chain, include/taccel.h): link 0 the
    palm (fixed to the base pose), then per finger proximal (abduction about z), two middle links and the
    distal link (flexions about −y), each driving its kinematic body; same geometry as fk_hand."""
    L = HAND_L
    ident = pose([0, 0, 0])
    parent, origin, axis, joint, body, kin = [-1], [ident], [np.array([0.0, 0.0, 1.0])], [-1], [ident], [2]
    frames = hand_base_frames()
    for fi, f in enumerate(HAND_FINGERS):
        base, Rb = frames[f]
        for j in range(4):
            parent.append(0 if j == 0 else len(parent) - 1)
            origin.append(pose(base, Rb) if j == 0 else pose([0, 0, -L[j - 1]]))
            axis.append(np.array([0.0, 0.0, 1.0]) if j == 0 else np.array([0.0, -1.0, 0.0]))
            joint.append(4 * fi + j)
            body.append(pose([0, 0, -L[j] / 2]))
            kin.append(3 + 4 * fi + j)
    return {"parent": np.array(parent), "origin": np.stack(origin), "axis": np.stack(axis), "joint": np.array(joint),
            "body": np.stack(body), "kin_body": np.array(kin), "n_joints": 16}


def scene_C5():
    """C5: Allegro-like hand — palm (60x60x15 mm) and 4 fingers of 4 kinematic link boxes,
    four fingertip pads (24x24x3 mm, 9x9x4 lattice) on the distal links' inner faces, a dynamic engraved
    tile (16x30x22 mm) standing on a static table.  Bodies: table, tile, palm, 16 links.  dt = 0.02 s."""
    # μ = MU_MANIP; the engraved faces under four pads: measured 8,505 barrier + 3,783 friction pairs in one
    # env at step 5 (the pads' 2.7 mm edges against the tile's 0.6 mm engraving cells) -> capacity 24576
    cfg = Config(dt=0.02, mu_friction=MU_MANIP, active_capacity_per_env=24576)
    tV, tT = box_surface((200 * MM, 200 * MM, 20 * MM), spacing=25 * MM)
    tileV, tileT = engraved_tile()
    pV, pT = box_surface((60 * MM, 60 * MM, 15 * MM))
    bodies = [AffineBody(tV, tT, kind=STATIC), AffineBody(tileV, tileT, kind=DYNAMIC), AffineBody(pV, pT, kind=KINEMATIC)]
    L = HAND_L
    pads = []
    R_pad = np.array([[0.0, 0.0, 1.0], [0.0, 1.0, 0.0], [-1.0, 0.0, 0.0]])   # pad z → link x (toward the tile)
    for fi, f in enumerate(HAND_FINGERS):
        for j in range(4):
            size = (8 * MM, 24 * MM, L[j]) if j == 3 else (8 * MM, 12 * MM, L[j] - 1 * MM)
            V, T = box_surface(size)
            bodies.append(AffineBody(V, T, kind=KINEMATIC))
        pads.append(make_pad(9, 9, 4, (24 * MM, 24 * MM, 3 * MM), mount_body=3 + 4 * fi + 3,
                             mount_T=pose([4 * MM, 0, 0], R_pad)))
    return Scene("C5", pads, bodies, np.array([0, 0, -9.81]), cfg, n_steps=200)


def hand_palm_pose():
    """Palm pose: with zero joint angles the distal links (and their pads) are centred HAND_PAD_LIFT above
    the tile centre, so the 24 mm pads clear the table top and overhang the 22 mm tile at its top."""
    L0, L1, L2, L3 = HAND_L
    return pose([0, 0, TILE[2] / 2 + 0.08 * MM + HAND_PAD_LIFT + L3 / 2 + L2 + L1 + L0 + HAND_PALM_HALF])


def hand_script(env_id: int, n_steps: int):
    """C5 joint script (16 joints): steps 0-79 each finger closes its pad onto the tile by τ_d ~ U[0.5, 1.5]
    mm (per pad) with the parallelogram flexion q1 = a, q2 = −a, q3 = 0 (the tip translates by L1 sin a,
    the pad stays parallel to the face); steps 80-199 the abduction joints oscillate ±2° together."""
    rng = env_rng("C5", env_id)
    tau = rng.uniform(0.5, 1.5, 4) * MM
    L1 = HAND_L[1]
    qs = []
    for k in range(n_steps):
        q = np.zeros((4, 4))
        for fi in range(4):
            reach = (0.2 * MM + tau[fi]) * min(k + 1, 80) / 80.0
            a = math.asin(reach / L1)
            q[fi, 1], q[fi, 2] = a, -a
            if k >= 80:
                q[fi, 0] = math.radians(2.0) * math.sin(2 * math.pi * (k + 1 - 80) / 120.0)
        qs.append(q)
    return np.stack(qs)


def _c5_env(scene, env_id, n_steps):
    y_palm = hand_palm_pose()
    y_table = pose([0, 0, -10 * MM])
    y_tile = pose([0, 0, TILE[2] / 2 + 0.08 * MM])
    links0 = fk_hand(y_palm, np.zeros((4, 4)))
    y0 = np.concatenate([np.stack([y_table, y_tile, y_palm]), links0])
    qs = hand_script(env_id, n_steps)
    tk = np.stack([np.concatenate([y_palm[None], fk_hand(y_palm, q)]) for q in qs])
    return y0, tk


def make_scene(name: str) -> Scene:
    if name == "C5":
        return scene_C5()
    if name == "C4" or name.startswith("C4:"):
        return scene_C4(int(name.split(":")[1]) if ":" in name else 0)
    if name in ("P1", "P2", "P2m"):
        return scene_pair(name)
    if name in ("C1", "C1b", "C1c"):
        return scene_C1(name)
    if name == "C2":
        return scene_C2(False)
    if name == "C3":
        return scene_C2(True)
    raise ValueError(f"unknown scene {name}")


# ----------------------------------------------------------------------------------------------
# per-env seeded inputs
# ----------------------------------------------------------------------------------------------

def env_rng(name: str, env_id: int) -> np.random.Generator:
    key = (SEED_BASE + CFG_INDEX[name.split(":")[0]]) * (1 << 32) + int(env_id)
    return np.random.Generator(np.random.Philox(key=key))


@dataclasses.dataclass
class EnvInputs:
    x0: np.ndarray        # (E, V, 3) initial soft vertex world positions
    y0: np.ndarray        # (E, NA, 12) initial affine states (all bodies, static included)
    ykin: np.ndarray      # (S, E, NK, 12) per-step kinematic targets s^y


def _soft_world(scene: Scene, y0: np.ndarray, jitter: Optional[np.random.Generator] = None):
    xs = []
    for pad in scene.soft:
        if pad.mount_body >= 0:
            yp = compose(y0[pad.mount_body], pad.mount_T)
        else:
            yp = pad.mount_T
        xs.append(apply_pose(yp, pad.rest_pos))
    return np.concatenate(xs, 0)


def _c1_env(scene, env_id, n_steps):
    rng = env_rng(scene.name, env_id)
    if env_id == 0:
        yaw, off, gap, rate = 7.0, (0.37 * MM, -0.21 * MM), 0.2 * MM, 0.12 * MM
    else:
        yaw = rng.uniform(3.0, 11.0)
        off = tuple(rng.uniform(-1.0, 1.0, 2) * MM)
        gap = rng.uniform(0.15, 0.25) * MM
        rate = rng.uniform(0.08, 0.14) * MM
    pad_top = 2.5 * MM + 4 * MM
    y_base = pose([0, 0, 0])
    if scene.name == "C1c":
        y0 = np.stack([y_base])
        return y0, np.zeros((n_steps, 0, 12))
    if scene.name == "C1b":
        gap = 1.0 * MM
    cube_y = pose([off[0], off[1], pad_top + gap + 5 * MM], rot_z(math.radians(yaw)))
    y0 = np.stack([y_base, cube_y])
    if scene.name == "C1b":
        return y0, np.zeros((n_steps, 0, 12))
    tk = []
    for s in range(n_steps):
        yt = cube_y.copy()
        yt[2] -= rate * (s + 1)
        tk.append(yt[None])
    return y0, np.stack(tk)


def _c2_env(scene, env_id, n_steps):
    rng = env_rng(scene.name, env_id)
    dx, dy = rng.uniform(-0.1, 0.1, 2) * MM
    yaw0 = math.radians(rng.uniform(-0.5, 0.5))
    tau_d = rng.uniform(0.5, 1.5) * MM
    A_x = rng.uniform(0.5, 1.5) * MM
    A_th = math.radians(rng.uniform(1.0, 2.0))
    # static hole at origin (top face z=0); peg (centre frame) resting 0.08 mm above the floor
    y_hole = pose([0, 0, 0])
    y_peg = pose([dx, dy, -15 * MM + 0.08 * MM + 30 * MM], rot_z(yaw0))
    grip_z = 32 * MM
    pad_th = 4 * MM
    gap0 = 0.2 * MM
    # finger centre x so that the pad surface is gap0 away from the peg face (|x| = 6 mm)
    fx = 6 * MM + gap0 + pad_th + 3 * MM
    y_fl = pose([-fx + dx, dy, grip_z])
    y_fr = pose([fx + dx, dy, grip_z])
    y0 = np.stack([y_hole, y_peg, y_fl, y_fr])
    close = 40
    tk = []
    for k in range(n_steps):
        if k < close:
            sq = (gap0 + tau_d) * (k + 1) / close
            ox, th = 0.0, 0.0
        else:
            sq = gap0 + tau_d
            ox = A_x * math.sin(2 * math.pi * 2 * (k + 1 - close) / 160.0)
            th = A_th * math.sin(2 * math.pi * (k + 1 - close) / 160.0)
        R = rot_z(th)
        c = np.array([dx + ox, dy, grip_z])
        yl = pose(c + R @ np.array([-fx + sq, 0, 0]), R)
        yr = pose(c + R @ np.array([fx - sq, 0, 0]), R)
        tk.append(np.stack([yl, yr]))
    return y0, np.stack(tk)


def _c4_env(scene, env_id, n_steps):
    """C4 per-env script: gripper yaw θ ~ U[0, 2π) about the object's vertical axis, press τ_d ~ U[0.5, 1.5]
    mm, wiggle amplitude A_x ~ U[0.5, 1.5] mm.  Steps 0-59 close from a 0.2 mm gap to τ_d; steps 60-199 the
    closed gripper oscillates along its squeeze axis, x = A_x sin(2π·2(k−60)/140)."""
    rng = env_rng(scene.name, env_id)
    th = rng.uniform(0.0, 2.0 * math.pi)
    tau_d = rng.uniform(0.5, 1.5) * MM
    A_x = rng.uniform(0.5, 1.5) * MM
    oV = scene.affine[1].rest_pos
    zc = -oV[:, 2].min() + 0.08 * MM                        # object's lowest vertex 0.08 mm above the table
    R = rot_z(th)
    dirv = R @ np.array([1.0, 0.0, 0.0])
    s_pos, s_neg = (oV @ dirv).max(), (-(oV @ dirv)).max()    # support distances along ±squeeze axis
    pad_th, gap0, half = 4 * MM, 0.2 * MM, 3 * MM
    y_table = pose([0, 0, -10 * MM])
    y_obj = pose([0, 0, zc])
    c = np.array([0.0, 0.0, zc])
    fl = -(s_neg + gap0 + pad_th + half)
    fr = s_pos + gap0 + pad_th + half
    y0 = np.stack([y_table, y_obj, pose(c + R @ np.array([fl, 0, 0]), R), pose(c + R @ np.array([fr, 0, 0]), R)])
    close = 60
    tk = []
    for k in range(n_steps):
        if k < close:
            sq, ox = (gap0 + tau_d) * (k + 1) / close, 0.0
        else:
            sq, ox = gap0 + tau_d, A_x * math.sin(2 * math.pi * 2 * (k + 1 - close) / 140.0)
        cc = c + R @ np.array([ox, 0.0, 0.0])
        tk.append(np.stack([pose(cc + R @ np.array([fl + sq, 0, 0]), R), pose(cc + R @ np.array([fr - sq, 0, 0]), R)]))
    return y0, np.stack(tk)


def env_inputs(scene: Scene, env_ids, n_steps: Optional[int] = None) -> EnvInputs:
    """Initial states (zero velocities) and per-step kinematic targets for the given global
    env ids.  Deterministic per env id."""
    n_steps = scene.n_steps if n_steps is None else n_steps
    ys, tks, xs = [], [], []
    for e in env_ids:
        if scene.name.startswith("P"):
            y0 = np.stack([pose([-7 * MM, -3 * MM, -0.5 * scene.config.dhat - 2.5 * MM])]) if scene.affine else np.zeros((0, 12))
            y0, tk = y0, np.zeros((n_steps, 0, 12))
        elif scene.name.startswith("C1"):
            y0, tk = _c1_env(scene, int(e), n_steps)
        elif scene.name.startswith("C4"):
            y0, tk = _c4_env(scene, int(e), n_steps)
        elif scene.name == "C5":
            y0, tk = _c5_env(scene, int(e), n_steps)
        else:
            y0, tk = _c2_env(scene, int(e), n_steps)
        ys.append(y0)
        tks.append(tk)
        xs.append(_soft_world(scene, y0))
    ykin = np.stack(tks, 1) if len(tks) else np.zeros((n_steps, 0, 0, 12))
    return EnvInputs(x0=np.stack(xs), y0=np.stack(ys), ykin=ykin)
