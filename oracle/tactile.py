"""Oracle depth and normal maps of the coated surface (test infrastructure only — see oracle/__init__.py).

P:L163-165: "we extract the depth and normal maps d(u,v), n(u,v) for pixel coordinates (u,v) from the
deformed coated surface ∂⁺G̃".  The camera model is silent; reading R22 (include/taccel.h
tac_get_depth_maps): an orthographic camera in the pad's sensor frame looking along −z; pixel (i, j) of an
H×W map samples (x₀ + j(x₁−x₀)/(W−1), y₀ + i(y₁−y₀)/(H−1)) over the rest extent of the pad's coated
vertices; a coated triangle (surface triangle with three coated vertices) covers a pixel when its
barycentric coordinates in the deformed xy projection are all ≥ −1e-9; depth = z_ref − z (largest over
covering triangles; z_ref = max rest z of the coated vertices), normal = normalised sum of the covering
triangles' area vectors oriented +z; uncovered → NaN depth, zero normal.  Written per pixel and per
triangle, in plain loops over numpy arrays."""
from __future__ import annotations

import numpy as np

from .mesh import Model
from .readout import gel_deformation


def coated_triangles(model: Model, pad: int):
    """Surface triangles of pad `pad` whose three vertices are coated, in canonical surface order, as
    indices into the pad's coated-vertex list."""
    sc = model.scene
    off = sum(p.rest_pos.shape[0] for p in sc.soft[:pad])
    coat = [off + int(c) for c in sc.soft[pad].coated]
    where = {v: i for i, v in enumerate(coat)}
    out = []
    for t in model.tris:
        if all(int(v) in where for v in t):
            out.append([where[int(v)] for v in t])
    return np.asarray(out, np.int64).reshape(-1, 3), coat


def depth_maps(model: Model, x, y, H: int, W: int):
    """(depth [pads, H, W], normal [pads, H, W, 3]) of one env at (x, y)."""
    sc = model.scene
    disp = gel_deformation(model, x, y)                    # per pad: (coated displacements, markers...)
    D = np.full((len(sc.soft), H, W), np.nan)
    N = np.zeros((len(sc.soft), H, W, 3))
    for p, pad in enumerate(sc.soft):
        tris, coat = coated_triangles(model, p)
        Xr = pad.rest_pos[np.asarray(pad.coated)]
        X = Xr + disp[p][0]                                 # deformed coated vertices, sensor frame
        x0, x1, y0, y1, zref = Xr[:, 0].min(), Xr[:, 0].max(), Xr[:, 1].min(), Xr[:, 1].max(), Xr[:, 2].max()
        for i in range(H):
            for j in range(W):
                cx, cy = x0 + j * (x1 - x0) / (W - 1), y0 + i * (y1 - y0) / (H - 1)
                best, nsum, hit = -np.inf, np.zeros(3), False
                for a, b, c in tris:
                    A, B, C = X[a], X[b], X[c]
                    ar = (B[0] - A[0]) * (C[1] - A[1]) - (B[1] - A[1]) * (C[0] - A[0])
                    if ar == 0.0:
                        continue
                    wa = ((B[0] - cx) * (C[1] - cy) - (B[1] - cy) * (C[0] - cx)) / ar
                    wb = ((C[0] - cx) * (A[1] - cy) - (C[1] - cy) * (A[0] - cx)) / ar
                    wc = ((A[0] - cx) * (B[1] - cy) - (A[1] - cy) * (B[0] - cx)) / ar
                    if min(wa, wb, wc) < -1e-9:
                        continue
                    hit = True
                    best = max(best, zref - (wa * A[2] + wb * B[2] + wc * C[2]))
                    av = np.cross(B - A, C - A)
                    nsum += av if av[2] >= 0 else -av
                if hit:
                    D[p, i, j] = best
                    n = np.linalg.norm(nsum)
                    N[p, i, j] = nsum / n if n > 0 else 0.0
    return D, N
