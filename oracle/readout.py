"""Oracle tactile readout (test infrastructure only — see oracle/__init__.py).

P:L153: a gel pad G_i is attached to link l_j through ^{l_j}_{G_i}T; markers are
barycentric points p̃ = Σ α_u x̃_u of coated-surface triangles and the marker flow is ΔP = p̃ − p.
Reading R18: displacements are reported in the pad (sensor) frame using the link's
CURRENT affine state:  δ_v = R_mᵀ(A_l⁻¹(x_v − t_l) − t_m) − X_v  with mount_T = (t_m, R_m) and
X_v the rest position in the pad frame; marker world position p̃ = Σ α_u x_u and flow
Δp = Σ α_u δ_u (which equals p̃ − p expressed in the sensor frame).
"""
from __future__ import annotations

import numpy as np

from .mesh import Model


def pad_frame(model: Model, pad_index: int, y):
    pad = model.scene.soft[pad_index]
    tm = np.asarray(pad.mount_T[:3], np.float64)
    Rm = np.asarray(pad.mount_T[3:], np.float64).reshape(3, 3)
    if pad.mount_body >= 0:
        tl = y[pad.mount_body, :3]
        Al = y[pad.mount_body, 3:].reshape(3, 3)
    else:
        tl, Al = np.zeros(3), np.eye(3)
    return tl, Al, tm, Rm


def gel_deformation(model: Model, x, y):
    """Per pad: coated-vertex displacement δ (NC,3) in the sensor frame, marker world positions
    (NM,3) and marker flows (NM,3)."""
    out = []
    off = 0
    for pi, pad in enumerate(model.scene.soft):
        nv = len(pad.rest_pos)
        tl, Al, tm, Rm = pad_frame(model, pi, y)
        xs = x[off:off + nv]
        local = np.linalg.solve(Al, (xs - tl).T).T                    # A_l⁻¹(x − t_l)
        delta = (local - tm) @ Rm - np.asarray(pad.rest_pos, np.float64)   # R_mᵀ(· − t_m) − X
        coated = delta[np.asarray(pad.coated, np.int64)]
        mt = np.asarray(pad.marker_tri, np.int64)
        mb = np.asarray(pad.marker_bary, np.float64)
        mpos = (mb[:, :, None] * xs[mt]).sum(1)
        mflow = (mb[:, :, None] * delta[mt]).sum(1)
        out.append((coated, mpos, mflow))
        off += nv
    return out
