"""Oracle forward kinematics (test infrastructure only — see oracle/__init__.py).

Robot links are affine bodies driven by kinematic targets computed from joint targets (P:L147-157:
"the robot is a kinematic tree of links... actions are converted to kinematic constraints").  The chain
semantics are those of include/taccel.h tac_chain_desc, written here with plain 4×4 homogeneous
matrices: J_i = J_parent · H(origin_i) · H(Rot(axis_i, q_j)), body target J_i · H(body_i), with the
rotation matrix of an axis-angle pair exp(θ[a]×) evaluated by scipy's matrix exponential (not the
Rodrigues closed form the CUDA kernel uses)."""
from __future__ import annotations

import numpy as np
import scipy.linalg as sla


def hom(y):
    """4×4 homogeneous matrix of a 12-vector pose (t, R row-major)."""
    H = np.eye(4)
    H[:3, 3] = y[:3]
    H[:3, :3] = np.asarray(y[3:], np.float64).reshape(3, 3)
    return H


def pose_of(H):
    return np.r_[H[:3, 3], H[:3, :3].ravel()]


def axis_angle(a, th):
    """Rotation by θ about the unit axis a: exp(θ [a]×)."""
    K = np.array([[0.0, -a[2], a[1]], [a[2], 0.0, -a[0]], [-a[1], a[0], 0.0]])
    H = np.eye(4)
    H[:3, :3] = sla.expm(th * K)
    return H


def forward(chain, base, q):
    """Body targets (n_links, 12) of one env: base pose (12,), joint values q (n_joints,)."""
    n = len(chain["parent"])
    J = [None] * n
    out = np.zeros((n, 12))
    for i in range(n):
        p = chain["parent"][i]
        Hp = hom(base) if p < 0 else J[p]
        Hi = Hp @ hom(chain["origin"][i])
        if chain["joint"][i] >= 0:
            Hi = Hi @ axis_angle(chain["axis"][i], q[chain["joint"][i]])
        J[i] = Hi
        out[i] = pose_of(Hi @ hom(chain["body"][i]))
    return out
