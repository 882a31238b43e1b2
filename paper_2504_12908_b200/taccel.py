"""Thin ctypes binding of libtaccel_cuda.so (include/taccel.h) — argument marshalling only.

Every step of the method runs in the CUDA library; this module only converts the seeded scene
description (``paper_2504_12908_b200.scenes.Scene``) into the C descriptors, owns the device
workspace (a torch uint8 tensor) and passes tensor pointers.  There is no CPU fallback: if the
shared library is missing or CUDA is unavailable, constructing a Batch raises.
"""
from __future__ import annotations

import ctypes
import os
import re
from typing import Optional

import numpy as np
import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libtaccel_cuda.so")
HEADER = os.path.join(os.path.dirname(_HERE), "include", "taccel.h")

c_double_p = ctypes.POINTER(ctypes.c_double)
c_int_p = ctypes.POINTER(ctypes.c_int32)

STATUS = {0: "TAC_OK", 1: "TAC_E_INVALID", 2: "TAC_E_VALIDATION", 3: "TAC_E_ENV_FAILED", 4: "TAC_E_CAPACITY",
          5: "TAC_E_WORKSPACE", 6: "TAC_E_CUDA"}
ENV_STATUS = {0: "OK", 1: "NEWTON_STALL", 2: "AL_INFEASIBLE", 3: "CAPACITY", 4: "NONFINITE", 5: "BAD_STATE",
              6: "DISABLED"}


class SoftDesc(ctypes.Structure):
    _fields_ = [("n_verts", ctypes.c_int32), ("n_tets", ctypes.c_int32), ("rest_pos", c_double_p), ("tets", c_int_p),
                ("youngs", ctypes.c_double), ("poisson", ctypes.c_double), ("density", ctypes.c_double),
                ("mount_body", ctypes.c_int32), ("mount_T", ctypes.c_double * 12),
                ("n_attached", ctypes.c_int32), ("attached", c_int_p), ("n_coated", ctypes.c_int32),
                ("coated", c_int_p), ("n_markers", ctypes.c_int32), ("marker_tri", c_int_p),
                ("marker_bary", c_double_p)]


class AffineDesc(ctypes.Structure):
    _fields_ = [("n_verts", ctypes.c_int32), ("n_tris", ctypes.c_int32), ("rest_pos", c_double_p), ("tris", c_int_p),
                ("kind", ctypes.c_int32), ("density", ctypes.c_double), ("kappa_s", ctypes.c_double)]


class SceneDesc(ctypes.Structure):
    _fields_ = [("n_soft", ctypes.c_int32), ("n_affine", ctypes.c_int32), ("soft", ctypes.POINTER(SoftDesc)),
                ("affine", ctypes.POINTER(AffineDesc)), ("collide", ctypes.POINTER(ctypes.c_uint8)),
                ("gravity", ctypes.c_double * 3)]


class Config(ctypes.Structure):
    _fields_ = [("dt", ctypes.c_double), ("dhat", ctypes.c_double), ("kappa", ctypes.c_double),
                ("max_step_rel", ctypes.c_double),
                ("newton_tol_rel", ctypes.c_double), ("al_tol_rel", ctypes.c_double), ("pcg_eta", ctypes.c_double),
                ("armijo_c", ctypes.c_double), ("accd_s", ctypes.c_double), ("al_rho0", ctypes.c_double),
                ("max_newton", ctypes.c_int32), ("max_al_rounds", ctypes.c_int32), ("max_pcg", ctypes.c_int32),
                ("max_accd_iters", ctypes.c_int32), ("ee_mollifier", ctypes.c_int32),
                ("hessian_mode", ctypes.c_int32), ("ls_expand", ctypes.c_int32),
                ("hold_cap", ctypes.c_int32), ("lm_mu0", ctypes.c_double), ("bp_margin", ctypes.c_double),
                ("cand_capacity_per_env", ctypes.c_int32), ("active_capacity_per_env", ctypes.c_int32),
                ("mu_friction", ctypes.c_double), ("eps_v", ctypes.c_double),
                ("pcg_eta_max", ctypes.c_double)]


class EnvStats(ctypes.Structure):
    _fields_ = [("status", ctypes.c_int32), ("newton_iters", ctypes.c_int32), ("pcg_iters", ctypes.c_int32),
                ("ls_backtracks", ctypes.c_int32), ("n_active", ctypes.c_int32), ("al_rounds", ctypes.c_int32),
                ("n_candidates", ctypes.c_int32), ("alpha_min", ctypes.c_double), ("energy", ctypes.c_double),
                ("constraint_residual", ctypes.c_double), ("pcg_iters_total", ctypes.c_int64),
                ("pcg_alg_bytes_total", ctypes.c_double), ("diag", ctypes.c_double * 4),
                ("min_dist", ctypes.c_double), ("n_residual", ctypes.c_int32), ("n_couplings", ctypes.c_int32),
                ("lm_mu", ctypes.c_double), ("n_friction", ctypes.c_int32), ("capacity_flags", ctypes.c_int32)]


class ChainDesc(ctypes.Structure):
    _fields_ = [("n_links", ctypes.c_int32), ("n_joints", ctypes.c_int32), ("parent", c_int_p), ("origin", c_double_p),
                ("axis", c_double_p), ("joint", c_int_p), ("body", c_double_p), ("kin_body", c_int_p)]


def header_symbols():
    """Function names declared in include/taccel.h."""
    txt = open(HEADER).read()
    return sorted(set(re.findall(r"\b(tac_\w+)\s*\(", txt)))


_lib = None


def load():
    """Load libtaccel_cuda.so (raises if it was not built — there is no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"{LIB_PATH} is missing: run __graft_entry__.build() (nvcc, sm_100a)")
        lib = ctypes.CDLL(LIB_PATH)
        vp = ctypes.c_void_p
        sig = {
            "tac_workspace_size": [ctypes.POINTER(SceneDesc), ctypes.c_int32, ctypes.POINTER(Config), ctypes.POINTER(ctypes.c_size_t)],
            "tac_batch_create": [ctypes.POINTER(SceneDesc), ctypes.c_int32, ctypes.POINTER(Config), ctypes.c_int32, vp,
                                 ctypes.c_size_t, vp, ctypes.POINTER(vp)],
            "tac_batch_destroy": [vp],
            "tac_batch_dims": [vp, c_int_p],
            "tac_set_state": [vp, ctypes.c_int32, ctypes.c_int32, vp, vp, vp, vp, vp, vp],
            "tac_set_targets": [vp, ctypes.c_int32, ctypes.c_int32, vp, vp],
            "tac_step": [vp, ctypes.c_int32, vp, vp],
            "tac_step_schedule": [vp, ctypes.c_int32, vp, vp, vp, vp, vp, vp],
            "tac_get_state": [vp, ctypes.c_int32, ctypes.c_int32, vp, vp, vp, vp, vp],
            "tac_get_gel_deformation": [vp, ctypes.c_int32, ctypes.c_int32, vp, vp, vp, vp],
            "tac_get_stats": [vp, ctypes.POINTER(EnvStats), vp],
            "tac_debug_eval": [vp, ctypes.c_int32, vp, vp, vp, vp, ctypes.c_double, ctypes.c_int32, vp, vp, vp, vp, vp],
            "tac_debug_active_pairs": [vp, ctypes.c_int32, vp, vp, vp, ctypes.c_int32, c_int_p, vp],
            "tac_debug_candidates": [vp, ctypes.c_int32, vp, vp, vp, vp, ctypes.c_int32, c_int_p, vp],
            "tac_debug_accd": [vp, ctypes.c_int32, vp, vp, vp, c_double_p, vp],
            "tac_debug_pcg": [vp, ctypes.c_int32, vp, vp, ctypes.c_int32, ctypes.c_double, vp, c_int_p, c_double_p, vp],
            "tac_debug_inject_fault": [vp, ctypes.c_int32, ctypes.c_int32, vp],
            "tac_set_chain": [vp, ctypes.POINTER(ChainDesc)],
            "tac_set_joint_targets": [vp, ctypes.c_int32, ctypes.c_int32, vp, vp, vp],
            "tac_get_targets": [vp, ctypes.c_int32, ctypes.c_int32, vp, vp],
            "tac_debug_trace": [vp, ctypes.c_int32, ctypes.c_int32, vp, c_int_p],
            "tac_get_depth_maps": [vp, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32, vp, vp, vp],
            "tac_profile_enable": [vp, ctypes.c_int32],
            "tac_profile_read": [vp, c_double_p, ctypes.POINTER(ctypes.c_int64), ctypes.c_int32],
            "tac_profile_iterations": [vp, c_int_p, c_double_p, ctypes.c_int32, c_int_p],
        }
        for name, args in sig.items():
            f = getattr(lib, name)
            f.argtypes = args
            f.restype = ctypes.c_int
        lib.tac_last_error.restype = ctypes.c_char_p
        lib.tac_profile_phase_name.restype = ctypes.c_char_p
        lib.tac_pcg_kernel_name.restype = ctypes.c_char_p
        lib.tac_pcg_kernel_name.argtypes = [vp]
        lib.tac_profile_phase_name.argtypes = [ctypes.c_int32]
        _lib = lib
    return _lib


class TaccelError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"{STATUS.get(code, code)}: {msg}")
        self.code = code


def _check(code):
    if code != 0:
        raise TaccelError(code, load().tac_last_error().decode())


def _ptr(a):
    if a is None:
        return None
    if isinstance(a, torch.Tensor):
        return ctypes.c_void_p(a.data_ptr())
    return a.ctypes.data_as(ctypes.c_void_p)


def _f64(a):
    if isinstance(a, torch.Tensor):
        assert a.dtype == torch.float64 and a.is_contiguous()
        return a
    return np.ascontiguousarray(a, dtype=np.float64)


def make_config(cfg) -> Config:
    c = Config()
    for name, _ in Config._fields_:
        setattr(c, name, getattr(cfg, name))
    return c


class _Descs:
    """Keeps the numpy arrays behind the C descriptors alive."""

    def __init__(self, scene):
        self.keep = []
        softs = (SoftDesc * max(1, len(scene.soft)))()
        for i, pad in enumerate(scene.soft):
            s = softs[i]
            rp = self._d(pad.rest_pos)
            tt = self._i(pad.tets)
            s.n_verts, s.n_tets = rp.shape[0], tt.shape[0]
            s.rest_pos, s.tets = rp.ctypes.data_as(c_double_p), tt.ctypes.data_as(c_int_p)
            s.youngs, s.poisson, s.density = pad.youngs, pad.poisson, pad.density
            s.mount_body = pad.mount_body
            for k in range(12):
                s.mount_T[k] = float(pad.mount_T[k])
            att, coat = self._i(pad.attached), self._i(pad.coated)
            mt, mb = self._i(pad.marker_tri), self._d(pad.marker_bary)
            s.n_attached, s.attached = len(att), att.ctypes.data_as(c_int_p)
            s.n_coated, s.coated = len(coat), coat.ctypes.data_as(c_int_p)
            s.n_markers, s.marker_tri, s.marker_bary = len(mt), mt.ctypes.data_as(c_int_p), mb.ctypes.data_as(c_double_p)
        affs = (AffineDesc * max(1, len(scene.affine)))()
        for i, b in enumerate(scene.affine):
            a = affs[i]
            rp, tr = self._d(b.rest_pos), self._i(b.tris)
            a.n_verts, a.n_tris = rp.shape[0], tr.shape[0]
            a.rest_pos, a.tris = rp.ctypes.data_as(c_double_p), tr.ctypes.data_as(c_int_p)
            a.kind, a.density, a.kappa_s = int(b.kind), b.density, b.kappa_s
        self.scene = SceneDesc()
        self.scene.n_soft, self.scene.n_affine = len(scene.soft), len(scene.affine)
        self.scene.soft = ctypes.cast(softs, ctypes.POINTER(SoftDesc))
        self.scene.affine = ctypes.cast(affs, ctypes.POINTER(AffineDesc))
        if scene.collide is not None:
            col = np.ascontiguousarray(scene.collide, dtype=np.uint8)
            self.keep.append(col)
            self.scene.collide = col.ctypes.data_as(ctypes.POINTER(ctypes.c_uint8))
        for k in range(3):
            self.scene.gravity[k] = float(scene.gravity[k])
        self.keep += [softs, affs]
        self.cfg = make_config(scene.config)

    def _d(self, a):
        a = np.ascontiguousarray(a, dtype=np.float64)
        self.keep.append(a)
        return a

    def _i(self, a):
        a = np.ascontiguousarray(a, dtype=np.int32)
        self.keep.append(a)
        return a


def workspace_size(scene, n_envs: int) -> int:
    d = _Descs(scene)
    out = ctypes.c_size_t()
    _check(load().tac_workspace_size(ctypes.byref(d.scene), n_envs, ctypes.byref(d.cfg), ctypes.byref(out)))
    return out.value


class Batch:
    """A batch of n_envs envs of one scene template on one CUDA device."""

    def __init__(self, scene, n_envs: int, device: int = 0, stream: Optional[torch.cuda.Stream] = None):
        if not torch.cuda.is_available():
            raise RuntimeError("CUDA is not available: the taccel hot path has no CPU fallback")
        self.lib = load()
        self.scene = scene
        self.n_envs = n_envs
        self.device = torch.device("cuda", device)
        self.stream = stream if stream is not None else torch.cuda.current_stream(self.device)
        d = _Descs(scene)
        size = ctypes.c_size_t()
        _check(self.lib.tac_workspace_size(ctypes.byref(d.scene), n_envs, ctypes.byref(d.cfg), ctypes.byref(size)))
        self.workspace = torch.empty(size.value + 256, dtype=torch.uint8, device=self.device)
        base = self.workspace.data_ptr()
        pad = (-base) % 256
        self.handle = ctypes.c_void_p()
        _check(self.lib.tac_batch_create(ctypes.byref(d.scene), n_envs, ctypes.byref(d.cfg), device,
                                         ctypes.c_void_p(base + pad), size.value, self._s(), ctypes.byref(self.handle)))
        dims = (ctypes.c_int32 * 10)()
        _check(self.lib.tac_batch_dims(self.handle, dims))
        (self.V, self.T, self.NA, self.NK, self.n_coated, self.n_markers, self.n_dof, self.n_vertices,
         self.n_tris, self.n_edges) = list(dims)

    def _s(self):
        return ctypes.c_void_p(self.stream.cuda_stream)

    def __del__(self):
        h = getattr(self, "handle", None)
        if h is not None and h.value:
            self.lib.tac_batch_destroy(h)
            self.handle = None

    # ---- state / targets -------------------------------------------------------------------
    def set_state(self, x, y, xdot=None, ydot=None, env0: int = 0):
        x, y = _f64(x), _f64(y)
        n = x.shape[0]
        st = np.zeros(n, np.uint8)
        _check(self.lib.tac_set_state(self.handle, env0, n, _ptr(x), _ptr(_f64(xdot) if xdot is not None else None),
                                      _ptr(y), _ptr(_f64(ydot) if ydot is not None else None), _ptr(st), self._s()))
        return st

    def set_targets(self, y_kin, env0: int = 0):
        y_kin = _f64(y_kin)
        _check(self.lib.tac_set_targets(self.handle, env0, y_kin.shape[0], _ptr(y_kin), self._s()))

    def set_chain(self, chain: dict):
        """Kinematic tree for on-device forward kinematics (keys: parent, origin, axis, joint, body,
        kin_body, n_joints — see include/taccel.h tac_chain_desc)."""
        keep = {k: (np.ascontiguousarray(chain[k], np.int32) if k in ("parent", "joint", "kin_body")
                    else np.ascontiguousarray(chain[k], np.float64)) for k in ("parent", "origin", "axis", "joint", "body", "kin_body")}
        d = ChainDesc()
        d.n_links, d.n_joints = len(keep["parent"]), int(chain["n_joints"])
        for k in ("parent", "joint", "kin_body"):
            setattr(d, k, keep[k].ctypes.data_as(c_int_p))
        for k in ("origin", "axis", "body"):
            setattr(d, k, keep[k].ctypes.data_as(c_double_p))
        _check(self.lib.tac_set_chain(self.handle, ctypes.byref(d)))

    def set_joint_targets(self, q, base=None, env0: int = 0):
        q = _f64(q)
        _check(self.lib.tac_set_joint_targets(self.handle, env0, q.shape[0], _ptr(_f64(base)) if base is not None else None,
                                              _ptr(q), self._s()))

    def get_targets(self, env0: int = 0, n: Optional[int] = None):
        n = self.n_envs - env0 if n is None else n
        out = np.zeros((n, self.NK, 12))
        _check(self.lib.tac_get_targets(self.handle, env0, n, _ptr(out), self._s()))
        return out

    def step(self, n_steps: int = 1, raise_on_failure: bool = False):
        st = np.zeros(self.n_envs, np.uint8)
        code = self.lib.tac_step(self.handle, n_steps, _ptr(st), self._s())
        if code not in (0, 3) or (code == 3 and raise_on_failure):
            _check(code)
        return st

    def step_schedule(self, y_kin_sched, out=None, raise_on_failure: bool = False):
        """Advance all envs through len(y_kin_sched) steps, each env independently (no lockstep);
        `out` = (coated [S,E,NC,3], marker_pos [S,E,NM,3], marker_flow [S,E,NM,3]) or None."""
        sched = _f64(y_kin_sched)
        n_steps = sched.shape[0]
        st = np.zeros(self.n_envs, np.uint8)
        c, mp, mf = out if out is not None else (None, None, None)
        code = self.lib.tac_step_schedule(self.handle, n_steps, _ptr(sched), _ptr(c), _ptr(mp), _ptr(mf), _ptr(st),
                                          self._s())
        if code not in (0, 3) or (code == 3 and raise_on_failure):
            _check(code)
        return st

    def get_state(self, env0: int = 0, n: Optional[int] = None, device=None):
        n = self.n_envs - env0 if n is None else n
        dev = self.device if device is None else device
        x = torch.empty((n, self.V, 3), dtype=torch.float64, device=dev)
        xd = torch.empty_like(x)
        y = torch.empty((n, self.NA, 12), dtype=torch.float64, device=dev)
        yd = torch.empty_like(y)
        _check(self.lib.tac_get_state(self.handle, env0, n, _ptr(x), _ptr(xd), _ptr(y), _ptr(yd), self._s()))
        return x, xd, y, yd

    def get_gel_deformation(self, env0: int = 0, n: Optional[int] = None, device=None, out=None):
        n = self.n_envs - env0 if n is None else n
        dev = self.device if device is None else device
        if out is None:
            out = (torch.empty((n, self.n_coated, 3), dtype=torch.float64, device=dev),
                   torch.empty((n, self.n_markers, 3), dtype=torch.float64, device=dev),
                   torch.empty((n, self.n_markers, 3), dtype=torch.float64, device=dev))
        c, mp, mf = out
        _check(self.lib.tac_get_gel_deformation(self.handle, env0, n, _ptr(c), _ptr(mp), _ptr(mf), self._s()))
        return out

    def get_depth_maps(self, H: int, W: int, env0: int = 0, n: Optional[int] = None, device=None, normals: bool = True):
        """Depth [n, pads, H, W] and normal [n, pads, H, W, 3] maps of the coated surfaces (tac_get_depth_maps)."""
        n = self.n_envs - env0 if n is None else n
        dev = self.device if device is None else device
        npads = len(self.scene.soft)
        d = torch.empty((n, npads, H, W), dtype=torch.float64, device=dev)
        nm = torch.empty((n, npads, H, W, 3), dtype=torch.float64, device=dev) if normals else None
        _check(self.lib.tac_get_depth_maps(self.handle, env0, n, H, W, _ptr(d), _ptr(nm), self._s()))
        return d, nm

    def stats(self):
        arr = (EnvStats * self.n_envs)()
        _check(self.lib.tac_get_stats(self.handle, arr, self._s()))
        out = [{k: getattr(s, k) for k, _ in EnvStats._fields_} for s in arr]
        for d in out:
            d["diag"] = list(d["diag"])
        return out

    # ---- tracing ---------------------------------------------------------------------------------
    NPHASES = 16

    def profile(self, enable: bool = True):
        _check(self.lib.tac_profile_enable(self.handle, 1 if enable else 0))

    def profile_read(self, reset: bool = False):
        ms = (ctypes.c_double * self.NPHASES)()
        n = (ctypes.c_int64 * self.NPHASES)()
        _check(self.lib.tac_profile_read(self.handle, ms, n, 1 if reset else 0))
        return {self.lib.tac_profile_phase_name(i).decode(): (ms[i], n[i]) for i in range(self.NPHASES)}

    def profile_iterations(self):
        n = ctypes.c_int32()
        _check(self.lib.tac_profile_iterations(self.handle, None, None, 0, ctypes.byref(n)))
        act = (ctypes.c_int32 * max(n.value, 1))()
        ms = (ctypes.c_double * max(n.value, 1))()
        _check(self.lib.tac_profile_iterations(self.handle, act, ms, n.value, ctypes.byref(n)))
        return list(act)[:n.value], list(ms)[:n.value]

    # ---- parity hooks (host numpy) ------------------------------------------------------------
    def debug_eval(self, env, x, y, lam_att=None, lam_kin=None, rho=0.0, v=None, exact=False):
        x, y = _f64(x), _f64(y)
        et = np.zeros(7)
        g = np.zeros(self.n_dof)
        hv = np.zeros(self.n_dof) if v is not None else None
        _check(self.lib.tac_debug_eval(self.handle, env, _ptr(x), _ptr(y),
                                       _ptr(_f64(lam_att)) if lam_att is not None else None,
                                       _ptr(_f64(lam_kin)) if lam_kin is not None else None, float(rho),
                                       1 if exact else 0, _ptr(_f64(v)) if v is not None else None, _ptr(et), _ptr(g), _ptr(hv), self._s()))
        return et, g, hv

    def _pairs(self, fn, env, x, y, *extra):
        cnt = ctypes.c_int32()
        _check(fn(self.handle, env, _ptr(_f64(x)), _ptr(_f64(y)), *extra, None, 0, ctypes.byref(cnt), self._s()))
        out = np.zeros((max(cnt.value, 1), 3), np.int32)
        _check(fn(self.handle, env, _ptr(_f64(x)), _ptr(_f64(y)), *extra, _ptr(out), cnt.value, ctypes.byref(cnt), self._s()))
        return out[:cnt.value]

    def debug_active_pairs(self, env, x, y):
        return self._pairs(self.lib.tac_debug_active_pairs, env, x, y)

    def debug_candidates(self, env, x, y, p=None):
        return self._pairs(self.lib.tac_debug_candidates, env, x, y, _ptr(_f64(p)) if p is not None else None)

    def debug_accd(self, env, x, y, p):
        a = ctypes.c_double()
        _check(self.lib.tac_debug_accd(self.handle, env, _ptr(_f64(x)), _ptr(_f64(y)), _ptr(_f64(p)), ctypes.byref(a), self._s()))
        return a.value

    def debug_pcg(self, env, x, y, exact=False, mu=0.0, with_mu=False):
        p = np.zeros(self.n_dof)
        it = ctypes.c_int32()
        mu_used = ctypes.c_double()
        _check(self.lib.tac_debug_pcg(self.handle, env, _ptr(_f64(x)), _ptr(_f64(y)), 1 if exact else 0, float(mu), _ptr(p),
                                      ctypes.byref(it), ctypes.byref(mu_used), self._s()))
        return (p, it.value, mu_used.value) if with_mu else (p, it.value)

    def debug_trace_start(self, env, cap=4096):
        _check(self.lib.tac_debug_trace(self.handle, env, cap, None, None))

    def debug_trace_read(self, cap=4096):
        rows = np.zeros((cap, 10))
        n = ctypes.c_int32()
        _check(self.lib.tac_debug_trace(self.handle, 0, cap, _ptr(rows), ctypes.byref(n)))
        return rows[:min(n.value, cap)]

    def debug_inject_fault(self, env, status):
        _check(self.lib.tac_debug_inject_fault(self.handle, env, int(status), self._s()))

    @property
    def pcg_kernel(self) -> str:
        return self.lib.tac_pcg_kernel_name(self.handle).decode()
