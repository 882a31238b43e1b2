"""Oracle time step (test infrastructure only — see oracle/__init__.py).

One backward-Euler step as the argmin of the barrier-augmented incremental potential with AL
kinematic constraints (P:L89-97 Eq. IP, P:L127-131 Eq. unified_ipc_variational
Eq. unified_ipc_AL, P:L370 velocity update).  The paper gives no minimiser; the machinery follows
SURVEY §8(c)-14..17 (readings R14-R17 in DESIGN.md):

  x̃ = xⁿ + Δt ẋⁿ;  λ = 0, ρ = ρ₀;  q = qⁿ (feasible start)
  repeat AL rounds:
    repeat Newton:
      𝒜 = active set at q;  g, H = assemble (PSD-projected);  p = −H⁻¹g (exact sparse solve)
      if ‖p‖_emb,∞ ≤ τ_N·L_env: inner converged
      C′ = swept candidates over [q, q+p];  α = min(1, ACCD over C′)
      halve α until no det F ≤ 0 and E(q+αp) ≤ E(q) + c·α·gᵀp  (α < 1e-10 → NEWTON_STALL)
      q ← q + αp
    r = max constraint residual on embedded vertices;  r ≤ τ_AL·L_env → done
    if r > ½ r_prev: ρ ← 2ρ;   λ ← λ − ρ·(S q − s)
  ẋⁿ⁺¹ = (xⁿ⁺¹ − xⁿ)/Δt,  ẏⁿ⁺¹ = (yⁿ⁺¹ − yⁿ)/Δt
"""
from __future__ import annotations

import dataclasses

import numpy as np
import scipy.sparse as sp
import scipy.sparse.linalg as spla

from . import contact as C
from . import energy as En
from .mesh import Model, all_positions, embed, env_scale

ENV_OK, NEWTON_STALL, AL_INFEASIBLE, CAPACITY, NONFINITE, BAD_STATE, DISABLED = range(7)


@dataclasses.dataclass
class State:
    x: np.ndarray     # (V,3)
    v: np.ndarray     # (V,3)
    y: np.ndarray     # (NA,12)
    ydot: np.ndarray  # (NA,12)


@dataclasses.dataclass
class StepStats:
    status: int = ENV_OK
    newton_iters: int = 0
    ls_backtracks: int = 0
    al_rounds: int = 0
    pcg_iters: int = 0
    alpha_min: float = 1.0
    n_active: int = 0
    energy: float = 0.0
    constraint_residual: float = 0.0
    min_dist: float = np.inf


def embedded_inf_norm(model: Model, p, y_like=None):
    """‖p‖_emb,∞: max |p_i| over soft DoFs and max component of J_v p_b over the vertices of every
    non-static affine body (reading R14)."""
    V = model.V
    m = float(np.abs(p[:3 * V]).max()) if V else 0.0
    for bi, xb in enumerate(model.body_xbar):
        s = model.dof_slot[bi]
        if s < 0:
            continue
        pb = p[3 * V + 12 * s:3 * V + 12 * s + 12]
        m = max(m, float(np.abs(embed(pb, xb)).max()))
    return m


def constraint_residual(model: Model, ctx: En.Context, x, y):
    """max over ∂⁻G vertices of ‖x_v − s_v‖ and over kinematic bodies' vertices of
    ‖(t−t_s) + (A−A_s) x̄_v‖ (reading R13)."""
    r = 0.0
    if len(model.att_vert):
        r = float(np.sqrt(((x[model.att_vert] - ctx.s_att) ** 2).sum(1)).max())
    for k, b in enumerate(model.kin_bodies):
        d = y[b] - ctx.s_kin[k]
        r = max(r, float(np.sqrt((embed(d, model.body_xbar[b]) ** 2).sum(1)).max()))
    return r


def any_inverted(model: Model, x):
    if len(model.tets) == 0:
        return False
    X = x[model.tets]
    Ds = np.stack([X[:, 1] - X[:, 0], X[:, 2] - X[:, 0], X[:, 3] - X[:, 0]], 2)
    F = Ds @ model.Dm_inv
    return bool((np.linalg.det(F) <= 0).any())


def forcing_eta(cfg, rz0, hist):
    """Relaxed PCG tolerance of one Newton iteration (reading R24; "carefully relaxing convergence
    tolerances"), Eisenstat–Walker choice 2 with γ = 0.9, α = 2 in the preconditioned gradient norm
    ‖g‖² = r₀ᵀz₀ of the solve:  η_k = γ·r₀ᵀz₀(k) / r₀ᵀz₀(k−1),  safeguard η_k ≥ γ η_{k−1}² when γ η_{k−1}² > 0.1,
    clamped to [pcg_eta, pcg_eta_max];  the first solve of a time step uses pcg_eta_max.  hist holds
    (r₀ᵀz₀, η) of the previous accepted solve of this step, or None."""
    if hist is None:
        return cfg.pcg_eta_max
    rz_prev, eta_prev = hist
    eta = 0.9 * rz0 / rz_prev
    if 0.9 * eta_prev * eta_prev > 0.1:
        eta = max(eta, 0.9 * eta_prev * eta_prev)
    return min(max(eta, cfg.pcg_eta), cfg.pcg_eta_max)


def block_jacobi_pcg(model: Model, H, g, eta, max_iter, info=None):
    """Block-Jacobi PCG for H p = −g from p₀ = 0 (3×3 per soft vertex, 12×12 per body); stop
    at rᵀz ≤ η² r₀ᵀz₀ or max_iter (reading R15; P:L325 names PCG).  Returns (None, it) if a
    search direction with dᵀHd ≤ 0 is met (H not SPD).  eta may be a function of r₀ᵀz₀ (the relaxed
    tolerance of reading R24); info (a dict) receives the r₀ᵀz₀ and η used."""
    n = len(g)
    V = model.V
    blocks = [(3 * v, 3) for v in range(V)] + [(3 * V + 12 * s, 12) for s in range(model.n_dof_bodies)]
    Hd = H.toarray() if n <= 4000 else None
    inv = []
    for o, k in blocks:
        B = Hd[o:o + k, o:o + k] if Hd is not None else H[o:o + k, o:o + k].toarray()
        inv.append(np.linalg.inv(B))

    def prec(r):
        z = np.zeros_like(r)
        for (o, k), Bi in zip(blocks, inv):
            z[o:o + k] = Bi @ r[o:o + k]
        return z

    p = np.zeros(n)
    r = -g.copy()
    z = prec(r)
    d = z.copy()
    rz = r @ z
    rz0 = rz
    if callable(eta):
        eta = eta(rz0)
    if info is not None:
        info["rz0"], info["eta"] = rz0, eta
    it = 0
    while it < max_iter and rz > eta * eta * rz0:
        q = H @ d
        dq = d @ q
        if not (dq > 0):
            return None, it + 1          # negative curvature: H is not SPD
        a = rz / dq
        p += a * d
        r -= a * q
        z = prec(r)
        rz_new = r @ z
        d = z + (rz_new / rz) * d
        rz = rz_new
        it += 1
    return p, it


def mass_matrix(model: Model):
    """M over the DoFs: lumped m_v I₃ per soft vertex and M^y per non-static body."""
    n = model.n_dof
    rows, cols, vals = [np.arange(3 * model.V)], [np.arange(3 * model.V)], [np.repeat(model.mass, 3)]
    for bi in range(len(model.body_xbar)):
        s_ = model.dof_slot[bi]
        if s_ < 0:
            continue
        idx = np.arange(3 * model.V + 12 * s_, 3 * model.V + 12 * s_ + 12)
        R, Cc = np.meshgrid(idx, idx, indexing="ij")
        rows.append(R.ravel()); cols.append(Cc.ravel()); vals.append(model.body_My[bi].ravel())
    return sp.coo_matrix((np.concatenate(vals), (np.concatenate(rows), np.concatenate(cols))), shape=(n, n)).tocsr()


def sweep_factor(cfg, p_inf):
    """K_eff (reading R17b): the largest power of two ≤ ls_expand with K_eff·‖p‖_emb,∞ ≤ d̂, at
    least 1 — the expansion sweep never reaches further than d̂ beyond a normal Newton step."""
    K = 1
    while 2 * K <= cfg.ls_expand and 2.0 * K * p_inf <= cfg.dhat:
        K *= 2
    return K


def _pcg_eta(cfg, ew):
    """the PCG tolerance: fixed η (R15), or the relaxed forcing of R24 when pcg_eta_max > 0"""
    if getattr(cfg, "pcg_eta_max", 0.0) > 0.0:
        return lambda rz0: forcing_eta(cfg, rz0, ew.get("hist"))
    return cfg.pcg_eta


def _solve_spd(model, H, g, solver, cfg, stats, ew=None):
    """Newton direction from the EXACT Hessian if it is SPD (Cholesky succeeds / CG meets no
    negative curvature) and the direction is a descent direction; None otherwise (reading R14b)."""
    if solver == "direct":
        Hd = H.toarray()
        try:
            Lc = np.linalg.cholesky(Hd)
        except np.linalg.LinAlgError:
            return None
        import scipy.linalg as sla
        p = sla.cho_solve((Lc, True), -g)
    else:
        ew = {} if ew is None else ew
        info = {}
        p, it = block_jacobi_pcg(model, H, g, _pcg_eta(cfg, ew), cfg.max_pcg, info)
        stats.pcg_iters += it
        if p is None:
            return None
        ew["last"] = (info["rz0"], info["eta"])
    if not (g @ p < 0) and np.any(g):
        return None
    return p


def step(model: Model, st: State, y_kin_target, solver="direct", L_env=None, trace=None):
    """Advance one env by one time step; returns (new State, StepStats)."""
    cfg = model.scene.config
    dt = cfg.dt
    stats = StepStats()
    L = env_scale(model, st.x, st.y) if L_env is None else L_env
    ctx = En.make_context(model, st.x, st.v, st.y, st.ydot, y_kin_target, dt)
    x, y = st.x.copy(), st.y.copy()
    r_prev = np.inf
    done = False
    hold = 0          # projected iterations left before the exact Hessian is tried again
    nfail = 0         # consecutive failed exact attempts (back-off 2, 4, ... 64)
    mode = cfg.hessian_mode
    mu = 0.0          # mass-scaled Levenberg-Marquardt shift (hessian_mode 2, reading R14c)
    ew = {}           # relaxed-tolerance history of this step (reading R24): (r₀ᵀz₀, η) of the last accepted solve
    Mreg = mass_matrix(model) if mode == 2 else None
    for al_round in range(cfg.max_al_rounds):
        stats.al_rounds = al_round + 1
        converged = False
        while stats.newton_iters < cfg.max_newton:
            P = all_positions(model, x, y)
            pairs = C.active_pairs(model, P)
            p = None
            mu_used = 0.0
            if mode == 2:
                g, H = En.assemble(model, ctx, x, y, pairs, project=False)
                while True:
                    p = _solve_spd(model, H + mu * Mreg if mu > 0 else H, g, solver, cfg, stats, ew)
                    if p is not None or mu > 1e12:
                        break
                    mu = max(cfg.lm_mu0, 10.0 * mu)
                mu_used = mu
                mu = mu * 0.1 if mu * 0.1 >= cfg.lm_mu0 else 0.0
            if mode == 1 and hold == 0:
                g, H = En.assemble(model, ctx, x, y, pairs, project=False)
                p = _solve_spd(model, H, g, solver, cfg, stats, ew)
                if p is None:
                    nfail += 1
                    hold = min(2 ** nfail, cfg.hold_cap)
                else:
                    nfail = 0
            if p is None:
                g, H = En.assemble(model, ctx, x, y, pairs)
                if solver == "direct":
                    p = spla.spsolve(sp.csc_matrix(H), -g)
                else:
                    info = {}
                    p, it = block_jacobi_pcg(model, H, g, _pcg_eta(cfg, ew), cfg.max_pcg, info)
                    stats.pcg_iters += it
                    ew["last"] = (info["rz0"], info["eta"])
                hold = max(hold - 1, 0)
            stats.newton_iters += 1
            if "last" in ew:
                ew["hist"] = ew.pop("last")
            if p is None or not np.all(np.isfinite(p)):
                stats.status = NONFINITE
                break
            p_inf = embedded_inf_norm(model, p)
            if p_inf <= cfg.newton_tol_rel * L and mu_used == 0.0:
                converged = True
                break
            # reading R14d: under an LM shift the step is no convergence measure; converged when the
            # mass-scaled gradient step M⁻¹g is below τ_N·L_env (embedded ∞-norm)
            if mu_used > 0.0 and embedded_inf_norm(model, spla.spsolve(Mreg.tocsc(), g)) <= cfg.newton_tol_rel * L:
                converged = True
                break
            if p_inf > cfg.max_step_rel * L:            # step cap (reading R17c)
                p = p * (cfg.max_step_rel * L / p_inf)
            dx, dy = En.unpack(model, p, np.zeros_like(y))
            Pd = _disp_positions(model, dx, dy)
            K = sweep_factor(cfg, embedded_inf_norm(model, p))
            cand = C.candidate_pairs(model, P, P + K * Pd)
            alpha_max = K * C.accd_bound(model, P, K * Pd, cand)
            alpha = min(1.0, alpha_max)
            E0 = En.total_energy(model, ctx, x, y, pairs)
            gp = float(g @ p)

            def trial(a):
                xa, ya = x + a * dx, y + a * dy
                if any_inverted(model, xa):
                    return None, xa, ya
                Pa = all_positions(model, xa, ya)
                return En.total_energy(model, ctx, xa, ya, C.active_pairs(model, Pa, cand)), xa, ya

            while True:
                E1, xt, yt = trial(alpha)
                if E1 is not None and E1 <= E0 + cfg.armijo_c * alpha * gp:
                    break
                alpha *= 0.5
                stats.ls_backtracks += 1
                if alpha < 1e-10:
                    break
            # expansion (reading R17b): after a full step, keep doubling α while the energy keeps
            # decreasing, α stays under the ACCD bound of the K-times longer sweep and Armijo holds
            if alpha == 1.0 and K > 1:
                while 2.0 * alpha <= alpha_max:
                    E2, x2, y2 = trial(2.0 * alpha)
                    if E2 is None or not (E2 < E1) or not (E2 <= E0 + cfg.armijo_c * 2.0 * alpha * gp):
                        break
                    alpha, E1, xt, yt = 2.0 * alpha, E2, x2, y2
            if alpha < 1e-10:
                stats.status = NEWTON_STALL
                break
            stats.alpha_min = min(stats.alpha_min, alpha)
            if trace is not None:
                trace.append(dict(alpha=alpha, E0=E0, E1=E1, p_inf=embedded_inf_norm(model, p), hold=hold,
                                  n_act=len(pairs)))
            x, y = xt, yt
        if stats.status != ENV_OK:
            break
        if not converged:
            stats.status = NEWTON_STALL
            break
        res = constraint_residual(model, ctx, x, y)
        stats.constraint_residual = res
        if trace is not None:
            trace.append(dict(al_round=al_round, residual=res, rho=ctx.rho, newton=stats.newton_iters))
        if res <= cfg.al_tol_rel * L:
            done = True
            break
        if res > 0.5 * r_prev:
            ctx.rho *= 2.0
        r_prev = res
        if len(model.att_vert):
            ctx.lam_att = ctx.lam_att - ctx.rho * (x[model.att_vert] - ctx.s_att)
        for k, b in enumerate(model.kin_bodies):
            ctx.lam_kin[k] = ctx.lam_kin[k] - ctx.rho * (y[b] - ctx.s_kin[k])
    if stats.status == ENV_OK and not done:
        stats.status = AL_INFEASIBLE
    if stats.status != ENV_OK:
        return dataclasses.replace(st), stats          # rollback to xⁿ
    P = all_positions(model, x, y)
    pairs = C.active_pairs(model, P)
    stats.n_active = len(pairs)
    stats.energy = En.total_energy(model, ctx, x, y, pairs)
    new = State(x=x, v=(x - st.x) / dt, y=y, ydot=(y - st.y) / dt)
    for bi in range(len(model.body_xbar)):
        if model.dof_slot[bi] < 0:
            new.ydot[bi] = 0.0
            new.y[bi] = st.y[bi]
    return new, stats


def _disp_positions(model: Model, dx, dy):
    """Vertex displacements of a DoF step: soft dx, affine J_v p_b (static bodies 0)."""
    Pd = np.zeros((model.NVall, 3))
    Pd[:model.V] = dx
    o = model.V
    for bi, xb in enumerate(model.body_xbar):
        if model.dof_slot[bi] >= 0:
            Pd[o:o + len(xb)] = embed(dy[bi], xb)
        o += len(xb)
    return Pd
