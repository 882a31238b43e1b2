"""Preconditioner study for NEXT 4 (CPU, oracle-assembled Newton systems of dumped GPU states).

python tools/precond_study.py gpurun_out/states_C3.npz [env] [steps...]

For the state before step k (ctx of step k) and the state after it (x^{k+1}, the converged point: the
Hessian the late Newton iterations see) the exact Hessian H (+ μM if not SPD) and g are assembled by the
oracle; PCG (p0 = 0, stop rᵀz ≤ η² r₀ᵀz₀, η = 1e-4; reading R15) runs with several preconditioners and the
iteration counts and the relative A-norm error of the result are printed.
"""
import sys
import time

import numpy as np
import scipy.linalg as sla
import scipy.sparse as sp

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
from paper_2504_12908_b200 import scenes as S
from oracle import contact as C
from oracle import energy as En
from oracle import mesh as M
from oracle import solver as SO


def pcg(A, b, prec, eta=1e-4, maxit=5000):
    x = np.zeros_like(b)
    r = b.copy()
    z = prec(r)
    d = z.copy()
    rz = r @ z
    rz0 = rz
    it = 0
    while it < maxit and rz > eta * eta * rz0:
        q = A @ d
        dq = d @ q
        if not dq > 0:
            return x, -it
        a = rz / dq
        x += a * d
        r -= a * q
        z = prec(r)
        rzn = r @ z
        d = z + (rzn / rz) * d
        rz = rzn
        it += 1
    return x, it


def block_jacobi(mod, A):
    V = mod.V
    blocks = [(3 * v, 3) for v in range(V)] + [(3 * V + 12 * s, 12) for s in range(mod.n_dof_bodies)]
    Ad = A.tocsr()
    inv = [np.linalg.inv(Ad[o:o + k, o:o + k].toarray()) for o, k in blocks]
    soft = sp.block_diag(inv[:V], format="csr")
    body = sp.block_diag(inv[V:], format="csr") if mod.n_dof_bodies else None
    Binv = sp.block_diag([soft, body], format="csr") if body is not None else soft
    return Binv


def aggregates(mod, a, layers=True):
    """soft vertices binned by rest position (pad frame) into a×a lattice-cell columns per pad."""
    V = mod.V
    X = mod.X
    body = mod.vert_body[:V]
    agg = np.full(V, -1)
    nag = 0
    for pb in np.unique(body):
        idx = np.nonzero(body == pb)[0]
        Xp = X[idx]
        # lattice spacing from the smallest positive coordinate differences
        ux = np.unique(np.round(Xp[:, 0], 9)); uy = np.unique(np.round(Xp[:, 1], 9)); uz = np.unique(np.round(Xp[:, 2], 9))
        ix = np.searchsorted(ux, np.round(Xp[:, 0], 9)) // a
        iy = np.searchsorted(uy, np.round(Xp[:, 1], 9)) // a
        iz = np.searchsorted(uz, np.round(Xp[:, 2], 9)) // (a if layers else 10 ** 6)
        key = (ix * 10000 + iy) * 100 + iz
        uk, inv = np.unique(key, return_inverse=True)
        agg[idx] = nag + inv
        nag += len(uk)
    return agg, nag


def coarse_basis(mod, agg, nag, rot=False, xpos=None):
    V = mod.V
    nb = 12 * mod.n_dof_bodies
    k = 6 if rot else 3
    rows, cols, vals = [], [], []
    for v in range(V):
        for c in range(3):
            rows.append(3 * v + c); cols.append(k * agg[v] + c); vals.append(1.0)
    if rot:
        cen = np.zeros((nag, 3))
        cnt = np.bincount(agg, minlength=nag)
        np.add.at(cen, agg, xpos)
        cen /= cnt[:, None]
        for v in range(V):
            r = xpos[v] - cen[agg[v]]
            # rotation about axis j: ω × r
            for j in range(3):
                e = np.zeros(3); e[j] = 1.0
                w = np.cross(e, r)
                for c in range(3):
                    if w[c] != 0.0:
                        rows.append(3 * v + c); cols.append(k * agg[v] + 3 + j); vals.append(w[c])
    for i in range(nb):
        rows.append(3 * V + i); cols.append(k * nag + i); vals.append(1.0)
    return sp.csr_matrix((vals, (rows, cols)), shape=(3 * V + nb, k * nag + nb))


def study(path, env=0, steps=None):
    D = np.load(path)
    cfgname = path.rsplit("states_", 1)[1].split(".")[0]
    sc = S.make_scene(cfgname)
    mod = M.prepare(sc)
    cfg = sc.config
    Mreg = SO.mass_matrix(mod)
    st = list(D["steps"])
    ks = [k for k in st if (k + 1) in st] if not steps else steps
    for k in ks:
        i0, i1 = st.index(k), st.index(k + 1)
        xn, vn, yn, ydn = D["x"][i0][env], D["v"][i0][env], D["y"][i0][env], D["ydot"][i0][env]
        L = M.env_scale(mod, xn, yn)
        ctx = En.make_context(mod, xn, vn, yn, ydn, D["ykin"][i0][env], cfg.dt)
        for label, (x, y) in (("x^n", (xn, yn)), ("x^n+1", (D["x"][i1][env], D["y"][i1][env]))):
            P = M.all_positions(mod, x, y)
            pairs = C.active_pairs(mod, P)
            t0 = time.time()
            g, H = En.assemble(mod, ctx, x, y, pairs, project=False)
            H = H.tocsr()
            mu = 0.0
            while True:
                A = H + mu * Mreg if mu > 0 else H
                try:
                    Lc = np.linalg.cholesky(A.toarray())
                    break
                except np.linalg.LinAlgError:
                    mu = max(cfg.lm_mu0, 10 * mu)
            pex = sla.cho_solve((Lc, True), -g)
            nA = np.sqrt(pex @ (A @ pex))
            print(f"step {k} {label}: pairs {len(pairs)} mu {mu:g} assemble {time.time() - t0:.1f}s |p|inf/L {np.abs(pex).max() / L:.2e}",
                  flush=True)
            Binv = block_jacobi(mod, A)
            res = {}

            def run(name, prec):
                p, it = pcg(A, -g, prec, cfg.pcg_eta)
                e = p - pex
                res[name] = (it, np.sqrt(e @ (A @ e)) / nA)

            run("BJ", lambda r: Binv @ r)
            for a in (2, 3, 4):
                agg, nag = aggregates(mod, a)
                for rot in (False, True):
                    Pc = coarse_basis(mod, agg, nag, rot, x if rot else None)
                    Ac = (Pc.T @ A @ Pc).toarray()
                    try:
                        cf = sla.cho_factor(Ac)
                    except np.linalg.LinAlgError:
                        res[f"{'RB' if rot else 'T'}agg{a}"] = (0, float('nan'))
                        continue
                    nm = f"{'RB' if rot else 'T'}agg{a}({Pc.shape[1]})"
                    run(nm + "+", lambda r, Pc=Pc, cf=cf: Binv @ r + Pc @ sla.cho_solve(cf, Pc.T @ r))

                    def hyb(r, Pc=Pc, cf=cf):
                        z = Pc @ sla.cho_solve(cf, Pc.T @ r)
                        z = z + Binv @ (r - A @ z)
                        return z + Pc @ sla.cho_solve(cf, Pc.T @ (r - A @ z))
                    run(nm + "*", hyb)
            print("   " + "  ".join(f"{n}:{it}/{err:.0e}" for n, (it, err) in res.items()), flush=True)


if __name__ == "__main__":
    a = sys.argv[1:]
    study(a[0], int(a[1]) if len(a) > 1 else 0, [int(s) for s in a[2:]] or None)
