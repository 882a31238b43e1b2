// pcg_cluster.cuh — env-resident block-Jacobi PCG over a thread-block cluster (k_pcg_cl<NC>), included
// by kernels.cu.  Solves (H + μM) p = −g of one env per cluster of NC CTAs (P:L325 names PCG as the
// bottleneck; readings R14c, R15).
//
// Layout: the env's soft rows are split into NC contiguous ranges of `rpr` rows; CTA r holds, in its
// shared memory, the upper 3×3 edge blocks of every soft edge touching its rows (the lower block is the
// transpose), its block-row index lists, its rows' search direction u (read by neighbouring CTAs through
// distributed shared memory), its rows' soft–body coupling blocks, and a copy of the bodies' u.  Every
// other per-row vector (x, r, p, s, the 3×3 diagonal block and its block-Jacobi inverse) lives in the
// REGISTERS of the thread that owns the row.  CTA 0 also owns the DoF bodies (one 16-lane half-warp per
// body, lane = row: its Hb row and block-Jacobi inverse row in registers) and the few matrix-free
// ("residual") contact pairs.
//
// Iteration: standard (Hestenes–Stiefel) block-Jacobi PCG, the oracle's algorithm (R15):
//   q = Ad; α = rᵀz / dᵀq (dᵀq ≤ 0 → not SPD); x += αd; r −= αq; z = M⁻¹r; β = rᵀz_new / rᵀz; d = z + βd,
// with three fused phases per iteration separated by barriers: A after the SpMV and dᵀq partials (and
// the body coupling sums), B after the x/r/z update and rᵀz partials, C after d is rewritten.  (A
// single-reduction Chronopoulos–Gear variant was tried: its recurrence for dᵀAd lost positivity on
// near-singular exact contact Hessians, escalating the LM shift where the oracle's PCG did not.)  All
// sums run in fixed orders (warp butterflies, warps in order, ranks in order), so results are bitwise
// reproducible and independent of the batch size.
#include <cooperative_groups.h>

namespace tac {
namespace cg = cooperative_groups;


template <int NC>
__device__ __forceinline__ void cl_barrier() {
  if constexpr (NC == 1) __syncthreads();
  else cg::this_cluster().sync();
}

// sum of two per-thread values over the whole cluster, identical in every thread (fixed order).
// `red` = this CTA's scratch (≥ 2·nwarps + 4 doubles); slot selects the CTA-total pair (0 or 1) so
// back-to-back reductions do not overwrite totals other CTAs may still be reading.
// sum of two per-thread values over the whole cluster, identical in every thread (fixed order).
// `red` = this CTA's scratch (72 doubles): totals in [2·slot, 2·slot+2), warp partials in
// [8 + 32·slot, 8 + 32·slot + 2·nwarps) — separate regions per slot, so two reductions back to back
// (the PCG's dᵀq and rᵀz) never overwrite values another warp or CTA may still be reading.
template <int NC>
__device__ __forceinline__ void cl_sum2(double& a, double& b, double* red, double* const* rred, int slot) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  double* part = red + 8 + 32 * slot;
  a = warp_sum(a);
  b = warp_sum(b);
  if (lane == 0) { part[2 * w] = a; part[2 * w + 1] = b; }
  if constexpr (NC == 1) {                       // one CTA: every thread sums the warp partials in order
    __syncthreads();
    double ta = 0.0, tb = 0.0;
    for (int k = 0; k < nw; ++k) { ta += part[2 * k]; tb += part[2 * k + 1]; }
    a = ta;
    b = tb;
    (void)rred;
  } else {                                       // CTA totals, then every rank's totals in rank order
    __syncthreads();
    if (threadIdx.x == 0) {
      double ta = 0.0, tb = 0.0;
      for (int k = 0; k < nw; ++k) { ta += part[2 * k]; tb += part[2 * k + 1]; }
      red[2 * slot] = ta;
      red[2 * slot + 1] = tb;
    }
    cl_barrier<NC>();
    double ta = 0.0, tb = 0.0;
#pragma unroll
    for (int r = 0; r < NC; ++r) { ta += rred[r][2 * slot]; tb += rred[r][2 * slot + 1]; }
    a = ta;
    b = tb;
  }
}

// residual (matrix-free) pairs of one env, one pair per lane over all warps of CTA 0: soft-slot outputs
// to sout (vertex-sorted slot positions), body-slot outputs pulled back through J_vᵀ and added to the
// warp partials; returns this thread's share of uᵀH_k u (δ).  Rare (pairs joining two soft bodies or
// two DoF bodies), so kept out of line to spare the main loop's registers.
template <int NC>
__device__ __noinline__ double cl_residual_pairs(const Dev& D, int e, int nres, int rpr, const double* usm, const double* ub,
                                                 double* wpart, double* const* ru) {
  const int lane = threadIdx.x & 31, tid = threadIdx.x, ND = D.ND;
  const double* aH = D.act_H + (size_t)e * D.res_cap * PH;
  const int* aslot = D.act_slot + (size_t)e * 4 * D.act_cap;
  const double* axb = D.act_xb + (size_t)e * 12 * D.act_cap;
  const int* spos = D.spos + (size_t)e * 4 * D.act_cap;
  double* sout = D.sout + (size_t)e * 4 * D.act_cap * 3;
  const int* rl = D.res_list + (size_t)e * D.act_cap;
  auto soft_u = [&](int vv) -> v3 {
    if constexpr (NC == 1) return ld3(usm + 3 * vv);
    else return ld3(ru[vv / rpr] + 3 * (vv % rpr));
  };
  double dloc = 0.0;
  for (int base = 32 * (tid >> 5); base < nres; base += blockDim.x) {
    const int idx = base + lane;
    double out[12];
    int bds[4] = {-1, -1, -1, -1};
    v3 xbs[4];
#pragma unroll
    for (int i = 0; i < 12; ++i) out[i] = 0.0;
    if (idx < nres) {
      const int k = rl[idx];
      double xl[12];
      const int4 code4 = reinterpret_cast<const int4*>(aslot)[k];
      const int codes[4] = {code4.x, code4.y, code4.z, code4.w};
      for (int s = 0; s < 4; ++s) {
        const int cd = codes[s];
        v3 q = mk(0, 0, 0);
        if (cd >= 0) q = soft_u(cd);
        else if (cd != INT_MIN) {
          const int sl = -1 - cd;
          xbs[s] = ld3(axb + 12 * k + 3 * s);
          q = embed(ub + 12 * sl, xbs[s]);
          bds[s] = sl;
        }
        xl[3 * s] = q.x; xl[3 * s + 1] = q.y; xl[3 * s + 2] = q.z;
      }
      const double* Hk = aH + (size_t)idx * PH;
#pragma unroll
      for (int a = 0; a < 12; ++a)
#pragma unroll
        for (int c = a; c < 12; ++c) {
          const double h = Hk[sym_idx(a, c, 12)];
          out[a] += h * xl[c];
          if (c != a) out[c] += h * xl[a];
        }
      double qq = 0.0;
#pragma unroll
      for (int i = 0; i < 12; ++i) qq += xl[i] * out[i];
      dloc += qq;
      for (int s = 0; s < 4; ++s) {
        const int j = spos[4 * k + s];
        if (j >= 0) st3(sout + 3 * j, mk(out[3 * s], out[3 * s + 1], out[3 * s + 2]));
      }
    }
    const bool touches = bds[0] >= 0 || bds[1] >= 0 || bds[2] >= 0 || bds[3] >= 0;
    if (__ballot_sync(0xffffffffu, touches) == 0u) continue;
    for (int d = 0; d < ND; ++d) {
      const bool m = bds[0] == d || bds[1] == d || bds[2] == d || bds[3] == d;
      if (__ballot_sync(0xffffffffu, m) == 0u) continue;
      double cc[12];
#pragma unroll
      for (int i = 0; i < 12; ++i) cc[i] = 0.0;
      if (m)
        for (int s = 0; s < 4; ++s) {
          if (bds[s] != d) continue;
          for (int i = 0; i < 3; ++i) {
            const double oi = out[3 * s + i];
            cc[i] += oi;
            cc[3 + 3 * i] += oi * xbs[s].x; cc[4 + 3 * i] += oi * xbs[s].y; cc[5 + 3 * i] += oi * xbs[s].z;
          }
        }
#pragma unroll
      for (int i = 0; i < 12; ++i) cc[i] = warp_sum(cc[i]);
      if (lane == 0) {
        double* wp = wpart + ((size_t)(tid >> 5) * ND + d) * 12;
#pragma unroll
        for (int i = 0; i < 12; ++i) wp[i] += cc[i];
      }
    }
  }
  __threadfence();
  return dloc;
}

// LM retry (R14c), bodies: (CTA 0, first body warp) every body's 12×12 block-Jacobi inverse of
// (diagonal block + μM^y) by warp Cholesky, then the shifted body blocks and inverses into shared
// memory.  Out of line: runs only after a failed solve.
__device__ __noinline__ void cl_reinvert_bodies(const Dev& D, int e, double mu, bool rank0, bool body_warp0, double* sHb,
                                                double* sPb) {
  __shared__ double chol_L[144], chol_A[144];
  const int ND = D.ND, lane = threadIdx.x & 31;
  if (rank0 && body_warp0) {
    for (int d = 0; d < ND; ++d) {
      const double* Db = D.Dg_b + ((size_t)e * ND + d) * 144;
      const double* Mb = D.My + (size_t)D.dof_body[d] * 144;
      for (int i = lane; i < 144; i += 32) chol_A[i] = Db[i] + mu * Mb[i];
      __syncwarp();
      chol_inverse12_warp(chol_A, D.Pinv_b + ((size_t)e * ND + d) * 144, chol_L, lane);
      __syncwarp();
    }
  }
  __syncthreads();
  if (rank0)
    for (int i = threadIdx.x; i < 144 * ND; i += blockDim.x) {
      const int d = i / 144;
      sHb[i] = D.Hb[(size_t)e * ND * 144 + i] + mu * D.My[(size_t)D.dof_body[d] * 144 + i % 144];
      sPb[i] = D.Pinv_b[(size_t)e * ND * 144 + i];
    }
  __syncthreads();
}

template <int NC>
__global__ void __launch_bounds__(CL_MAX_THREADS, 1) k_pcg_cl(const __grid_constant__ Dev D, const __grid_constant__ ClPlan Pl, int env0, int force) {
  const int rank = NC == 1 ? 0 : (int)cg::this_cluster().block_rank();
  const int e = D.elist ? D.elist[blockIdx.x / NC] : env0 + (int)blockIdx.x / NC;
  EnvCtl& C = D.ctl[e];
  if (env_skip(D, e, force)) return;            // uniform over the cluster (all CTAs read the same phase)
  extern __shared__ __align__(16) unsigned char cl_dsm[];
  const int V = D.V, ND = D.ND, n = D.n, rpr = Pl.rpr;
  const int nw = blockDim.x >> 5, lane = threadIdx.x & 31, tid = threadIdx.x;
  const ClSmem L = cl_smem(rpr, Pl.nle_max, Pl.nlb_max, ND, nw, Pl.cplcap);
  double* U = reinterpret_cast<double*>(cl_dsm + L.U);
  double* usm = reinterpret_cast<double*>(cl_dsm + L.u);
  double* ub = reinterpret_cast<double*>(cl_dsm + L.ub);
  double* pbody = reinterpret_cast<double*>(cl_dsm + L.pbody);
  double* wpart = reinterpret_cast<double*>(cl_dsm + L.wpart);
  int2* blk = reinterpret_cast<int2*>(cl_dsm + L.blk);
  int* rp = reinterpret_cast<int*>(cl_dsm + L.rptr);
  int* cpp = reinterpret_cast<int*>(cl_dsm + L.cpp);
  int* cpld = reinterpret_cast<int*>(cl_dsm + L.cpld);
  double* cval = reinterpret_cast<double*>(cl_dsm + L.cval);
  double* red = reinterpret_cast<double*>(cl_dsm + L.red);
  // remote views (distributed shared memory) of every rank's u, body partials and totals
  __shared__ double* ru[NC];
  __shared__ double* rred[NC];
  __shared__ double* rpb[NC];
  const double* ub0 = ub;
  if constexpr (NC == 1) {
    if (threadIdx.x == 0) { ru[0] = usm; rred[0] = red; rpb[0] = pbody; }
  } else {
    cg::cluster_group cl = cg::this_cluster();
    if (threadIdx.x < NC) {
      ru[threadIdx.x] = cl.map_shared_rank(usm, (int)threadIdx.x);
      rred[threadIdx.x] = cl.map_shared_rank(red, (int)threadIdx.x);
      rpb[threadIdx.x] = cl.map_shared_rank(pbody, (int)threadIdx.x);
    }
    ub0 = cl.map_shared_rank(ub, 0);
  }

  // ---------------------------------------------------------------- staging (once per launch)
  const int v0 = rank * rpr, nrows = min(rpr, V - v0);
  const int le0 = Pl.eptr[rank], nle = Pl.eptr[rank + 1] - le0;
  const int lb0 = Pl.bptr[rank], nlb = Pl.bptr[rank + 1] - lb0;
  const double* Ho = D.Ho + (size_t)e * D.NNZ * 9;
  for (int i = tid; i < 9 * nle; i += blockDim.x) U[i] = Ho[9 * (size_t)D.eup[Pl.edge[le0 + i / 9]] + i % 9];
  for (int i = tid; i < nlb; i += blockDim.x) blk[i] = Pl.blk[lb0 + i];
  for (int i = tid; i <= nrows; i += blockDim.x) {
    rp[i] = Pl.lrptr[rank * (rpr + 1) + i];
    cpp[i] = D.cpl_ptr[(size_t)e * (V + 1) + v0 + i];
  }
  __syncthreads();
  const int c0 = cpp[0], ncl = cpp[nrows] - c0;
  const bool cstaged = ncl <= Pl.cplcap;             // else the couplings are read from global memory
  const double* cv_g = D.cpl_val + (size_t)e * 36 * D.cpl_cap;
  const int* cd_g = D.cpl_d + (size_t)e * D.cpl_cap;
  if (cstaged) {
    for (int i = tid; i < ncl; i += blockDim.x) {
      cpld[i] = cd_g[c0 + i];
#pragma unroll 4
      for (int k = 0; k < 36; ++k) cval[(size_t)k * Pl.cplcap + i] = cv_g[(size_t)k * D.cpl_cap + c0 + i];
    }
  }

  // roles
  const bool vt = tid < Pl.nvt;
  const int vl = tid;                                   // local row of a vertex thread
  const int v = v0 + vl;
  const bool vown = vt && vl < nrows;
  const int bw = vt ? -1 : (tid - Pl.nvt) >> 5, brow = lane & 15, bd = 2 * bw + (lane >> 4);
  const bool bown = !vt && rank == 0 && brow < 12 && bd < ND;
  const int hl = lane & 16;                             // first lane of this body's half-warp

  // per-row state in registers
  v3 x = mk(0, 0, 0), r = mk(0, 0, 0), pp = mk(0, 0, 0), ss = mk(0, 0, 0), uu = mk(0, 0, 0);
  double Ps[9], mv = 0.0;
  double* sHd = reinterpret_cast<double*>(cl_dsm + L.hd);          // [9][rpr] diagonal blocks of this CTA's rows
  double xb = 0.0, rb = 0.0, pb = 0.0, sb = 0.0, ubr = 0.0;   // body row
  double* sHb = reinterpret_cast<double*>(cl_dsm + L.hb);          // [ND][144] H_b + μ M^y (CTA 0)
  double* sPb = sHb + 144 * (size_t)ND;                           // [ND][144] block-Jacobi inverse
  const double* g = D.g + (size_t)e * n;
  if (vown) {
#pragma unroll
    for (int k = 0; k < 9; ++k) {
      sHd[k * rpr + vl] = D.Hd[(size_t)e * V * 9 + (size_t)k * V + v];
      Ps[k] = D.Pinv_s[(size_t)e * V * 9 + (size_t)k * V + v];
    }
    mv = D.mass[v];
  }
  const double mu_in = C.mu;
  if (rank == 0)
    for (int i = tid; i < 144 * ND; i += blockDim.x) {
      const int d = i / 144;
      sHb[i] = D.Hb[(size_t)e * ND * 144 + i] + mu_in * D.My[(size_t)D.dof_body[d] * 144 + i % 144];
      sPb[i] = D.Pinv_b[(size_t)e * ND * 144 + i];
    }
  __syncthreads();                                      // staged body blocks / couplings visible

  // residual (matrix-free) pairs: CTA 0 (cl_residual_pairs); their soft-slot outputs are added after barrier A
  const double* sout = D.sout + (size_t)e * 4 * D.act_cap * 3;
  const int nres = C.n_res;
  const int* ccp = D.cptr + (size_t)e * (V + 1);
  const int* rcn = D.rcnt + (size_t)e * V;
  double mu = C.mu;
  bool bad = false, zero_g = false;
  int it_total = 0;
  double gp = 0.0;
  double rz0_used = 0.0, eta_used = 0.0;
  auto uv_at = [&](int colpk) -> v3 {                  // u of a soft vertex (local or remote rank)
    const int rk = colpk >> 16, lr = colpk & 0xffff;
    if constexpr (NC == 1) return ld3(usm + 3 * lr);
    else return ld3(ru[rk] + 3 * lr);
  };

  for (int attempt = 0;; ++attempt) {
    if (attempt > 0) {                                 // LM retry (R14c): re-invert with the new μ
      if (vown) {
        const double* ds = D.Dg_s + (size_t)e * V * 9;
        double Pv[9];
#pragma unroll
        for (int k = 0; k < 9; ++k) Pv[k] = ds[(size_t)k * V + v];
        const double sh = mu * mv;
        Pv[0] += sh; Pv[4] += sh; Pv[8] += sh;
        inv33(Pv, Ps);
      }
      cl_reinvert_bodies(D, e, mu, rank == 0, !vt && (tid - Pl.nvt) < 32, sHb, sPb);
    }
    // x = 0, r = −g, z = M⁻¹ r, d = z (d lives in shared memory: the SpMV gathers neighbours' d)
    if (vown) {
      x = mk(0, 0, 0);
      r = -ld3(g + 3 * v);
      uu = mk(Ps[0] * r.x + Ps[1] * r.y + Ps[2] * r.z, Ps[3] * r.x + Ps[4] * r.y + Ps[5] * r.z,
              Ps[6] * r.x + Ps[7] * r.y + Ps[8] * r.z);          // uu = d
      st3(usm + 3 * vl, uu);
    }
    double zb = 0.0;
    if (bown) {
      xb = 0.0;
      rb = -g[3 * V + 12 * bd + brow];
    }
    if (!vt) {
      double z_ = 0.0;
#pragma unroll
      for (int c = 0; c < 12; ++c) z_ += (bown ? sPb[144 * bd + 12 * brow + c] : 0.0) * __shfl_sync(0xffffffffu, rb, hl | c);
      zb = z_;
      ubr = z_;                                                    // d_b = z_b
      if (bown) ub[12 * bd + brow] = ubr;
    }
    double rz;
    {
      double a0 = vown ? dot(r, uu) : 0.0, b0 = 0.0;
      if (bown) a0 = rb * zb;
      cl_sum2<NC>(a0, b0, red, rred, 0);
      rz = a0;
    }
    const double eta_k = pcg_forcing(D, C, rz), stop = eta_k * eta_k * rz;   // R24 (fixed η by default)
    rz0_used = rz; eta_used = eta_k;
    zero_g = rz == 0.0;
    bad = !(rz == rz);
    if constexpr (NC > 1) {
      for (int i = tid; i < 12 * ND; i += blockDim.x) ub[i] = ub0[i];
    }
    __syncthreads();
    int it = 0;
    while (!bad && it < D.max_pcg && rz > stop) {
      // ---------------- q = (H + μM) d and the partials of dᵀq
      double dloc = 0.0;
      v3 w = mk(0, 0, 0);
      if (vown) {
        const double* hd = sHd + vl;
        w = mk(hd[0] * uu.x + hd[rpr] * uu.y + hd[2 * rpr] * uu.z, hd[3 * rpr] * uu.x + hd[4 * rpr] * uu.y + hd[5 * rpr] * uu.z,
               hd[6 * rpr] * uu.x + hd[7 * rpr] * uu.y + hd[8 * rpr] * uu.z);
        const int j1 = rp[vl + 1];
#pragma unroll 2
        for (int j = rp[vl]; j < j1; ++j) {
          const int2 bk = blk[j];
          const double* Bk = U + 9 * (bk.x >> 1);
          const v3 uj = uv_at(bk.y);
          w += (bk.x & 1) ? mul33T(Bk, uj) : mul33(Bk, uj);
        }
        if (mu != 0.0) w += (mu * mv) * uu;
        double cu = 0.0;                                  // d_vᵀ C d_b (counted again for the body side)
        for (int c = cpp[vl] - c0, c1 = cpp[vl + 1] - c0; c < c1; ++c) {
          const int d = cstaged ? cpld[c] : cd_g[c0 + c];
          const double* ud = ub + 12 * d;
          v3 cu3 = mk(0, 0, 0);
#pragma unroll
          for (int b = 0; b < 12; ++b) {
            const double ubb = ud[b];
            const double a0 = cstaged ? cval[(size_t)b * Pl.cplcap + c] : cv_g[(size_t)b * D.cpl_cap + c0 + c];
            const double a1 = cstaged ? cval[(size_t)(12 + b) * Pl.cplcap + c] : cv_g[(size_t)(12 + b) * D.cpl_cap + c0 + c];
            const double a2 = cstaged ? cval[(size_t)(24 + b) * Pl.cplcap + c] : cv_g[(size_t)(24 + b) * D.cpl_cap + c0 + c];
            cu3 += mk(a0 * ubb, a1 * ubb, a2 * ubb);
          }
          w += cu3;
          cu += dot(uu, cu3);
        }
        dloc = dot(uu, w) + cu;
      }
      // body coupling partials Σ_c Cᵀ d_v per warp (fixed butterfly), one body at a time
      if (vt && ND > 0) {
        int cb = vown ? cpp[vl] - c0 : 0, ce = vown ? cpp[vl + 1] - c0 : 0;
        for (int d = 0; d < ND; ++d) {
          double ob[12];
#pragma unroll
          for (int i = 0; i < 12; ++i) ob[i] = 0.0;
          bool mine = false;
          for (int c = cb; c < ce; ++c) {
            const int dd = cstaged ? cpld[c] : cd_g[c0 + c];
            if (dd != d) continue;
            mine = true;
#pragma unroll
            for (int b = 0; b < 12; ++b) {
              const double a0 = cstaged ? cval[(size_t)b * Pl.cplcap + c] : cv_g[(size_t)b * D.cpl_cap + c0 + c];
              const double a1 = cstaged ? cval[(size_t)(12 + b) * Pl.cplcap + c] : cv_g[(size_t)(12 + b) * D.cpl_cap + c0 + c];
              const double a2 = cstaged ? cval[(size_t)(24 + b) * Pl.cplcap + c] : cv_g[(size_t)(24 + b) * D.cpl_cap + c0 + c];
              ob[b] += a0 * uu.x + a1 * uu.y + a2 * uu.z;
            }
          }
          const unsigned any = __ballot_sync(0xffffffffu, mine);
          if (any) {
#pragma unroll
            for (int i = 0; i < 12; ++i) ob[i] = warp_sum(ob[i]);
          }
          if (lane == 0) {
            double* wp = wpart + ((size_t)(tid >> 5) * ND + d) * 12;
#pragma unroll
            for (int i = 0; i < 12; ++i) wp[i] = any ? ob[i] : 0.0;
          }
        }
      } else if (!vt) {
        for (int i = lane; i < 12 * ND; i += 32) wpart[(size_t)(tid >> 5) * ND * 12 + i] = 0.0;
      }
      // residual pairs (CTA 0): outputs to sout (soft slots) and the warp partials (body slots)
      if (rank == 0 && nres > 0) dloc += cl_residual_pairs<NC>(D, e, nres, rpr, usm, ub, wpart, ru);
      // body rows (CTA 0): own part (H_b + μM) d_b
      double wb = 0.0;
      if (!vt) {
        double hu = 0.0;
#pragma unroll
        for (int c = 0; c < 12; ++c) {
          const double uc = __shfl_sync(0xffffffffu, ubr, hl | c);
          hu += (bown ? sHb[144 * bd + 12 * brow + c] : 0.0) * uc;
        }
        if (bown) {
          wb = hu;
          dloc += ubr * hu;
        }
      }
      // per-CTA body partial (clusters): Σ over warps in order, read by CTA 0 after barrier A
      if constexpr (NC > 1) {
        __syncthreads();
        for (int i = tid; i < 12 * ND; i += blockDim.x) {
          double t = 0.0;
          for (int k = 0; k < nw; ++k) t += wpart[(size_t)k * ND * 12 + i];
          pbody[i] = t;
        }
      }
      // ---------------- barrier A: dᵀq over the cluster → α
      double dq = dloc, unused = 0.0;
      cl_sum2<NC>(dq, unused, red, rred, 0);
      if (!(dq > 0.0)) { bad = true; break; }            // not SPD along d (uniform over the cluster)
      const double alpha = rz / dq;
      double rzl = 0.0;
      if (vown) {
        for (int j = ccp[v], j1 = ccp[v] + rcn[v]; j < j1; ++j) w += ld3(sout + 3 * j);   // residual pair outputs
        x += alpha * uu;
        r = r - alpha * w;
        pp = mk(Ps[0] * r.x + Ps[1] * r.y + Ps[2] * r.z, Ps[3] * r.x + Ps[4] * r.y + Ps[5] * r.z,
                Ps[6] * r.x + Ps[7] * r.y + Ps[8] * r.z);          // pp = z
        rzl = dot(r, pp);
      }
      if (!vt) {
        if (bown) {
          if constexpr (NC == 1) {
            for (int k = 0; k < nw; ++k) wb += wpart[((size_t)k * ND + bd) * 12 + brow];
          } else {
#pragma unroll
            for (int rr = 0; rr < NC; ++rr) wb += rpb[rr][12 * bd + brow];
          }
          xb += alpha * ubr;
          rb -= alpha * wb;
        }
        double z_ = 0.0;
#pragma unroll
        for (int c = 0; c < 12; ++c) z_ += (bown ? sPb[144 * bd + 12 * brow + c] : 0.0) * __shfl_sync(0xffffffffu, rb, hl | c);
        zb = z_;
        if (bown) rzl = rb * zb;
      }
      // ---------------- barrier B: rᵀz over the cluster → β
      double rzn = rzl, unused2 = 0.0;
      cl_sum2<NC>(rzn, unused2, red, rred, 1);
      const double beta = rzn / rz;
      rz = rzn;
      ++it;
      if (!(rz == rz)) { bad = true; break; }
      if (vown) {
        uu = pp + beta * uu;
        st3(usm + 3 * vl, uu);
      }
      if (bown) {
        ubr = zb + beta * ubr;
        ub[12 * bd + brow] = ubr;
      }
      // ---------------- barrier C: d (and the bodies' d) visible to the cluster
      cl_barrier<NC>();
      if constexpr (NC > 1) {
        for (int i = tid; i < 12 * ND; i += blockDim.x) ub[i] = ub0[i];
        __syncthreads();
      }
    }
    it_total += it;
    cl_barrier<NC>();                                   // every read of the last reduction's values is done
    // gᵀx over the cluster (descent test of the LM rule)
    double gl = 0.0, dummy = 0.0;
    if (vown) gl = dot(ld3(g + 3 * v), x);
    if (bown) gl = g[3 * V + 12 * bd + brow] * xb;
    cl_sum2<NC>(gl, dummy, red, rred, 1);
    gp = gl;
    if (D.hmode != 2 || (!bad && (gp < 0.0 || zero_g)) || mu > 1e12) break;
    mu = fmax(D.lm_mu0, 10.0 * mu);
    bad = false;
    cl_barrier<NC>();                                   // totals read before the next attempt rewrites them
  }
  // write the direction; CTA 0 finishes (norm, step cap, statistics) after the cluster barrier
  double* p_out = D.p + (size_t)e * n;
  if (vown) st3(p_out + 3 * v, x);
  if (bown) p_out[3 * V + 12 * bd + brow] = xb;
  __threadfence();
  cl_barrier<NC>();
  if (rank != 0) return;
  if (threadIdx.x == 0 && !bad && rz0_used > 0.0) { C.ew_rz0 = rz0_used; C.ew_eta = eta_used; C.ew_has = 1; }
  pcg_finish_noinline(D, e, p_out, red, mu, bad, zero_g, it_total, gp);
}

}  // namespace tac
