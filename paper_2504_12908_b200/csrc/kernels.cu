// kernels.cu — sm_100a fp64 kernels of the batched IPC + ABD Newton step.
// One CTA per environment for every per-env phase (envs are independent); per-env
// reductions are deterministic block reductions with a fixed thread→element assignment, so every
// env's result is bitwise independent of the batch size and of how envs are sharded.
#include <algorithm>
#include <cfloat>
#include <climits>
#include "eigen.cuh"
#include "elastic.cuh"
#include "geometry.cuh"
#include "impl.cuh"
#include "launch.h"
#include <cstdlib>

namespace tac {

// ------------------------------------------------------------------------------------------
// small helpers
// ------------------------------------------------------------------------------------------
__device__ __forceinline__ const double* body_y(const Dev& D, int e, int b) {
  int s = D.dof_slot[b];
  return s >= 0 ? D.q + (size_t)e * D.n + 3 * D.V + 12 * s : D.ystat + ((size_t)e * D.NA + b) * 12;
}
__device__ __forceinline__ double* envp(double* base, int e, size_t per) { return base + (size_t)e * per; }
// env of a CTA: env0 + b, or the b-th entry of the compacted active-env list of this Newton iteration
__device__ __forceinline__ int env_at(const Dev& D, int env0, int b) { return D.elist ? D.elist[b] : env0 + b; }
// append env e to the active-env list of the next Newton iteration (order is irrelevant: every per-env
// result depends only on the env) and count it
__device__ __forceinline__ void mark_active(const Dev& D, int e) {
  const int slot = atomicAdd(D.any_active, 1);
  if (D.elist_out) {
    D.elist_out[slot] = e;
    // PCG split (per env, from its own history only → batch-independent): envs in the long tail of a
    // step (≥ tail_newton Newton iterations) solve with the cluster-resident kernel, the rest streamed
    if (D.tail_newton > 0) {
      const bool tail = D.ctl[e].newton >= D.tail_newton;
      const int s2 = atomicAdd(D.any_active + (tail ? 1 : 2), 1);
      D.elist_out[(size_t)D.E * (tail ? 1 : 2) + s2] = e;
    }
  }
}

// f-factor of the affine Jacobian: column α of J_v is e_{i(α)} scaled by f(α) (1 for t, x̄_j for A_ij)
__device__ __forceinline__ int jrow(int alpha) { return alpha < 3 ? alpha : (alpha - 3) / 3; }
__device__ __forceinline__ double jf(int alpha, const double* xb) { return alpha < 3 ? 1.0 : xb[(alpha - 3) % 3]; }

__device__ __forceinline__ void pair_vids(const Dev& D, int kind, int a, int b, int* vid) {
  if (kind == 0) {
    vid[0] = a; vid[1] = D.tris[3 * b]; vid[2] = D.tris[3 * b + 1]; vid[3] = D.tris[3 * b + 2];
  } else {
    vid[0] = D.edges[2 * a]; vid[1] = D.edges[2 * a + 1]; vid[2] = D.edges[2 * b]; vid[3] = D.edges[2 * b + 1];
  }
}
__device__ __forceinline__ double pair_area(const Dev& D, int kind, int a, int b) {
  return kind == 0 ? D.A_v[a] : 0.5 * (D.A_e[a] + D.A_e[b]);
}
__device__ __forceinline__ double pair_eps(const Dev& D, int kind, int a, int b) {
  return kind == 0 ? 1.0 : 1e-3 * D.elen2[a] * D.elen2[b];
}

// distance between the axis-aligned boxes of the pair's two primitives (PT: {x0} vs {x1,x2,x3}; EE:
// {x0,x1} vs {x2,x3}) — a lower bound of the primitive distance, used to skip exact classification
// where it cannot change a result
__device__ __forceinline__ double prim_box_dist(int kind, const v3* X) {
  v3 alo = X[0], ahi = X[0], blo = X[3], bhi = X[3];
  if (kind == 1) { alo = vmin(alo, X[1]); ahi = vmax(ahi, X[1]); }
  else { blo = vmin(blo, X[1]); bhi = vmax(bhi, X[1]); }
  blo = vmin(blo, X[2]); bhi = vmax(bhi, X[2]);
  const double gx = fmax(0.0, fmax(blo.x - ahi.x, alo.x - bhi.x));
  const double gy = fmax(0.0, fmax(blo.y - ahi.y, alo.y - bhi.y));
  const double gz = fmax(0.0, fmax(blo.z - ahi.z, alo.z - bhi.z));
  return sqrt(gx * gx + gy * gy + gz * gz);
}

__device__ __forceinline__ bool env_skip(const Dev& D, int e, int force) {
  return !force && D.ctl[e].phase != PHASE_ACTIVE;
}

// packed-upper (r,c) table for 12×12
__constant__ unsigned char c_unpack_r[PH], c_unpack_c[PH];

// ------------------------------------------------------------------------------------------
// positions: P = φ(q) for every contact vertex; Pd = displacement of p (J_v p_b for bodies)
// ------------------------------------------------------------------------------------------
__device__ double embedded_inf_norm(const Dev& D, int e, const double* p, double* red) {
  double pm = 0.0;
  for (int i = threadIdx.x; i < 3 * D.V; i += blockDim.x) pm = fmax(pm, fabs(p[i]));
  for (int i = threadIdx.x; i < D.NAV; i += blockDim.x) {
    int gv = D.affv_list[i];
    int sl = D.dof_slot[D.vert_aff[gv]];
    v3 u = embed(p + 3 * D.V + 12 * sl, ld3(D.vert_xbar + 3 * gv));
    pm = fmax(pm, fmax(fabs(u.x), fmax(fabs(u.y), fabs(u.z))));
  }
  return block_max(pm, red);
}

// K_eff (reading R17b): largest power of two ≤ ls_expand with K_eff·‖p‖_emb,∞ ≤ d̂
__device__ __forceinline__ double sweep_factor(const Dev& D, double pinf) {
  double K = 1.0;
  while (2.0 * K <= D.K && 2.0 * K * pinf <= D.dhat) K *= 2.0;
  return K;
}

__global__ void __launch_bounds__(NTHREADS) k_positions(Dev D, int env0, int with_p, int force) {
  const int e = env_at(D, env0, blockIdx.x);
  if (env_skip(D, e, force)) return;
  __shared__ double red[32];
  const double* q = D.q + (size_t)e * D.n;
  const double* p = D.p + (size_t)e * D.n;
  double* P = D.P + (size_t)e * D.NVall * 3;
  double* Pd = D.Pd + (size_t)e * D.NVall * 3;
  double Kf = 1.0;
  if (with_p) {
    Kf = sweep_factor(D, embedded_inf_norm(D, e, p, red));
    if (threadIdx.x == 0) D.ctl[e].Keff = Kf;
  }
  for (int gv = threadIdx.x; gv < D.NVall; gv += blockDim.x) {
    if (gv < D.V) {
      P[3 * gv] = q[3 * gv]; P[3 * gv + 1] = q[3 * gv + 1]; P[3 * gv + 2] = q[3 * gv + 2];
      // (validity of a reusable candidate list is checked below, after all positions exist)
      // Pd = K_eff·(displacement of p): the swept sets and ACCD cover α ∈ [0, K_eff]
      if (with_p) { Pd[3 * gv] = Kf * p[3 * gv]; Pd[3 * gv + 1] = Kf * p[3 * gv + 1]; Pd[3 * gv + 2] = Kf * p[3 * gv + 2]; }
    } else {
      int b = D.vert_aff[gv];
      v3 xb = ld3(D.vert_xbar + 3 * gv);
      st3(P + 3 * gv, embed(body_y(D, e, b), xb));
      if (with_p) {
        int s = D.dof_slot[b];
        v3 d = mk(0, 0, 0);
        if (s >= 0) d = embed(p + 3 * D.V + 12 * s, xb);
        st3(Pd + 3 * gv, Kf * d);
      }
    }
  }
  // reading R11b: the candidate list stays valid while every surface vertex's current sweep
  // [P, P + Pd] lies inside its reference box grown by δ
  if (D.bp_margin > 0.0) {
    __syncthreads();
    const double* rb = D.vref + (size_t)e * D.NSV * 6;
    const double dm = D.bp_margin;
    int ok = D.ctl[e].bp_ref;
    if (ok) {
      for (int i = threadIdx.x; i < D.NSV; i += blockDim.x) {
        const int gv = D.sverts[i];
        v3 a = ld3(P + 3 * gv), b = a;
        if (with_p) b = a + ld3(Pd + 3 * gv);
        const double* r = rb + 6 * i;
        if (!(fmin(a.x, b.x) >= r[0] - dm && fmin(a.y, b.y) >= r[1] - dm && fmin(a.z, b.z) >= r[2] - dm &&
              fmax(a.x, b.x) <= r[3] + dm && fmax(a.y, b.y) <= r[4] + dm && fmax(a.z, b.z) <= r[5] + dm))
          ok = 0;
      }
    }
    ok = __syncthreads_and(ok);
    if (threadIdx.x == 0) D.ctl[e].bp_valid = ok;
  }
}

// ------------------------------------------------------------------------------------------
// broad phase: per-env spatial hash (shared-memory bucket table), deterministic candidate list
// ------------------------------------------------------------------------------------------
struct Grid {
  double ox, oy, oz, inv_h;
  __device__ int ci(double x, double o) const {
    double f = floor((x - o) * inv_h);
    int i = (int)fmin(fmax(f, 0.0), 1023.0);
    return i;
  }
  __device__ void cell(v3 p, int* c) const { c[0] = ci(p.x, ox); c[1] = ci(p.y, oy); c[2] = ci(p.z, oz); }
};
// bucket of (cell, target kind): triangles and edges of the same cell hash apart, so a PT query only
// scans triangle entries and an EE query only edge entries (up to collisions)
__device__ __forceinline__ unsigned hcell(int i, int j, int k, int kind) {
  return (((unsigned)i * 73856093u) ^ ((unsigned)j * 19349663u) ^ ((unsigned)k * 83492791u) ^ (kind ? 0x9E3779B9u : 0u)) &
         (NBUCKET - 1);
}
constexpr int ENT_CODE_BITS = 26;
constexpr int QTMP = 32;              // per-query candidate slot of the broad phase (larger: re-run)      // hash entry: target code (2t + kind) | body id << 26
__device__ __forceinline__ int ccode(int i, int j, int k) { return i | (j << 10) | (k << 20); }

struct BoxCtx {
  const double* P; const double* Pd; int swept;
  double* tb;      // raw target boxes [NT+NE][6] (lo, hi), filled in pass 1 of k_broad
  int NT;
  double infl;     // target inflation: d̂ (exact) or d̂ + 2δ (reusable list, reading R11b)
  __device__ void vbox(int gv, v3& lo, v3& hi) const {
    v3 a = ld3(P + 3 * gv);
    lo = a; hi = a;
    if (swept) {
      v3 d = ld3(Pd + 3 * gv);
      v3 b = a + d;
      lo = vmin(lo, b); hi = vmax(hi, b);
    }
  }
  __device__ void box(const int* vs, int nv, v3& lo, v3& hi) const {
    vbox(vs[0], lo, hi);
    for (int i = 1; i < nv; ++i) { v3 l, h; vbox(vs[i], l, h); lo = vmin(lo, l); hi = vmax(hi, h); }
  }
};

__device__ __forceinline__ bool overlap(v3 qlo, v3 qhi, v3 tlo_i, v3 thi_i) {
  // query box raw, target box already inflated by d̂: lo_q ≤ hi_t + d̂ and lo_t − d̂ ≤ hi_q
  return qlo.x <= thi_i.x && qlo.y <= thi_i.y && qlo.z <= thi_i.z && tlo_i.x <= qhi.x && tlo_i.y <= qhi.y &&
         tlo_i.z <= qhi.z;
}

__device__ __forceinline__ int tbox_index(const BoxCtx& B, int code) { return (code & 1) ? B.NT + (code >> 1) : (code >> 1); }
__device__ __forceinline__ void raw_target_box(const Dev& D, const BoxCtx& B, int code, v3& lo, v3& hi) {
  int t = code >> 1;
  if ((code & 1) == 0) B.box(D.tris + 3 * t, 3, lo, hi);
  else B.box(D.edges + 2 * t, 2, lo, hi);
}
// inflated (by d̂) box of a target from the cache
__device__ __forceinline__ void target_box(const Dev& D, const BoxCtx& B, int code, v3& lo, v3& hi) {
  const double* c = B.tb + 6 * (size_t)tbox_index(B, code);
  lo = mk(c[0], c[1], c[2]); hi = mk(c[3], c[4], c[5]);
  v3 dh = mk(B.infl, B.infl, B.infl);
  lo = lo - dh; hi = hi + dh;
}

constexpr int MAXB = 32;   // bodies per env (pads + affine)
// body-level culling (exact: the box predicate is monotone).  A target (inflated box) can only
// meet queries of bodies whose raw box it overlaps; a query (raw box) only targets inside some
// allowed body's box grown by the inflation.
__device__ __forceinline__ bool target_reaches(const Dev& D, double (*bb)[6], int tbody, v3 tlo_i, v3 thi_i) {
  for (int b = 0; b < D.NB; ++b) {
    if (!D.allowed[(size_t)b * D.NB + tbody]) continue;
    if (bb[b][0] <= thi_i.x && bb[b][1] <= thi_i.y && bb[b][2] <= thi_i.z && tlo_i.x <= bb[b][3] &&
        tlo_i.y <= bb[b][4] && tlo_i.z <= bb[b][5])
      return true;
  }
  return false;
}
__device__ __forceinline__ bool query_reaches(const Dev& D, double (*bb)[6], int qbody, v3 qlo, v3 qhi, double infl) {
  for (int b = 0; b < D.NB; ++b) {
    if (!D.allowed[(size_t)qbody * D.NB + b]) continue;
    if (qlo.x <= bb[b][3] + infl && qlo.y <= bb[b][4] + infl && qlo.z <= bb[b][5] + infl &&
        bb[b][0] - infl <= qhi.x && bb[b][1] - infl <= qhi.y && bb[b][2] - infl <= qhi.z)
      return true;
  }
  return false;
}

template <bool EMIT>
__device__ int bp_query(const Dev& D, const BoxCtx& B, const Grid& G, const int* cnt_off, const int* ent, const int* big,
                        int nbig, int qi, int* out_a, int* out_b, double (*bb)[6], int out_cap = INT_MAX) {
  const bool pt = qi < D.NSV;
  int qa, qbody;
  v3 qlo, qhi;
  if (pt) {
    qa = D.sverts[qi];
    qbody = D.vert_body[qa];
    B.vbox(qa, qlo, qhi);
  } else {
    qa = qi - D.NSV;
    qbody = D.edge_body[qa];
    const double* c = B.tb + 6 * (size_t)(B.NT + qa);
    qlo = mk(c[0], c[1], c[2]); qhi = mk(c[3], c[4], c[5]);
  }
  const int want = pt ? 0 : 1;
  if (!query_reaches(D, bb, qbody, qlo, qhi, B.infl)) return 0;
  const unsigned char* allow = D.allowed + (size_t)qbody * D.NB;
  unsigned amask = 0u;                 // bodies this query may touch (NB ≤ MAXB = 32)
  for (int b = 0; b < D.NB; ++b) amask |= allow[b] ? (1u << b) : 0u;
  int lo[3], hi[3];
  G.cell(qlo, lo); G.cell(qhi, hi);
  long ncell = (long)(hi[0] - lo[0] + 1) * (hi[1] - lo[1] + 1) * (hi[2] - lo[2] + 1);
  int count = 0;
  const int kindbit = pt ? 0 : (1 << 30);
  auto accept = [&](int code, v3 tlo, v3 thi) {
    if (EMIT && count < out_cap) { out_a[count] = kindbit | qa; out_b[count] = code >> 1; }
    ++count;
  };
  if (ncell > 4096) {  // huge query box: brute force over all targets of the kind
    int ntg = pt ? D.NT : D.NE;
    for (int t = 0; t < ntg; ++t) {
      if (!pt && t <= qa) continue;
      int tb = pt ? D.tri_body[t] : D.edge_body[t];
      if (!allow[tb]) continue;
      int code = 2 * t + want;
      v3 tlo, thi;
      target_box(D, B, code, tlo, thi);
      if (overlap(qlo, qhi, tlo, thi)) accept(code, tlo, thi);
    }
    return count;
  }
  for (int x = lo[0]; x <= hi[0]; ++x)
    for (int y = lo[1]; y <= hi[1]; ++y)
      for (int z = lo[2]; z <= hi[2]; ++z) {
        unsigned h = hcell(x, y, z, want);
        int cc = ccode(x, y, z);
        for (int j = cnt_off[h]; j < cnt_off[h + 1]; ++j) {
          if (ent[2 * j + 1] != cc) continue;
          const int e0 = ent[2 * j];
          const int code = e0 & ((1 << ENT_CODE_BITS) - 1);
          if ((code & 1) != want) continue;
          int t = code >> 1;
          if (!pt && t <= qa) continue;
          if (!((amask >> (e0 >> ENT_CODE_BITS)) & 1u)) continue;
          v3 tlo, thi;
          target_box(D, B, code, tlo, thi);
          if (!overlap(qlo, qhi, tlo, thi)) continue;
          int tl[3];
          G.cell(tlo, tl);
          if (max(lo[0], tl[0]) != x || max(lo[1], tl[1]) != y || max(lo[2], tl[2]) != z) continue;
          accept(code, tlo, thi);
        }
      }
  for (int j = 0; j < nbig; ++j) {
    int code = big[j];
    if ((code & 1) != want) continue;
    int t = code >> 1;
    if (!pt && t <= qa) continue;
    int tb = pt ? D.tri_body[t] : D.edge_body[t];
    if (!allow[tb]) continue;
    v3 tlo, thi;
    target_box(D, B, code, tlo, thi);
    if (overlap(qlo, qhi, tlo, thi)) accept(code, tlo, thi);
  }
  return count;
}

constexpr int BROAD_THREADS = 512;
__global__ void __launch_bounds__(BROAD_THREADS) k_broad(Dev D, int env0, int swept, int force) {
  const int e = env_at(D, env0, blockIdx.x);
  EnvCtl& C = D.ctl[e];
  if (!force && (C.phase != PHASE_ACTIVE || (swept && (C.inner_conv || C.xfail)))) return;
  // reading R11b: reuse the candidate list while every surface vertex stays within δ of the
  // reference box it had at the last (margin-inflated) build
  if (!force && D.bp_margin > 0.0 && C.bp_valid) return;
  const double margin = force ? 0.0 : D.bp_margin;
  __shared__ int cnt[NBUCKET + 1];
  __shared__ int cur[NBUCKET];
  __shared__ int sh[33];
  __shared__ int nbig_s, ovf_s, next_q;
  BoxCtx B{D.P + (size_t)e * D.NVall * 3, D.Pd + (size_t)e * D.NVall * 3, swept,
           D.tbox + (size_t)e * (D.NT + D.NE) * 6, D.NT, D.dhat + 2.0 * margin};
  // reference boxes of the surface vertices for the reuse test
  if (margin > 0.0) {
    double* rb = D.vref + (size_t)e * D.NSV * 6;
    for (int i = threadIdx.x; i < D.NSV; i += blockDim.x) {
      v3 lo, hi;
      B.vbox(D.sverts[i], lo, hi);
      rb[6 * i] = lo.x; rb[6 * i + 1] = lo.y; rb[6 * i + 2] = lo.z; rb[6 * i + 3] = hi.x; rb[6 * i + 4] = hi.y; rb[6 * i + 5] = hi.z;
    }
  }
  if (threadIdx.x == 0) C.bp_ref = margin > 0.0 ? 1 : 0;
  int* ent = D.ent + (size_t)e * D.ent_cap * 2;
  int* big = D.big + (size_t)e * BIG_CAP;
  // body boxes (surface vertices of each body are a contiguous range of sverts): warp per body
  __shared__ double bb[MAXB][6];
  {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
    for (int b = w; b < D.NB; b += nw) {
      double l0 = 1e300, l1 = 1e300, l2 = 1e300, h0 = -1e300, h1 = -1e300, h2 = -1e300;
      for (int i = D.body_sv_ptr[b] + lane; i < D.body_sv_ptr[b + 1]; i += 32) {
        v3 lo, hi;
        B.vbox(D.sverts[i], lo, hi);
        l0 = fmin(l0, lo.x); l1 = fmin(l1, lo.y); l2 = fmin(l2, lo.z);
        h0 = fmax(h0, hi.x); h1 = fmax(h1, hi.y); h2 = fmax(h2, hi.z);
      }
      l0 = warp_min(l0); l1 = warp_min(l1); l2 = warp_min(l2);
      h0 = warp_max(h0); h1 = warp_max(h1); h2 = warp_max(h2);
      if (lane == 0) { bb[b][0] = l0; bb[b][1] = l1; bb[b][2] = l2; bb[b][3] = h0; bb[b][4] = h1; bb[b][5] = h2; }
    }
  }
  __syncthreads();
  // grid origin: min corner over all bodies
  double mx = 1e300, my = 1e300, mz = 1e300;
  for (int b = 0; b < D.NB; ++b) { mx = fmin(mx, bb[b][0]); my = fmin(my, bb[b][1]); mz = fmin(mz, bb[b][2]); }
  Grid G;
  G.ox = mx - B.infl;
  G.oy = my - B.infl;
  G.oz = mz - B.infl;
  G.inv_h = 1.0 / D.cell;
  for (int i = threadIdx.x; i <= NBUCKET; i += blockDim.x) cnt[i] = 0;
  if (threadIdx.x == 0) { nbig_s = 0; ovf_s = 0; }
  __syncthreads();
  const int ntarget = D.NT + D.NE;
  // pass 1: raw boxes of every target into the cache; count cell entries (inflated box)
  for (int i = threadIdx.x; i < ntarget; i += blockDim.x) {
    int code = i < D.NT ? 2 * i : 2 * (i - D.NT) + 1;
    v3 lo, hi;
    raw_target_box(D, B, code, lo, hi);
    double* c = B.tb + 6 * (size_t)i;
    c[0] = lo.x; c[1] = lo.y; c[2] = lo.z; c[3] = hi.x; c[4] = hi.y; c[5] = hi.z;
    v3 dh = mk(B.infl, B.infl, B.infl);
    lo = lo - dh; hi = hi + dh;
    if (!target_reaches(D, bb, i < D.NT ? D.tri_body[i] : D.edge_body[i - D.NT], lo, hi)) continue;
    int l[3], h[3];
    G.cell(lo, l); G.cell(hi, h);
    long nc = (long)(h[0] - l[0] + 1) * (h[1] - l[1] + 1) * (h[2] - l[2] + 1);
    if (nc > MAXCELLS) {
      int k = atomicAdd(&nbig_s, 1);
      if (k < BIG_CAP) big[k] = code; else ovf_s |= 2;
      continue;
    }
    for (int x = l[0]; x <= h[0]; ++x)
      for (int y = l[1]; y <= h[1]; ++y)
        for (int z = l[2]; z <= h[2]; ++z) atomicAdd(&cnt[hcell(x, y, z, code & 1)], 1);
  }
  __syncthreads();
  // exclusive scan of bucket counts (16 per thread for 256 threads)
  {
    const int per = (NBUCKET + blockDim.x - 1) / blockDim.x;
    int b0 = threadIdx.x * per;
    int s = 0;
    for (int i = 0; i < per && b0 + i < NBUCKET; ++i) s += cnt[b0 + i];
    int tot;
    int ex = block_excl_scan(s, sh, &tot);
    int run = ex;
    for (int i = 0; i < per && b0 + i < NBUCKET; ++i) {
      int c = cnt[b0 + i];
      cnt[b0 + i] = run;
      cur[b0 + i] = run;
      run += c;
    }
    __syncthreads();
    if (threadIdx.x == 0) cnt[NBUCKET] = tot;
    if (tot > D.ent_cap && threadIdx.x == 0) ovf_s |= 4;
    __syncthreads();
  }
  if (ovf_s) {
    if (threadIdx.x == 0) { C.overflow |= ovf_s; C.cap_seen = ovf_s; C.ncand = 0; }
    return;
  }
  // pass 2: fill entries
  for (int i = threadIdx.x; i < ntarget; i += blockDim.x) {
    int code = i < D.NT ? 2 * i : 2 * (i - D.NT) + 1;
    v3 lo, hi;
    target_box(D, B, code, lo, hi);
    if (!target_reaches(D, bb, i < D.NT ? D.tri_body[i] : D.edge_body[i - D.NT], lo, hi)) continue;
    int l[3], h[3];
    G.cell(lo, l); G.cell(hi, h);
    long nc = (long)(h[0] - l[0] + 1) * (h[1] - l[1] + 1) * (h[2] - l[2] + 1);
    if (nc > MAXCELLS) continue;
    for (int x = l[0]; x <= h[0]; ++x)
      for (int y = l[1]; y <= h[1]; ++y)
        for (int z = l[2]; z <= h[2]; ++z) {
          int pos = atomicAdd(&cur[hcell(x, y, z, code & 1)], 1);
          ent[2 * pos] = code | ((i < D.NT ? D.tri_body[i] : D.edge_body[i - D.NT]) << ENT_CODE_BITS);
          ent[2 * pos + 1] = ccode(x, y, z);
        }
  }
  __syncthreads();
  const int nbig = min(nbig_s, BIG_CAP);
  // queries: PT (surface vertices) then EE (edges).  Each query runs once, emitting into a private
  // slot of QTMP entries (sorted by target there) and recording its count; one block scan in query
  // order; then the slots are copied to the candidate list.  A query with more than QTMP candidates
  // is re-run straight into the list.
  int* ca = D.cand_a + (size_t)e * D.cand_cap;
  int* cb = D.cand_b + (size_t)e * D.cand_cap;
  const int nq = D.NSV + D.NE;
  int* qc = D.qcnt + (size_t)e * (D.NSV + D.NE);
  int* qta = D.qtmp + (size_t)e * (D.NSV + D.NE) * 2 * QTMP;
  auto sort_seg = [](int* sa, int* sb, int c) {           // insertion sort by target index
    for (int i = 1; i < c; ++i) {
      int kb = sb[i], ka = sa[i];
      int j = i - 1;
      while (j >= 0 && sb[j] > kb) { sb[j + 1] = sb[j]; sa[j + 1] = sa[j]; --j; }
      sb[j + 1] = kb; sa[j + 1] = ka;
    }
  };
  // queries handed out 32 at a time to warps (dynamic balance; each query's output depends only on qi)
  if (threadIdx.x == 0) next_q = 0;
  __syncthreads();
  for (;;) {
    int qb = 0;
    if ((threadIdx.x & 31) == 0) qb = atomicAdd(&next_q, 32);
    qb = __shfl_sync(0xffffffffu, qb, 0);
    if (qb >= nq) break;
    const int qi = qb + (threadIdx.x & 31);
    if (qi >= nq) continue;
    int* ta = qta + (size_t)qi * 2 * QTMP;
    const int c = bp_query<true>(D, B, G, cnt, ent, big, nbig, qi, ta, ta + QTMP, bb, QTMP);
    if (c <= QTMP) sort_seg(ta, ta + QTMP, c);
    qc[qi] = c;
  }
  __syncthreads();
  int total;
  {
    const int per = (nq + blockDim.x - 1) / blockDim.x;
    const int q0 = min((int)threadIdx.x * per, nq), q1 = min(q0 + per, nq);
    int sum = 0;
    for (int q = q0; q < q1; ++q) sum += qc[q];
    int ex = block_excl_scan(sum, sh, &total);
    for (int q = q0; q < q1; ++q) { const int c = qc[q]; qc[q] = ex; ex += c; }
  }
  __syncthreads();
  if (threadIdx.x == 0) next_q = 0;
  __syncthreads();
  for (;;) {
    int qb = 0;
    if ((threadIdx.x & 31) == 0) qb = atomicAdd(&next_q, 32);
    qb = __shfl_sync(0xffffffffu, qb, 0);
    if (qb >= nq) break;
    const int qi = qb + (threadIdx.x & 31);
    if (qi >= nq) continue;
    const int base = qc[qi], c = (qi + 1 < nq ? qc[qi + 1] : total) - base;
    if (c <= 0 || base + c > D.cand_cap) continue;
    if (c <= QTMP) {
      const int* ta = qta + (size_t)qi * 2 * QTMP;
      for (int i = 0; i < c; ++i) { ca[base + i] = ta[i]; cb[base + i] = ta[QTMP + i]; }
    } else {
      bp_query<true>(D, B, G, cnt, ent, big, nbig, qi, ca + base, cb + base, bb);
      sort_seg(ca + base, cb + base, c);
    }
  }
  if (threadIdx.x == 0) {
    C.ncand = min(total, D.cand_cap);
    if (total > D.cand_cap) { C.overflow |= 1; C.cap_seen |= 1; C.cap_need = max(C.cap_need, total); }
  }
}

// ------------------------------------------------------------------------------------------
// lagged friction (reading R20): at the first narrow phase of a step (positions = xⁿ) the
// barrier's active pairs are frozen as friction pairs — contact normal n̂ and closest-point weights Γ
// (PT: p − Σβ_i t_i; EE: (1−s)a₀ + s a₁ − (1−t)b₀ − t b₁), λⁿ = κ A_k m_k |b′(d_k)| and the slots'
// relative positions yⁿ_j = x_j − x_0; every narrow phase of the step appends them after the barrier
// pairs (kind + 2) so the pair kernels, condensation and SpMV carry them like contact pairs
// ------------------------------------------------------------------------------------------
__device__ void closest_weights(int kind, int type, const v3* X, double* g) {
  g[0] = 1.0; g[1] = 0.0; g[2] = 0.0; g[3] = 0.0;
  if (kind == 0) {
    if (type == PT_T) {
      const v3 e1 = X[2] - X[1], e2 = X[3] - X[1], w = X[0] - X[1];
      const double a11 = dot(e1, e1), a12 = dot(e1, e2), a22 = dot(e2, e2), b1 = dot(e1, w), b2 = dot(e2, w);
      const double det = a11 * a22 - a12 * a12;
      const double be1 = (a22 * b1 - a12 * b2) / det, be2 = (a11 * b2 - a12 * b1) / det;
      g[1] = -(1.0 - be1 - be2); g[2] = -be1; g[3] = -be2;
    } else if (type < PT_V0) {
      const int i = type - PT_E0, j = (i + 1) % 3;
      const v3 a = X[1 + i], e = X[1 + j] - a;
      const double t = dot(X[0] - a, e) / dot(e, e);
      g[1 + i] -= 1.0 - t;
      g[1 + j] -= t;
    } else {
      g[1 + type - PT_V0] = -1.0;
    }
    return;
  }
  const int ss = type / 3, ts = type % 3;
  const v3 d1 = X[1] - X[0], d2 = X[3] - X[2], r = X[0] - X[2];
  double sp, tp;
  if (ss == 1 && ts == 1) {
    const double A = dot(d1, d1), B = dot(d1, d2), E = dot(d2, d2), Cc = dot(d1, r), F = dot(d2, r);
    const double den = A * E - B * B;
    sp = (B * F - Cc * E) / den;
    tp = (A * F - B * Cc) / den;
  } else if (ss == 1) {
    tp = ts == 0 ? 0.0 : 1.0;
    sp = dot((ts == 0 ? X[2] : X[3]) - X[0], d1) / dot(d1, d1);
  } else if (ts == 1) {
    sp = ss == 0 ? 0.0 : 1.0;
    tp = dot((ss == 0 ? X[0] : X[1]) - X[2], d2) / dot(d2, d2);
  } else {
    sp = ss == 0 ? 0.0 : 1.0;
    tp = ts == 0 ? 0.0 : 1.0;
  }
  g[0] = 1.0 - sp; g[1] = sp; g[2] = -(1.0 - tp); g[3] = -tp;
}

// block-level (k_narrow): freeze the friction pairs once per step, append them after the nbar barrier
// pairs; returns the total number of active-list entries
__device__ int friction_pairs(const Dev& D, int e, int nbar) {
  EnvCtl& C = D.ctl[e];
  const size_t ea = (size_t)e * D.act_cap;
  int* info = D.act_info + ea * 4;
  int* avid = D.act_vid + ea * 4;
  int* aslot = D.act_slot + ea * 4;
  int* ares = D.act_res + ea;
  double* axb = D.act_xb + ea * 12;
  if (!C.fr_frozen) {
    const double* P = D.P + (size_t)e * D.NVall * 3;
    for (int k = threadIdx.x; k < nbar; k += blockDim.x) {
      const int4 inf = reinterpret_cast<const int4*>(info)[k];
      const int4 vv = reinterpret_cast<const int4*>(avid)[k];
      const v3 X[4] = {ld3(P + 3 * vv.x), ld3(P + 3 * vv.y), ld3(P + 3 * vv.z), ld3(P + 3 * vv.w)};
      double gw[4];
      closest_weights(inf.x, inf.y, X, gw);
      const v3 sep = gw[0] * X[0] + gw[1] * X[1] + gw[2] * X[2] + gw[3] * X[3];
      const double d = sqrt(dot(sep, sep));
      const v3 nh = (1.0 / d) * sep;
      const double dm = d - D.dhat, lg = log(d / D.dhat);
      const double b1 = -2.0 * dm * lg - dm * dm / d;                 // b′(d)
      double m = 1.0;
      if (inf.x == 1 && D.mollify) {
        const v3 cn = cross(X[1] - X[0], X[3] - X[2]);
        double m1, m2;
        mollifier(dot(cn, cn), pair_eps(D, inf.x, inf.z, inf.w), &m, &m1, &m2);
      }
      const double lam = D.kappa * pair_area(D, inf.x, inf.z, inf.w) * m * fabs(b1);
      double* fd = D.fr_dat + (ea + k) * 16;
      fd[0] = D.dt * D.dt * D.mu_f * lam;
      fd[1] = nh.x; fd[2] = nh.y; fd[3] = nh.z;
      fd[4] = gw[1]; fd[5] = gw[2]; fd[6] = gw[3];
      for (int j = 0; j < 3; ++j) { const v3 y = X[j + 1] - X[0]; fd[7 + 3 * j] = y.x; fd[8 + 3 * j] = y.y; fd[9 + 3 * j] = y.z; }
      reinterpret_cast<int4*>(D.fr_info + ea * 4)[k] = inf;
      reinterpret_cast<int4*>(D.fr_vid + ea * 4)[k] = vv;
      reinterpret_cast<int4*>(D.fr_slot + ea * 4)[k] = reinterpret_cast<const int4*>(aslot)[k];
      D.fr_res[ea + k] = ares[k];
      for (int i = 0; i < 12; ++i) D.fr_xb[(ea + k) * 12 + i] = axb[12 * k + i];
    }
    __syncthreads();
    if (threadIdx.x == 0) { C.n_fr = nbar; C.fr_frozen = 1; }
    __syncthreads();
  }
  const int nfr = C.n_fr;
  const int n = min(nbar + nfr, D.act_cap);
  for (int k = threadIdx.x; k < n - nbar; k += blockDim.x) {
    const int pos = nbar + k;
    int4 inf = reinterpret_cast<const int4*>(D.fr_info + ea * 4)[k];
    inf.x += 2;
    reinterpret_cast<int4*>(info)[pos] = inf;
    reinterpret_cast<int4*>(avid)[pos] = reinterpret_cast<const int4*>(D.fr_vid + ea * 4)[k];
    reinterpret_cast<int4*>(aslot)[pos] = reinterpret_cast<const int4*>(D.fr_slot + ea * 4)[k];
    ares[pos] = D.fr_res[ea + k];
    for (int i = 0; i < 12; ++i) axb[12 * pos + i] = D.fr_xb[(ea + k) * 12 + i];
  }
  __syncthreads();
  if (threadIdx.x == 0) { C.n_act = n; if (nbar + nfr > D.act_cap) { C.overflow |= 8; C.cap_seen |= 8; } }
  __syncthreads();
  return n;
}

// friction energy of one frozen pair at slot positions X: Δt²μλ f0(‖(I − n̂n̂ᵀ) Σ_j Γ_j (y_j − yⁿ_j)‖)
__device__ __forceinline__ double friction_energy(const double* fd, const v3* X, double eps) {
  v3 w = mk(0, 0, 0);
#pragma unroll
  for (int j = 0; j < 3; ++j) w += fd[4 + j] * ((X[j + 1] - X[0]) - ld3(fd + 7 + 3 * j));
  const v3 nh = ld3(fd + 1);
  const v3 v = w - dot(nh, w) * nh;
  const double z = sqrt(dot(v, v));
  const double f0 = z < eps ? -z * z * z / (3.0 * eps * eps) + z * z / eps + eps / 3.0 : z;
  return fd[0] * f0;
}

// ------------------------------------------------------------------------------------------
// narrow phase: active set 𝒜 = {k ∈ C : s_k < d̂²} (strict) in canonical order, plus
// deterministic soft-vertex and body contribution lists
// ------------------------------------------------------------------------------------------
// contact condensation test (impl.cuh): a pair stays matrix-free ("residual") if two of its soft
// slots are not adjacent in the soft BSR pattern or its slots span two different DoF bodies
__device__ bool pair_is_residual(const Dev& D, const int* vid) {
  // soft slots of one primitive are BSR-adjacent (triangle and edge edges are tet edges), and the two
  // primitives of a pair lie on different bodies (no self contact, reading R8), so two soft slots are
  // non-adjacent exactly when they lie on different soft bodies — no search of the BSR rows is needed
  int sbody = -1, body = -1;
  for (int s = 0; s < 4; ++s) {
    const int v = vid[s];
    if (v < D.V) {
      const int b = D.vert_body[v];
      if (sbody >= 0 && b != sbody) return true;
      sbody = b;
    } else {
      const int d = D.dof_slot[D.vert_aff[v]];
      if (d >= 0) {
        if (body >= 0 && body != d) return true;
        body = d;
      }
    }
  }
  return false;
}

template <int MINB>
__global__ void __launch_bounds__(NTHREADS, MINB) k_narrow(Dev D, int env0, int force) {
  const int e = env_at(D, env0, blockIdx.x);
  EnvCtl& C = D.ctl[e];
  if (env_skip(D, e, force)) return;
  extern __shared__ int dsm[];
  int* vcnt = dsm;                 // [V+1]
  int* vcur = dsm + D.V + 1;       // [V]
  __shared__ int sh[33];
  const double* P = D.P + (size_t)e * D.NVall * 3;
  const int* ca = D.cand_a + (size_t)e * D.cand_cap;
  const int* cb = D.cand_b + (size_t)e * D.cand_cap;
  int* info = D.act_info + (size_t)e * D.act_cap * 4;
  int* avid = D.act_vid + (size_t)e * D.act_cap * 4;
  const double dh2 = D.dhat * D.dhat;
  const int nc = C.ncand;
  int total = 0;
  double mind2 = 1.0 / 0.0;
  for (int t0 = 0; t0 < nc; t0 += blockDim.x) {
    int k = t0 + threadIdx.x;
    int flag = 0, kind = 0, type = 0, a = 0, b = 0, vid[4];
    if (k < nc) {
      kind = (ca[k] >> 30) & 1; a = ca[k] & ((1 << 30) - 1); b = cb[k];
      pair_vids(D, kind, a, b, vid);
      v3 X[4];
      for (int s = 0; s < 4; ++s) X[s] = ld3(P + 3 * vid[s]);
      if (prim_box_dist(kind, X) < D.dhat * (1.0 + 1e-9)) {   // else d ≥ box distance > d̂: inactive
        double d2;
        type = classify(kind, X, &d2);
        flag = d2 < dh2;
        mind2 = fmin(mind2, d2);
      }
    }
    int tot;
    int ex = block_excl_scan(flag, sh, &tot);
    int pos = total + ex;
    if (flag && pos < D.act_cap) {
      info[4 * pos] = kind; info[4 * pos + 1] = type; info[4 * pos + 2] = a; info[4 * pos + 3] = b;
      int* aslot = D.act_slot + (size_t)e * 4 * D.act_cap + 4 * pos;
      double* axb = D.act_xb + (size_t)e * 12 * D.act_cap + 12 * pos;
      for (int s = 0; s < 4; ++s) {
        avid[4 * pos + s] = vid[s];
        int code;
        if (vid[s] < D.V) code = vid[s];
        else {
          const int d = D.dof_slot[D.vert_aff[vid[s]]];
          code = d >= 0 ? -1 - d : INT_MIN;
          axb[3 * s] = D.vert_xbar[3 * vid[s]]; axb[3 * s + 1] = D.vert_xbar[3 * vid[s] + 1];
          axb[3 * s + 2] = D.vert_xbar[3 * vid[s] + 2];
        }
        aslot[s] = code;
      }
      D.act_res[(size_t)e * D.act_cap + pos] = pair_is_residual(D, vid) ? 1 : 0;
    }
    total += tot;
  }
  int nact = min(total, D.act_cap);
  {
    __shared__ double redm[32];
    mind2 = block_min(mind2, redm);
  }
  if (threadIdx.x == 0) { C.n_act = nact; C.min_d2 = mind2; if (total > D.act_cap) { C.overflow |= 8; C.cap_seen |= 8; } }
  __syncthreads();
  if (D.mu_f > 0.0) nact = friction_pairs(D, e, nact);
  // residual pairs (kept matrix-free in the SpMV), ascending
  {
    const int* ares = D.act_res + (size_t)e * D.act_cap;
    int* rl = D.res_list + (size_t)e * D.act_cap;
    int* aresw = D.act_res + (size_t)e * D.act_cap;
    int run = 0;
    for (int t0 = 0; t0 < nact; t0 += blockDim.x) {
      const int k = t0 + threadIdx.x;
      const int f = k < nact ? (ares[k] != 0) : 0;
      int tot;
      const int ex = block_excl_scan(f, sh, &tot);
      __syncthreads();
      if (f) {
        rl[run + ex] = k;
        aresw[k] = run + ex + 1;                  // residual index + 1: the slot of its 12×12 in act_H
      }
      run += tot;
    }
    if (threadIdx.x == 0) {
      C.n_res = run;
      if (run > D.res_cap) { C.overflow |= 16; C.cap_seen |= 16; }   // residual Hessians (act_H) capacity
    }
  }
  // soft-vertex contribution lists: count, scan, fill, per-vertex sort (deterministic)
  for (int v = threadIdx.x; v <= D.V; v += blockDim.x) vcnt[v] = 0;
  __syncthreads();
  for (int k = threadIdx.x; k < nact; k += blockDim.x)
    for (int s = 0; s < 4; ++s) { int gv = avid[4 * k + s]; if (gv < D.V) atomicAdd(&vcnt[gv], 1); }
  __syncthreads();
  int* cptr = D.cptr + (size_t)e * (D.V + 1);
  int* clist = D.clist + (size_t)e * 4 * D.act_cap;
  {
    int run_total = 0;
    for (int t0 = 0; t0 < D.V; t0 += blockDim.x) {
      int v = t0 + threadIdx.x;
      int c = v < D.V ? vcnt[v] : 0;
      int tot;
      int ex = block_excl_scan(c, sh, &tot);
      if (v < D.V) { cptr[v] = run_total + ex; vcur[v] = run_total + ex; }
      run_total += tot;
    }
    if (threadIdx.x == 0) cptr[D.V] = run_total;
  }
  __syncthreads();
  for (int k = threadIdx.x; k < nact; k += blockDim.x)
    for (int s = 0; s < 4; ++s) {
      int gv = avid[4 * k + s];
      if (gv < D.V) { int pos = atomicAdd(&vcur[gv], 1); clist[pos] = 4 * k + s; }
    }
  __syncthreads();
  int* spos = D.spos + (size_t)e * 4 * D.act_cap;
  for (int i = threadIdx.x; i < 4 * nact; i += blockDim.x) spos[i] = -1;
  __syncthreads();
  // per-vertex sort: residual-pair slots first, then by (pair, slot); only residual slots get an
  // output position (the SpMV's matrix-free pass writes them, the soft row sums the first rcnt[v])
  {
    const int* ares = D.act_res + (size_t)e * D.act_cap;
    int* rc = D.rcnt + (size_t)e * D.V;
    for (int v = threadIdx.x; v < D.V; v += blockDim.x) {
      int b0 = cptr[v], b1 = cptr[v + 1], nr = 0;
      if (b1 - b0 <= 32) {                                // sort a private copy (L1), not global memory
        int kk[32];
        const int c = b1 - b0;
        for (int i = 0; i < c; ++i) {
          const int key = clist[b0 + i];
          const int res = ares[key >> 2] != 0;         // ares holds the residual index + 1 (0: condensed)
          nr += res;
          kk[i] = key | ((res ? 0 : 1) << 30);
        }
        for (int i = 1; i < c; ++i) {
          int key = kk[i], j = i - 1;
          while (j >= 0 && kk[j] > key) { kk[j + 1] = kk[j]; --j; }
          kk[j + 1] = key;
        }
        for (int i = 0; i < c; ++i) {
          const int key = kk[i] & ((1 << 30) - 1);
          clist[b0 + i] = key;
          spos[key] = b0 + i;                             // soft slot → its vertex-sorted position
        }
      } else {
        for (int i = b0; i < b1; ++i) {
          const int res = ares[clist[i] >> 2] != 0;
          nr += res;
          clist[i] |= (res ? 0 : 1) << 30;
        }
        for (int i = b0 + 1; i < b1; ++i) {
          int key = clist[i], j = i - 1;
          while (j >= b0 && clist[j] > key) { clist[j + 1] = clist[j]; --j; }
          clist[j + 1] = key;
        }
        for (int i = b0; i < b1; ++i) clist[i] &= (1 << 30) - 1;
        for (int i = b0; i < b1; ++i) spos[clist[i]] = i;
      }
      rc[v] = nr;
    }
  }
}

// ------------------------------------------------------------------------------------------
// Neo-Hookean tets: gradient + F-space-projected 12×12 (SoA [90][T] per env)
// ------------------------------------------------------------------------------------------
__global__ void __launch_bounds__(NTHREADS) k_tets(Dev D, int env0, int force) {
  const int e = env_at(D, env0, blockIdx.y);
  const int sl = blockIdx.y;                   // slot in the assembly scratch (launch-local, < asm_envs)
  if (env_skip(D, e, force)) return;
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= D.T) return;
  const double* q = D.q + (size_t)e * D.n;
  int4 tv = reinterpret_cast<const int4*>(D.tets)[t];
  v3 x[4] = {ld3(q + 3 * tv.x), ld3(q + 3 * tv.y), ld3(q + 3 * tv.z), ld3(q + 3 * tv.w)};
  double Dmi[9];
#pragma unroll
  for (int i = 0; i < 9; ++i) Dmi[i] = D.Dmi[9 * t + i];
  const double scale = D.dt * D.dt * D.vol[t];
  // per-tet gradient and packed upper Hessian, SoA [90][T] (coalesced stores; an element-record layout in
  // assembly order was measured slower: its scattered 8-byte stores cost k_tets 3.5x, the gathers it saved
  // were latency-, not sector-bound)
  double* out = D.tetbuf + (size_t)sl * TETBUF * D.T + t;
  const size_t T = D.T;
  auto gst = [&](int i, double v) { out[(size_t)i * T] = v; };
  auto hst = [&](int r, int s, double v) { out[(size_t)(12 + sym_idx(r, s, 12)) * T] = v; };
  if (D.ctl[e].exact) nh_grad_hess_t(x, Dmi, D.mu[t], D.lam[t], scale, nullptr, gst, hst, false);
  else nh_grad_hess_t(x, Dmi, D.mu[t], D.lam[t], scale, nullptr, gst, hst, true);
}
// exact Hessians only (hessian_mode 2, every env): the projected branch (SVD, negative-mode subtraction)
// is not compiled in, so the kernel keeps a small register/stack footprint
__global__ void __launch_bounds__(NTHREADS) k_tets_x(Dev D, int env0, int force) {
  const int e = env_at(D, env0, blockIdx.y);
  const int sl = blockIdx.y;                   // slot in the assembly scratch (launch-local, < asm_envs)
  if (env_skip(D, e, force)) return;
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= D.T) return;
  const double* q = D.q + (size_t)e * D.n;
  int4 tv = reinterpret_cast<const int4*>(D.tets)[t];
  v3 x[4] = {ld3(q + 3 * tv.x), ld3(q + 3 * tv.y), ld3(q + 3 * tv.z), ld3(q + 3 * tv.w)};
  double Dmi[9];
#pragma unroll
  for (int i = 0; i < 9; ++i) Dmi[i] = D.Dmi[9 * t + i];
  const double scale = D.dt * D.dt * D.vol[t];
  // per-tet gradient and packed upper Hessian, SoA [90][T] (coalesced stores; an element-record layout in
  // assembly order was measured slower: its scattered 8-byte stores cost k_tets 3.5x, the gathers it saved
  // were latency-, not sector-bound)
  double* out = D.tetbuf + (size_t)sl * TETBUF * D.T + t;
  const size_t T = D.T;
  auto gst = [&](int i, double v) { out[(size_t)i * T] = v; };
  auto hst = [&](int r, int s, double v) { out[(size_t)(12 + sym_idx(r, s, 12)) * T] = v; };
  nh_grad_hess_t(x, Dmi, D.mu[t], D.lam[t], scale, nullptr, gst, hst, false);
}

// ------------------------------------------------------------------------------------------
// barrier pairs: warp per pair; closed-form ∇s/∇²s, barrier + mollifier composition, full 12×12
// PSD projection by warp Jacobi (readings R10-R12)
// ------------------------------------------------------------------------------------------
constexpr int PAIR_WARPS = 4;          // warps per CTA in k_pairs
constexpr int PAIRS_PER_WARP = 4;      // pairs handled sequentially by one warp
constexpr int PAIRS_PER_CTA = PAIR_WARPS * PAIRS_PER_WARP;
constexpr int PAIR_GRID_X = 12;       // CTAs per env (each loops over pair chunks)

struct PairScratch {
  JacobiScratch J;
  double gv[9], gcv[9];       // variable-space ∇s and ∇c
  double hv[81], hcv[81];     // variable-space ∇²s and ∇²c, index (3v+a)*9 + 3u+b
  double gs[12], gc[12];      // slot-space ∇s and ∇c
  // table-driven variable-space derivatives (array-indexed, no select chains)
  double W[3], E1[3], E2[3], Nn[3];   // sub-distance variables (PL: E1 = e)
  double U1[9], D1[9];                // TRI: ∂u/∂var, ∂D/∂var;  PL: ∂N/∂var, ∂D/∂var;  PP: ∂s/∂w
  double CE1[3], CE2[3], CN[3], CD1[9];  // mollifier c = ‖e1×e2‖²
  double gf[12], xb[12];              // final scaled gradient; rest positions x̄ of affine slots
};

__device__ __forceinline__ double skewv(const double* x, int a, int b) {   // ([x]×)_{ab}
  if (a == b) return 0.0;
  const double v = x[3 - a - b];
  return ((b - a + 3) % 3 == 2) ? v : -v;
}
__device__ __forceinline__ double dot3a(const double* x, const double* y) { return x[0] * y[0] + x[1] * y[1] + x[2] * y[2]; }
// ∂²D/∂var_v[a]∂var_u[b] for D = ‖e1×e2‖² (v, u ∈ {1, 2}; [x]×ᵀ[y]× = (x·y)I − y xᵀ)
__device__ __forceinline__ double tri_D2_fast(const double* e1, const double* e2, const double* n, int v, int a, int u, int b) {
  if (v == 0 || u == 0) return 0.0;
  const double dab = a == b ? 1.0 : 0.0;
  double r;
  if (v == 1 && u == 1) r = dot3a(e2, e2) * dab - e2[a] * e2[b];
  else if (v == 2 && u == 2) r = dot3a(e1, e1) * dab - e1[a] * e1[b];
  else if (v == 1) r = -(dot3a(e2, e1) * dab - e1[a] * e2[b]) - skewv(n, a, b);
  else r = -(dot3a(e1, e2) * dab - e2[a] * e1[b]) - skewv(n, b, a);
  return 2.0 * r;
}
// ∂²u/∂var_v[a]∂var_u[b] for u = w·(e1×e2)
__device__ __forceinline__ double tri_u2_fast(const double* w, const double* e1, const double* e2, int v, int a, int u, int b) {
  if (v == u) return 0.0;
  if (v > u) { int t = v; v = u; u = t; t = a; a = b; b = t; }
  if (v == 0 && u == 1) return -skewv(e2, a, b);
  if (v == 0 && u == 2) return skewv(e1, a, b);
  return -skewv(w, a, b);
}

// grid (ceil(act_cap / PAIRS_PER_CTA), envs): many CTAs per env so a single contact-heavy env is
// spread over the whole GPU; CTAs past the env's active count exit at once.
__global__ void __launch_bounds__(PAIR_WARPS * 32, 3) k_pairs(Dev D, int env0, int force) {
  const int e = env_at(D, env0, blockIdx.y);
  const int sl = blockIdx.y;                   // slot in the assembly scratch (launch-local, < asm_envs)
  if (env_skip(D, e, force)) return;
  const EnvCtl& C = D.ctl[e];
  if (C.exact) return;                                    // exact Hessians: k_pairs_x (thread per pair)
  const int nact = C.n_act;
  if ((int)blockIdx.x * PAIRS_PER_CTA >= nact) return;
  __shared__ PairScratch PS[PAIR_WARPS];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const double* P = D.P + (size_t)e * D.NVall * 3;
  const int* info = D.act_info + (size_t)e * D.act_cap * 4;
  const int* avid = D.act_vid + (size_t)e * D.act_cap * 4;
  double* aH = D.act_H + (size_t)e * D.res_cap * PH;
  PairScratch& S = PS[w];
  const bool project = !C.exact;
  // CTA b takes the pair chunks b, b + gridDim.x, ... (a fixed small grid: empty CTAs cost launch time)
  for (int base = blockIdx.x * PAIRS_PER_CTA; base < nact; base += gridDim.x * PAIRS_PER_CTA)
  for (int j = 0; j < PAIRS_PER_WARP; ++j) {
    const int k = base + w + PAIR_WARPS * j;
    if (k >= nact) break;
    const int kind = info[4 * k], type = info[4 * k + 1], a = info[4 * k + 2], b = info[4 * k + 3];
    v3 X[4];
    for (int s = 0; s < 4; ++s) X[s] = ld3(P + 3 * avid[4 * k + s]);
    SubDist SD;
    sd_make(SD, kind, type, X);
    const int nvar = SD.sub == SUB_PP ? 1 : (SD.sub == SUB_PL ? 2 : 3);
    double B, B1, B2;
    barrier_s(SD.s, D.dhat, &B, &B1, &B2);
    const bool useM = (kind == 1) && D.mollify;
    SubDist CC;
    sd_zero(CC);
    double m = 1.0, m1 = 0.0, m2 = 0.0;
    if (useM) {
      sd_make_cross(CC, X);
      mollifier(CC.D, pair_eps(D, kind, a, b), &m, &m1, &m2);
    }
    const bool molterm = useM && m1 != 0.0;
    const double scale = D.dt * D.dt * D.kappa * pair_area(D, kind, a, b);
    // 1) variable-space derivatives (table-driven): vectors to shared memory, then first-derivative
    //    tables (9 lanes), then the 81 second-derivative entries (all lanes)
    if (lane == 0) {
      S.W[0] = SD.w.x; S.W[1] = SD.w.y; S.W[2] = SD.w.z;
      S.E1[0] = SD.e1.x; S.E1[1] = SD.e1.y; S.E1[2] = SD.e1.z;
      S.E2[0] = SD.e2.x; S.E2[1] = SD.e2.y; S.E2[2] = SD.e2.z;
      S.Nn[0] = SD.n.x; S.Nn[1] = SD.n.y; S.Nn[2] = SD.n.z;
      S.CE1[0] = CC.e1.x; S.CE1[1] = CC.e1.y; S.CE1[2] = CC.e1.z;
      S.CE2[0] = CC.e2.x; S.CE2[1] = CC.e2.y; S.CE2[2] = CC.e2.z;
      S.CN[0] = CC.n.x; S.CN[1] = CC.n.y; S.CN[2] = CC.n.z;
    }
    __syncwarp();
    if (lane < 9) {
      const int v = lane / 3, a = lane % 3, a1 = (a + 1) % 3, a2 = (a + 2) % 3;
      double u1 = 0.0, d1 = 0.0, cd1 = 0.0;
      if (SD.sub == SUB_TRI) {
        if (v == 0) u1 = S.Nn[a];
        else if (v == 1) u1 = S.E2[a1] * S.W[a2] - S.E2[a2] * S.W[a1];                 // (e2×w)_a
        else u1 = S.W[a1] * S.E1[a2] - S.W[a2] * S.E1[a1];                             // (w×e1)_a
        if (v == 1) d1 = 2.0 * (S.E2[a1] * S.Nn[a2] - S.E2[a2] * S.Nn[a1]);            // 2(e2×n)_a
        else if (v == 2) d1 = 2.0 * (S.Nn[a1] * S.E1[a2] - S.Nn[a2] * S.E1[a1]);       // 2(n×e1)_a
      } else if (SD.sub == SUB_PL) {
        if (v == 0) u1 = 2.0 * (SD.D * S.W[a] - SD.we * S.E1[a]);
        else if (v == 1) u1 = 2.0 * (SD.ww * S.E1[a] - SD.we * S.W[a]);
        if (v == 1) d1 = 2.0 * S.E1[a];
      } else if (v == 0) {
        u1 = 2.0 * S.W[a];
      }
      if (useM) {
        if (v == 1) cd1 = 2.0 * (S.CE2[a1] * S.CN[a2] - S.CE2[a2] * S.CN[a1]);
        else if (v == 2) cd1 = 2.0 * (S.CN[a1] * S.CE1[a2] - S.CN[a2] * S.CE1[a1]);
      }
      S.U1[lane] = u1; S.D1[lane] = d1; S.CD1[lane] = cd1;
      double g1;
      if (SD.sub == SUB_TRI) g1 = 2.0 * SD.u * u1 * SD.iD - SD.u * SD.u * d1 * SD.iD2;
      else if (SD.sub == SUB_PL) g1 = u1 * SD.iD - SD.N * d1 * SD.iD2;
      else g1 = u1;
      S.gv[lane] = g1;
      S.gcv[lane] = cd1;
    }
    __syncwarp();
    for (int i = lane; i < 81; i += 32) {
      const int va = i / 9, ub = i % 9, v = va / 3, u = ub / 3, a_ = va % 3, b_ = ub % 3;
      double h = 0.0;
      if (v < nvar && u < nvar) {
        const double ua = S.U1[va], ubb = S.U1[ub], Da = S.D1[va], Db = S.D1[ub];
        const double dab = a_ == b_ ? 1.0 : 0.0;
        if (SD.sub == SUB_TRI) {
          const double U = SD.u;
          h = 2.0 * (ua * ubb + U * tri_u2_fast(S.W, S.E1, S.E2, v, a_, u, b_)) * SD.iD -
              2.0 * U * (ua * Db + Da * ubb) * SD.iD2 - U * U * tri_D2_fast(S.E1, S.E2, S.Nn, v, a_, u, b_) * SD.iD2 +
              2.0 * U * U * Da * Db * SD.iD3;
        } else if (SD.sub == SUB_PL) {
          double N2;
          if (v == 0 && u == 0) N2 = 2.0 * (SD.D * dab - S.E1[a_] * S.E1[b_]);
          else if (v == 1 && u == 1) N2 = 2.0 * (SD.ww * dab - S.W[a_] * S.W[b_]);
          else if (v == 0) N2 = 2.0 * (2.0 * S.W[a_] * S.E1[b_] - S.E1[a_] * S.W[b_] - SD.we * dab);
          else N2 = 2.0 * (2.0 * S.W[b_] * S.E1[a_] - S.E1[b_] * S.W[a_] - SD.we * dab);
          const double D2 = (v == 1 && u == 1) ? 2.0 * dab : 0.0;
          h = N2 * SD.iD - (ua * Db + Da * ubb) * SD.iD2 - SD.N * D2 * SD.iD2 + 2.0 * SD.N * Da * Db * SD.iD3;
        } else {
          h = (v == 0 && u == 0) ? 2.0 * dab : 0.0;
        }
      }
      S.hv[i] = h;
      S.hcv[i] = (molterm && v > 0 && u > 0) ? tri_D2_fast(S.CE1, S.CE2, S.CN, v, a_, u, b_) : 0.0;
    }
    __syncwarp();
    // 2) slot-space gradients (coefficients are ±1/0 combinations of the variables)
    if (lane < 12) {
      const int sl = lane / 3, ax = lane % 3;
      double g1 = 0.0, g2 = 0.0;
      for (int v = 0; v < 3; ++v) {
        g1 += SD.coef[v][sl] * S.gv[3 * v + ax];
        g2 += CC.coef[v][sl] * S.gcv[3 * v + ax];
      }
      S.gs[lane] = g1;
      S.gc[lane] = useM ? g2 : 0.0;
    }
    __syncwarp();
    if (lane < 12) {
      const double gfin = scale * (m * B1 * S.gs[lane] + B * m1 * S.gc[lane]);
      S.gf[lane] = gfin;
    }
    // 3) 12×12 (upper) from the variable blocks
    for (int i = lane; i < 144; i += 32) {
      const int r = i / 12, c = i % 12;
      double h = 0.0;
      if (r <= c) {
        const int k1 = r / 3, a1 = r % 3, k2 = c / 3, a2 = c % 3;
        double hs = 0.0, hc = 0.0;
        for (int v = 0; v < 3; ++v) {
          const int cv = SD.coef[v][k1], cw = CC.coef[v][k1];
          for (int u = 0; u < 3; ++u) {
            const int idx = (3 * v + a1) * 9 + 3 * u + a2;
            hs += (double)(cv * SD.coef[u][k2]) * S.hv[idx];
            if (molterm) hc += (double)(cw * CC.coef[u][k2]) * S.hcv[idx];
          }
        }
        h = m * (B2 * S.gs[r] * S.gs[c] + B1 * hs);
        if (molterm) h += B * (m2 * S.gc[r] * S.gc[c] + m1 * hc) + m1 * B1 * (S.gs[r] * S.gc[c] + S.gc[r] * S.gs[c]);
        h *= scale;
      }
      S.J.A[i] = h;
    }
    __syncwarp();
    if (project) {
      for (int i = lane; i < 144; i += 32) {
        int r = i / 12, c = i % 12;
        if (r > c) S.J.A[i] = S.J.A[12 * c + r];
      }
      __syncwarp();
      jacobi12_psd(S.J, lane, 32);
    }
    const int ridx = D.act_res[(size_t)e * D.act_cap + k];
    const bool res = ridx != 0;
    if (res && ridx <= D.res_cap)   // residual pairs stay matrix-free in the SpMV: packed upper 12×12, AoS
      for (int i = lane; i < PH; i += 32) aH[(size_t)(ridx - 1) * PH + i] = S.J.A[12 * c_unpack_r[i] + c_unpack_c[i]];
    // 4) condensed records (contact condensation, impl.cuh), read by k_assemble without touching H
    for (int i = lane; i < 144; i += 32) {
      const int r = i / 12, c = i % 12;
      if (r > c) S.J.A[i] = S.J.A[12 * c + r];
    }
    if (lane < 12) S.xb[lane] = D.act_xb[((size_t)e * D.act_cap + k) * 12 + lane];
    __syncwarp();
    const int4 c4 = reinterpret_cast<const int4*>(D.act_slot + (size_t)e * 4 * D.act_cap)[k];
    const int codes[4] = {c4.x, c4.y, c4.z, c4.w};
    int bd0 = -1, bd1 = -1;              // DoF bodies of the pair (≤2: one per primitive), ascending
    for (int t = 0; t < 4; ++t) {
      const int cd = codes[t];
      if (cd < 0 && cd != INT_MIN) {
        const int d = -1 - cd;
        if (bd0 < 0) bd0 = d;
        else if (d != bd0) bd1 = d;
      }
    }
    if (bd1 >= 0 && bd1 < bd0) { const int tmp = bd0; bd0 = bd1; bd1 = tmp; }
    const double* A = S.J.A;
    // per soft slot s, at its vertex-sorted position j: [g_s 3 | H_ss 9 | C_s = Σ_{t on body} H_st J_t 36 |
    // H_st for the (≤2) other soft slots t 18]; couplings and neighbour blocks are zero for residual pairs
    for (int s = 0; s < 4; ++s) {
      if (codes[s] < 0) continue;
      const int j = D.spos[(size_t)e * 4 * D.act_cap + 4 * k + s];
      int nbt[2] = {-1, -1}, nn = 0;
      for (int t = 0; t < 4; ++t)
        if (t != s && codes[t] >= 0 && nn < 2) nbt[nn++] = t;
      double* rec = D.srec + ((size_t)sl * 4 * D.act_cap + j) * SREC;
      for (int i = lane; i < SREC; i += 32) {
        double v = 0.0;
        if (i < 3) v = S.gf[3 * s + i];
        else if (i < 12) v = A[12 * (3 * s + (i - 3) / 3) + 3 * s + (i - 3) % 3];
        else if (i < 48) {
          if (!res && bd0 >= 0) {
            const int r = (i - 12) / 12, be = (i - 12) % 12, jr = jrow(be);
            for (int t = 0; t < 4; ++t)
              if (codes[t] == -1 - bd0) v += A[12 * (3 * s + r) + 3 * t + jr] * (be < 3 ? 1.0 : S.xb[3 * t + (be - 3) % 3]);
          }
        } else {
          const int nb = (i - 48) / 9, rc = (i - 48) % 9, t = nbt[nb];
          if (!res && t >= 0) v = A[12 * (3 * s + rc / 3) + 3 * t + rc % 3];
        }
        rec[i] = v;
      }
      if (lane < 2) {
        int jb = -1;
        const int t = nbt[lane];
        if (!res && t >= 0) {
          const int v = codes[s], wv = codes[t];
          for (int q = D.rptr[v]; q < D.rptr[v + 1]; ++q)
            if (D.rcol[q] == wv) { jb = q; break; }
        }
        D.snb[((size_t)sl * 4 * D.act_cap + j) * 2 + lane] = jb;
      }
      if (lane == 0) D.sbody[(size_t)sl * 4 * D.act_cap + j] = res ? -1 : bd0;
    }
    // per DoF body of the pair (ascending, ≤2): packed Σ_{s,t on body} J_sᵀ H_st J_t (78) and Σ_s J_sᵀ g_s (12)
    for (int rb = 0; rb < 2; ++rb) {
      const int bd = rb == 0 ? bd0 : bd1;
      if (bd < 0) break;
      double* out = D.brec + (((size_t)(sl % D.brec_envs) * D.act_cap + k) * 2 + rb) * BREC;
      for (int i = lane; i < BREC; i += 32) {
        double v = 0.0;
        if (i < PH) {
          const int al = c_unpack_r[i], be = c_unpack_c[i], ra = jrow(al), rbw = jrow(be);
          for (int s = 0; s < 4; ++s) {
            if (codes[s] != -1 - bd) continue;
            const double fs = al < 3 ? 1.0 : S.xb[3 * s + (al - 3) % 3];
            double inner = 0.0;
            for (int t = 0; t < 4; ++t)
              if (codes[t] == -1 - bd) inner += (be < 3 ? 1.0 : S.xb[3 * t + (be - 3) % 3]) * A[12 * (3 * s + ra) + 3 * t + rbw];
            v += fs * inner;
          }
        } else {
          const int al = i - PH, ra = jrow(al);
          for (int s = 0; s < 4; ++s)
            if (codes[s] == -1 - bd) v += (al < 3 ? 1.0 : S.xb[3 * s + (al - 3) % 3]) * S.gf[3 * s + ra];
        }
        out[i] = v;
      }
    }
    __syncwarp();
  }
}

// chunk partials of the body records for projected envs (k_pairs writes per-pair records brec):
// partial[chunk][d] = Σ over the chunk's 32 pairs in pair order (same layout as k_pairs_x)
__global__ void k_bpart_proj(Dev D, int env0, int force) {
  const int e = env_at(D, env0, blockIdx.y);
  const int sl = blockIdx.y;                   // slot in the assembly scratch (launch-local, < asm_envs)
  if (env_skip(D, e, force)) return;
  const EnvCtl& C = D.ctl[e];
  if (C.exact) return;
  const int nact = C.n_act, k0 = 32 * blockIdx.x;
  if (k0 >= nact) return;
  const int k1 = min(k0 + 32, nact);
  const size_t nchunk = (size_t)(D.act_cap + 31) >> 5;
  const int* aslot = D.act_slot + (size_t)e * 4 * D.act_cap;
  const int* ares = D.act_res + (size_t)e * D.act_cap;
  for (int t = threadIdx.x; t < D.ND * BPART; t += blockDim.x) {
    const int d = t / BPART, i = t % BPART;
    double sum = 0.0;
    for (int k = k0; k < k1; ++k) {
      int bd0 = -1, bd1 = -1;
      for (int s = 0; s < 4; ++s) {
        const int cd = aslot[4 * k + s];
        if (cd < 0 && cd != INT_MIN) {
          const int dd = -1 - cd;
          if (bd0 < 0) bd0 = dd;
          else if (dd != bd0) bd1 = dd;
        }
      }
      if (bd1 >= 0 && bd1 < bd0) { const int tmp = bd0; bd0 = bd1; bd1 = tmp; }
      const int rb = bd0 == d ? 0 : (bd1 == d ? 1 : -1);
      if (rb < 0) continue;
      const double* rec = D.brec + (((size_t)(sl % D.brec_envs) * D.act_cap + k) * 2 + rb) * BREC;
      const bool res = ares[k] != 0;
      if (i < 12) sum += rec[PH + i];
      else if (i < 12 + PH) { if (!res) sum += rec[i - 12]; }
      else if (res) sum += rec[i - 12 - PH];
    }
    D.bpart[(((size_t)sl * nchunk + blockIdx.x) * D.ND + d) * BPART + i] = sum;
  }
}

// ------------------------------------------------------------------------------------------
// barrier pairs, exact Hessian (hessian_mode ≥ 1 with C.exact; the LM default R14c): ONE THREAD
// PER PAIR, everything in registers.  Every sub-distance variable (w, e1, e2; and the EE mollifier's
// a1−a0, b1−b0) is a ±1 combination of the slots with zero coefficient sum, so the pair energy is a
// function of the relative coordinates y_j = x_j − x_0 (j = 1..3).  The thread builds the scaled
// gradient G_y (9) and Hessian H_y (9×9, packed upper 45) of κA_k m b(d) in y-space, then expands
// exactly the slot-space blocks the condensed records need (same record layout as k_pairs):
//   slot s row-block of H:  Q_s[(l,b)][r] = Σ_j σ_j(s) H_y[(j,r),(l,b)],  σ_j(0) = −1, σ_j(s) = δ_js
//   H_st[r][b] = Σ_l σ_l(t) Q_s[(l,b)][r];  g_s = Σ_j σ_j(s) G_y[j]
//   body pull-back weights w_l(β) = on_l f(β,l) − on_0 f(β,0), f(β,t) = 1 (β<3) or x̄_t[(β−3)%3]:
//   C_s[r][β] = Σ_l w_l(β) Q_s[(l,ρβ)][r],  body block [α,β] = Σ_{j,l} w_j(α) w_l(β) H_y[(j,ρα),(l,ρβ)]
// (P:L393 barrier, P:L419 weights; readings R7, R10-R12.)
// ------------------------------------------------------------------------------------------
__device__ __forceinline__ constexpr int s9(int r, int c) {      // packed upper index of a 9×9, r ≤ c
  return r * 9 - (r * (r - 1)) / 2 + (c - r);
}
__device__ __forceinline__ double hy_at(const double* Hy, int r, int c) { return r <= c ? Hy[s9(r, c)] : Hy[s9(c, r)]; }

// H_y += Σ_{v,u} cy[v][j] cy[u][l] · wgt · h(v,a,u,b) for the sub-distance SUB (var-space second
// derivatives as in k_pairs, evaluated with compile-time indices)
template <int SUB>
__device__ __forceinline__ void scatter_sub(double* Hy, const double (*cy)[3], double wgt, const double* W,
                                            const double* E1, const double* E2, const double* Nn, const double* u1,
                                            const double* d1, const SubDist& SD) {
  constexpr int NV = SUB == SUB_TRI ? 3 : (SUB == SUB_PL ? 2 : 1);
#pragma unroll
  for (int v = 0; v < NV; ++v)
#pragma unroll
    for (int a = 0; a < 3; ++a)
#pragma unroll
      for (int u = 0; u < NV; ++u)
#pragma unroll
        for (int b = 0; b < 3; ++b) {
          double h;
          const double dab = a == b ? 1.0 : 0.0;
          if constexpr (SUB == SUB_TRI) {
            const double ua = u1[3 * v + a], ub = u1[3 * u + b], Da = d1[3 * v + a], Db = d1[3 * u + b], U = SD.u;
            h = 2.0 * (ua * ub + U * tri_u2_fast(W, E1, E2, v, a, u, b)) * SD.iD - 2.0 * U * (ua * Db + Da * ub) * SD.iD2 -
                U * U * tri_D2_fast(E1, E2, Nn, v, a, u, b) * SD.iD2 + 2.0 * U * U * Da * Db * SD.iD3;
          } else if constexpr (SUB == SUB_PL) {
            const double ua = u1[3 * v + a], ub = u1[3 * u + b], Da = d1[3 * v + a], Db = d1[3 * u + b];
            double N2;
            if (v == 0 && u == 0) N2 = 2.0 * (SD.D * dab - E1[a] * E1[b]);
            else if (v == 1 && u == 1) N2 = 2.0 * (SD.ww * dab - W[a] * W[b]);
            else if (v == 0) N2 = 2.0 * (2.0 * W[a] * E1[b] - E1[a] * W[b] - SD.we * dab);
            else N2 = 2.0 * (2.0 * W[b] * E1[a] - E1[b] * W[a] - SD.we * dab);
            const double D2 = (v == 1 && u == 1) ? 2.0 * dab : 0.0;
            h = N2 * SD.iD - (ua * Db + Da * ub) * SD.iD2 - SD.N * D2 * SD.iD2 + 2.0 * SD.N * Da * Db * SD.iD3;
          } else {
            h = 2.0 * dab;
          }
          const double t = wgt * h;
#pragma unroll
          for (int j = 0; j < 3; ++j) {
            const double tj = cy[v][j] * t;
#pragma unroll
            for (int l = 0; l < 3; ++l)
              if (3 * j + a <= 3 * l + b) Hy[s9(3 * j + a, 3 * l + b)] += cy[u][l] * tj;
          }
        }
}

// sub-distance of a classified pair in y-coordinates (y_j = x_j − x_0): the variables' slot
// coefficients cy[v][j] (v = w, e1, e2; j = slot j+1) by selects, no runtime-indexed arrays
// (same variables as sd_make, geometry.cuh)
__device__ __forceinline__ v3 slot_sel(const v3* X, int s) {
  return s == 0 ? X[0] : (s == 1 ? X[1] : (s == 2 ? X[2] : X[3]));
}
__device__ __forceinline__ void sd_make_y(int kind, int type, const v3* X, SubDist& S, double (*cy)[3]) {
  int w0 = 0, w1 = 0, e0 = -1, e1 = -1, f0 = -1, f1 = -1;   // w = x_w0 − x_w1, e1 = x_e1 − x_e0, e2 = x_f1 − x_f0
  if (kind == 0) {
    if (type == PT_T) { S.sub = SUB_TRI; w0 = 0; w1 = 1; e0 = 1; e1 = 2; f0 = 1; f1 = 3; }
    else if (type < PT_V0) { const int i = type - PT_E0; S.sub = SUB_PL; w0 = 0; w1 = 1 + i; e0 = 1 + i; e1 = 1 + (i + 1) % 3; }
    else { S.sub = SUB_PP; w0 = 0; w1 = 1 + type - PT_V0; }
  } else {
    const int ss = type / 3, ts = type % 3;
    if (ss == 1 && ts == 1) { S.sub = SUB_TRI; w0 = 0; w1 = 2; e0 = 0; e1 = 1; f0 = 2; f1 = 3; }
    else if (ss == 1) { S.sub = SUB_PL; w0 = ts == 0 ? 2 : 3; w1 = 0; e0 = 0; e1 = 1; }
    else if (ts == 1) { S.sub = SUB_PL; w0 = ss == 0 ? 0 : 1; w1 = 2; e0 = 2; e1 = 3; }
    else { S.sub = SUB_PP; w0 = ss == 0 ? 0 : 1; w1 = ts == 0 ? 2 : 3; }
  }
#pragma unroll
  for (int j = 0; j < 3; ++j) {
    cy[0][j] = (w0 == j + 1 ? 1.0 : 0.0) - (w1 == j + 1 ? 1.0 : 0.0);
    cy[1][j] = e0 < 0 ? 0.0 : (e1 == j + 1 ? 1.0 : 0.0) - (e0 == j + 1 ? 1.0 : 0.0);
    cy[2][j] = f0 < 0 ? 0.0 : (f1 == j + 1 ? 1.0 : 0.0) - (f0 == j + 1 ? 1.0 : 0.0);
  }
  S.w = slot_sel(X, w0) - slot_sel(X, w1);
  S.e1 = e0 < 0 ? mk(0, 0, 0) : slot_sel(X, e1) - slot_sel(X, e0);
  S.e2 = f0 < 0 ? mk(0, 0, 0) : slot_sel(X, f1) - slot_sel(X, f0);
  if (S.sub == SUB_PP) {
    S.s = dot(S.w, S.w);
  } else if (S.sub == SUB_PL) {
    S.ww = dot(S.w, S.w); S.D = dot(S.e1, S.e1); S.we = dot(S.w, S.e1);
    const v3 c = cross(S.w, S.e1);
    S.N = dot(c, c);
    S.s = S.N / S.D;
    S.iD = 1.0 / S.D; S.iD2 = S.iD * S.iD; S.iD3 = S.iD2 * S.iD;
  } else {
    S.n = cross(S.e1, S.e2); S.u = dot(S.w, S.n); S.D = dot(S.n, S.n);
    S.s = S.u * S.u / S.D;
    S.iD = 1.0 / S.D; S.iD2 = S.iD * S.iD; S.iD3 = S.iD2 * S.iD;
  }
}

// butterfly reduce-scatter of 32 per-lane values over a warp: afterwards v[0] of lane l holds
// Σ_lanes v[l] (fixed exchange pattern → deterministic); 31 shuffles for 32 sums
__device__ __forceinline__ void warp_reduce_scatter32(double* v, int lane) {
#pragma unroll
  for (int m = 16, n = 32; m > 0; m >>= 1, n >>= 1) {
    const bool up = (lane & m) != 0;
#pragma unroll
    for (int i = 0; i < n / 2; ++i) {
      const double send = up ? v[i] : v[n / 2 + i];
      const double keep = up ? v[n / 2 + i] : v[i];
      v[i] = keep + __shfl_xor_sync(0xffffffffu, send, m);
    }
  }
}
__constant__ unsigned char c_colpk[PH];    // column-order position be(be+1)/2+al → packed sym_idx(al, be)

__global__ void __launch_bounds__(128) k_pairs_x(Dev D, int env0, int force) {
  const int e = env_at(D, env0, blockIdx.y);
  const int sl = blockIdx.y;                   // slot in the assembly scratch (launch-local, < asm_envs)
  if (env_skip(D, e, force)) return;
  const EnvCtl& C = D.ctl[e];
  if (!C.exact) return;                                   // projected Hessians: k_pairs (warp Jacobi)
  const int nact = C.n_act;
  const double* P = D.P + (size_t)e * D.NVall * 3;
  const int* info = D.act_info + (size_t)e * D.act_cap * 4;
  const int* avid = D.act_vid + (size_t)e * D.act_cap * 4;
  double* aH = D.act_H + (size_t)e * D.res_cap * PH;
  const size_t e4 = (size_t)e * 4 * D.act_cap;
  __shared__ double sHy[45][128];                         // H_y of this thread's pair (records phase)
  const int tx = threadIdx.x;
#define HYS(r, c) ((r) <= (c) ? sHy[s9(r, c)][tx] : sHy[s9(c, r)][tx])
  const int lane = tx & 31;
  const size_t nchunk = (size_t)(D.act_cap + 31) >> 5;
  // warp-uniform sweep: lane l of a warp takes pair kb + l (the warp's 32-pair chunk kb/32)
  for (int kb = blockIdx.x * blockDim.x + (tx & ~31); kb < nact; kb += gridDim.x * blockDim.x) {
    const int k = kb + lane;
    const bool live = k < nact;
    double Gy[9];
    int codes[4] = {INT_MIN, INT_MIN, INT_MIN, INT_MIN};
    bool res = false;
    int bd0 = -1, bd1 = -1;            // DoF bodies of the pair (≤2), ascending
    const double* axb = D.act_xb + ((size_t)e * D.act_cap + (live ? k : 0)) * 12;
    double wc[3], wm[9];               // body pull-back weights (non-residual pairs touch ≤ 1 DoF body)
    auto weights = [&](int bd) {
      const bool on0 = codes[0] == -1 - bd;
      const double x00 = on0 ? axb[0] : 0.0, x01 = on0 ? axb[1] : 0.0, x02 = on0 ? axb[2] : 0.0;
#pragma unroll
      for (int l = 0; l < 3; ++l) {
        const bool on = codes[l + 1] == -1 - bd;
        wc[l] = (on ? 1.0 : 0.0) - (on0 ? 1.0 : 0.0);
        wm[3 * l] = (on ? axb[3 * (l + 1)] : 0.0) - x00;
        wm[3 * l + 1] = (on ? axb[3 * (l + 1) + 1] : 0.0) - x01;
        wm[3 * l + 2] = (on ? axb[3 * (l + 1) + 2] : 0.0) - x02;
      }
    };
    if (live) {
    if (reinterpret_cast<const int4*>(info)[k].x >= 2) {
      // lagged friction pair (reading R20): φ(w) = Δt²μλ f0(‖P_T w‖), w = Σ_j Γ_j (y_j − yⁿ_j); in
      // y-space G_y[j] = Γ_j ∇φ, H_y[j][l] = Γ_j Γ_l ∇²φ with ∇φ = (f1(z)/z) P_T w and
      // ∇²φ = (f1(z)/z) P_T + (f1′(z) − f1(z)/z) ûûᵀ (PSD for the paper's f1; z = ‖P_T w‖, û = P_T w / z)
      const int4 vv = reinterpret_cast<const int4*>(avid)[k];
      const v3 X[4] = {ld3(P + 3 * vv.x), ld3(P + 3 * vv.y), ld3(P + 3 * vv.z), ld3(P + 3 * vv.w)};
      const double* fd = D.fr_dat + ((size_t)e * D.act_cap + (k - (C.n_act - C.n_fr))) * 16;
      const double eps = D.eps_v * D.dt;
      v3 w = mk(0, 0, 0);
#pragma unroll
      for (int j = 0; j < 3; ++j) w += fd[4 + j] * ((X[j + 1] - X[0]) - ld3(fd + 7 + 3 * j));
      const v3 nh = ld3(fd + 1);
      const v3 vt = w - dot(nh, w) * nh;
      const double z2 = dot(vt, vt), z = sqrt(z2), sc = fd[0];
      double a, bq;                                    // ∇²φ = sc (a P_T + bq v vᵀ)
      if (z < eps) { a = -z / (eps * eps) + 2.0 / eps; bq = z > 0.0 ? -1.0 / (eps * eps * z) : 0.0; }
      else { a = 1.0 / z; bq = -1.0 / (z * z2); }
      const double V3[3] = {vt.x, vt.y, vt.z}, N3[3] = {nh.x, nh.y, nh.z};
      double Hw[9];
#pragma unroll
      for (int r = 0; r < 3; ++r)
#pragma unroll
        for (int c = 0; c < 3; ++c) Hw[3 * r + c] = sc * (a * ((r == c ? 1.0 : 0.0) - N3[r] * N3[c]) + bq * V3[r] * V3[c]);
      const double gam[3] = {fd[4], fd[5], fd[6]};
#pragma unroll
      for (int j = 0; j < 3; ++j)
#pragma unroll
        for (int r = 0; r < 3; ++r) Gy[3 * j + r] = gam[j] * sc * a * V3[r];
#pragma unroll
      for (int r = 0; r < 9; ++r)
#pragma unroll
        for (int c = r; c < 9; ++c) sHy[s9(r, c)][tx] = gam[r / 3] * gam[c / 3] * Hw[3 * (r % 3) + (c % 3)];
    } else {
      const int4 inf = reinterpret_cast<const int4*>(info)[k];
      const int kind = inf.x, type = inf.y, pa = inf.z, pb = inf.w;
      const int4 vv = reinterpret_cast<const int4*>(avid)[k];
      SubDist SD;
      double cy[3][3];
      double m = 1.0, m1 = 0.0, m2 = 0.0;
      const bool useM = (kind == 1) && D.mollify;
      v3 CE1v = mk(0, 0, 0), CE2v = mk(0, 0, 0), CNv = mk(0, 0, 0);   // mollifier c = ‖(a1−a0)×(b1−b0)‖²
      {
        const v3 X[4] = {ld3(P + 3 * vv.x), ld3(P + 3 * vv.y), ld3(P + 3 * vv.z), ld3(P + 3 * vv.w)};
        sd_make_y(kind, type, X, SD, cy);
        if (useM) {
          CE1v = X[1] - X[0]; CE2v = X[3] - X[2]; CNv = cross(CE1v, CE2v);
          mollifier(dot(CNv, CNv), pair_eps(D, kind, pa, pb), &m, &m1, &m2);
        }
      }
      double B, B1, B2;
      barrier_s(SD.s, D.dhat, &B, &B1, &B2);
      const bool molterm = useM && m1 != 0.0;
      const double scale = D.dt * D.dt * D.kappa * pair_area(D, kind, pa, pb);
      const double W[3] = {SD.w.x, SD.w.y, SD.w.z}, E1[3] = {SD.e1.x, SD.e1.y, SD.e1.z},
                   E2[3] = {SD.e2.x, SD.e2.y, SD.e2.z}, Nn[3] = {SD.n.x, SD.n.y, SD.n.z};
      // var-space first derivatives (var v, component a): u1 (∂u / ∂N), d1 (∂D), g = ∂s
      double u1[9], d1[9], gys[9];
      {
        double gv[9];
#pragma unroll
        for (int v = 0; v < 3; ++v)
#pragma unroll
          for (int a = 0; a < 3; ++a) {
            const int a1 = (a + 1) % 3, a2 = (a + 2) % 3;
            double uu = 0.0, dd = 0.0, g1;
            if (SD.sub == SUB_TRI) {
              if (v == 0) uu = Nn[a];
              else if (v == 1) uu = E2[a1] * W[a2] - E2[a2] * W[a1];
              else uu = W[a1] * E1[a2] - W[a2] * E1[a1];
              if (v == 1) dd = 2.0 * (E2[a1] * Nn[a2] - E2[a2] * Nn[a1]);
              else if (v == 2) dd = 2.0 * (Nn[a1] * E1[a2] - Nn[a2] * E1[a1]);
              g1 = 2.0 * SD.u * uu * SD.iD - SD.u * SD.u * dd * SD.iD2;
            } else if (SD.sub == SUB_PL) {
              if (v == 0) uu = 2.0 * (SD.D * W[a] - SD.we * E1[a]);
              else if (v == 1) uu = 2.0 * (SD.ww * E1[a] - SD.we * W[a]);
              if (v == 1) dd = 2.0 * E1[a];
              g1 = uu * SD.iD - SD.N * dd * SD.iD2;
            } else {
              uu = v == 0 ? 2.0 * W[a] : 0.0;
              g1 = uu;
            }
            u1[3 * v + a] = uu; d1[3 * v + a] = dd; gv[3 * v + a] = g1;
          }
#pragma unroll
        for (int j = 0; j < 3; ++j)
#pragma unroll
          for (int a = 0; a < 3; ++a)
            gys[3 * j + a] = cy[0][j] * gv[a] + cy[1][j] * gv[3 + a] + cy[2][j] * gv[6 + a];
      }
      double Hy[45];
      // H_y = scale [ m (B2 gs gsᵀ + B1 ∇²s) + (mollifier) B (m2 gc gcᵀ + m1 ∇²c) + m1 B1 (gs gcᵀ + gc gsᵀ) ]
      {
        double gyc[9];
        const double CE1[3] = {CE1v.x, CE1v.y, CE1v.z}, CE2[3] = {CE2v.x, CE2v.y, CE2v.z}, CN[3] = {CNv.x, CNv.y, CNv.z};
        // cross variables in y: a1 − a0 = y1, b1 − b0 = y3 − y2 (EE slot order a0, a1, b0, b1)
        constexpr double cyc[3][3] = {{0, 0, 0}, {1, 0, 0}, {0, -1, 1}};
#pragma unroll
        for (int a = 0; a < 3; ++a) {
          const int a1 = (a + 1) % 3, a2 = (a + 2) % 3;
          const double c1 = useM ? 2.0 * (CE2[a1] * CN[a2] - CE2[a2] * CN[a1]) : 0.0;   // ∂c/∂(a1−a0)
          const double c2 = useM ? 2.0 * (CN[a1] * CE1[a2] - CN[a2] * CE1[a1]) : 0.0;   // ∂c/∂(b1−b0)
#pragma unroll
          for (int j = 0; j < 3; ++j) gyc[3 * j + a] = cyc[1][j] * c1 + cyc[2][j] * c2;
        }
        const double r1 = scale * m * B2, rc = molterm ? scale * B * m2 : 0.0, rx = molterm ? scale * m1 * B1 : 0.0;
#pragma unroll
        for (int r = 0; r < 9; ++r)
#pragma unroll
          for (int c = r; c < 9; ++c)
            Hy[s9(r, c)] = r1 * gys[r] * gys[c] + rc * gyc[r] * gyc[c] + rx * (gys[r] * gyc[c] + gyc[r] * gys[c]);
#pragma unroll
        for (int i = 0; i < 9; ++i) Gy[i] = scale * (m * B1 * gys[i] + B * m1 * gyc[i]);
        if (molterm) {                 // B m1 ∇²c, c = ‖e1×e2‖² on the cross variables (vars 1, 2)
          const double wC = scale * B * m1;
#pragma unroll
          for (int v = 1; v < 3; ++v)
#pragma unroll
            for (int a = 0; a < 3; ++a)
#pragma unroll
              for (int u = 1; u < 3; ++u)
#pragma unroll
                for (int b = 0; b < 3; ++b) {
                  const double t = wC * tri_D2_fast(CE1, CE2, CN, v, a, u, b);
#pragma unroll
                  for (int j = 0; j < 3; ++j) {
                    const double tj = cyc[v][j] * t;
#pragma unroll
                    for (int l = 0; l < 3; ++l)
                      if (3 * j + a <= 3 * l + b) Hy[s9(3 * j + a, 3 * l + b)] += cyc[u][l] * tj;
                  }
                }
        }
      }
      {
        const double wS = scale * m * B1;
        if (SD.sub == SUB_TRI) scatter_sub<SUB_TRI>(Hy, cy, wS, W, E1, E2, Nn, u1, d1, SD);
        else if (SD.sub == SUB_PL) scatter_sub<SUB_PL>(Hy, cy, wS, W, E1, E2, Nn, u1, d1, SD);
        else scatter_sub<SUB_PP>(Hy, cy, wS, W, E1, E2, Nn, u1, d1, SD);
      }
#pragma unroll
      for (int i = 0; i < 45; ++i) sHy[i][tx] = Hy[i];
    }
    // ---- records (H_y from shared memory) ----
    const int4 c4 = reinterpret_cast<const int4*>(D.act_slot + e4)[k];
    codes[0] = c4.x; codes[1] = c4.y; codes[2] = c4.z; codes[3] = c4.w;
    const int ridx = D.act_res[(size_t)e * D.act_cap + k];
    res = ridx != 0;
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      const int cd = codes[t];
      if (cd < 0 && cd != INT_MIN) {
        const int d = -1 - cd;
        if (bd0 < 0) bd0 = d;
        else if (d != bd0) bd1 = d;
      }
    }
    if (bd1 >= 0 && bd1 < bd0) { const int tmp = bd0; bd0 = bd1; bd1 = tmp; }
    // residual pairs: packed upper slot-space 12×12 for the matrix-free SpMV pass
    if (res && ridx <= D.res_cap) {
      double* Hk = aH + (size_t)(ridx - 1) * PH;
#pragma unroll
      for (int s = 0; s < 4; ++s) {
#pragma unroll
        for (int t = s; t < 4; ++t)
#pragma unroll
          for (int r = 0; r < 3; ++r)
#pragma unroll
            for (int b = 0; b < 3; ++b) {
              if (t == s && b < r) continue;
              double v = 0.0;          // Σ_{j,l} σ_j(s) σ_l(t) H_y[(j,r),(l,b)]
#pragma unroll
              for (int j = 0; j < 3; ++j)
#pragma unroll
                for (int l = 0; l < 3; ++l) {
                  const int sj = s == 0 ? -1 : (s == j + 1 ? 1 : 0), tl = t == 0 ? -1 : (t == l + 1 ? 1 : 0);
                  if (sj * tl != 0) v += (double)(sj * tl) * HYS(3 * j + r, 3 * l + b);
                }
              Hk[sym_idx(3 * s + r, 3 * t + b, 12)] = v;
            }
      }
    }
    if (bd0 >= 0) weights(bd0);
    // per soft slot s, at its vertex-sorted position j: [g_s 3 | H_ss 9 | C_s 36 | H_st (≤2 soft t) 18]
    auto csel = [&](int t) { return t == 0 ? codes[0] : (t == 1 ? codes[1] : (t == 2 ? codes[2] : codes[3])); };
#pragma unroll 1
    for (int s = 0; s < 4; ++s) {
      const int cs = csel(s);
      if (cs < 0) continue;
      const double sg[3] = {s == 0 ? -1.0 : (s == 1 ? 1.0 : 0.0), s == 0 ? -1.0 : (s == 2 ? 1.0 : 0.0),
                            s == 0 ? -1.0 : (s == 3 ? 1.0 : 0.0)};
      const int j = D.spos[e4 + 4 * k + s];
      double Q[27];                    // Q[(l,b)·3 + r] = Σ_j σ_j(s) H_y[(j,r),(l,b)]  (slot-s row block)
#pragma unroll
      for (int lb = 0; lb < 9; ++lb)
#pragma unroll
        for (int r = 0; r < 3; ++r) {
          double q = 0.0;
#pragma unroll
          for (int jj = 0; jj < 3; ++jj) q += sg[jj] * HYS(3 * jj + r, lb);
          Q[3 * lb + r] = q;
        }
      double* rec = D.srec + ((size_t)sl * 4 * D.act_cap + j) * SREC;
#pragma unroll
      for (int a = 0; a < 3; ++a) {
        double gg = 0.0;
#pragma unroll
        for (int jj = 0; jj < 3; ++jj) gg += sg[jj] * Gy[3 * jj + a];
        rec[a] = gg;
      }
      // slot-space block H_st from Q
      auto Hst = [&](int t, int r, int b) {
        double v = 0.0;
#pragma unroll
        for (int l = 0; l < 3; ++l) v += (t == 0 ? -1.0 : (t == l + 1 ? 1.0 : 0.0)) * Q[3 * (3 * l + b) + r];
        return v;
      };
#pragma unroll
      for (int r = 0; r < 3; ++r)
#pragma unroll
        for (int b = 0; b < 3; ++b) rec[3 + 3 * r + b] = Hst(s, r, b);
      // C_s = Σ_{t on bd0} H_st J_t (zero for residual pairs)
      const bool cpl = !res && bd0 >= 0;
#pragma unroll
      for (int r = 0; r < 3; ++r)
#pragma unroll
        for (int be = 0; be < 12; ++be) {
          double v = 0.0;
          if (cpl) {
            const int rb = be < 3 ? be : (be - 3) / 3;
#pragma unroll
            for (int l = 0; l < 3; ++l) v += (be < 3 ? wc[l] : wm[3 * l + (be - 3) % 3]) * Q[3 * (3 * l + rb) + r];
          }
          rec[12 + 12 * r + be] = v;
        }
      // soft neighbours (the other soft slots, ascending; zero for residual pairs)
      int nn = 0;
#pragma unroll 1
      for (int t = 0; t < 4; ++t) {
        if (t == s || csel(t) < 0 || nn >= 2) continue;
        const int nb = nn++;
#pragma unroll
        for (int r = 0; r < 3; ++r)
#pragma unroll
          for (int b = 0; b < 3; ++b) rec[48 + 9 * nb + 3 * r + b] = res ? 0.0 : Hst(t, r, b);
        int jb = -1;
        if (!res) {        // non-residual: all soft slots on one primitive → template block table
          const int4 inf = reinterpret_cast<const int4*>(info)[k];
          if ((inf.x & 1) == 0) {
            const int i = s - 1, j = t - 1;
            jb = D.tri_blk[6 * (size_t)inf.w + 2 * i + (j < i ? j : j - 1)];
          } else {
            jb = D.edge_blk[2 * (size_t)(s < 2 ? inf.z : inf.w) + (s & 1)];
          }
        }
        D.snb[((size_t)sl * 4 * D.act_cap + j) * 2 + nb] = jb;
      }
      for (int nb = nn; nb < 2; ++nb) {
        for (int i = 0; i < 9; ++i) rec[48 + 9 * nb + i] = 0.0;
        D.snb[((size_t)sl * 4 * D.act_cap + j) * 2 + nb] = -1;
      }
      D.sbody[(size_t)sl * 4 * D.act_cap + j] = res ? -1 : bd0;
    }
    }  // live
    // per (32-pair chunk, DoF body) partial sums of the body records, deterministic warp trees:
    // [Σ J_sᵀ g_s 12 | condensed packed Σ J_sᵀ H_st J_t 78 | residual-pair packed 78] (k_assemble sums
    // the chunks of a body in chunk order)
    const size_t chunk = (size_t)kb >> 5;
    for (int d = 0; d < D.ND; ++d) {
      const bool mine = bd0 == d || bd1 == d;
      double* out = D.bpart + (((size_t)sl * nchunk + chunk) * D.ND + d) * BPART;
      if (__ballot_sync(0xffffffffu, mine) == 0u) {
        for (int i = lane; i < BPART; i += 32) out[i] = 0.0;
        continue;
      }
      const bool anyres = __ballot_sync(0xffffffffu, mine && res) != 0u;
      if (mine) weights(d);
      else {
#pragma unroll
        for (int l = 0; l < 3; ++l) wc[l] = 0.0;
#pragma unroll
        for (int l = 0; l < 9; ++l) wm[l] = 0.0;
      }
      // 32-entry chunks, each reduced over the warp by a butterfly reduce-scatter (31 shuffles per
      // chunk instead of 5 per entry; fixed tree → deterministic); entries in column order
      // p = be(be+1)/2 + al, lane l stores entry 32c + l of chunk c
      {
        double val[32];
#pragma unroll
        for (int al = 0; al < 12; ++al) {
          const int ra = al < 3 ? al : (al - 3) / 3;
          double v = 0.0;
#pragma unroll
          for (int jj = 0; jj < 3; ++jj) v += (al < 3 ? wc[jj] : wm[3 * jj + (al - 3) % 3]) * Gy[3 * jj + ra];
          val[al] = mine ? v : 0.0;
        }
#pragma unroll
        for (int i = 12; i < 32; ++i) val[i] = 0.0;
        warp_reduce_scatter32(val, lane);
        if (lane < 12) out[lane] = val[0];
      }
      for (int pass = 0; pass < (anyres ? 2 : 1); ++pass) {
        double val[32];
#pragma unroll
        for (int be = 0; be < 12; ++be) {
          const int rb = be < 3 ? be : (be - 3) / 3;
          double zc[9];                // zc[(j,r)] = Σ_l w_l(β) H_y[(j,r),(l,ρβ)]
#pragma unroll
          for (int jr = 0; jr < 9; ++jr) {
            double z = 0.0;
            if (mine)
#pragma unroll
              for (int l = 0; l < 3; ++l) z += (be < 3 ? wc[l] : wm[3 * l + (be - 3) % 3]) * HYS(jr, 3 * l + rb);
            zc[jr] = z;
          }
#pragma unroll
          for (int al = 0; al <= be; ++al) {
            const int ra = al < 3 ? al : (al - 3) / 3;
            double v = 0.0;
#pragma unroll
            for (int jj = 0; jj < 3; ++jj) v += (al < 3 ? wc[jj] : wm[3 * jj + (al - 3) % 3]) * zc[3 * jj + ra];
            const int pos = be * (be + 1) / 2 + al;
            val[pos & 31] = (res == (pass == 1)) ? v : 0.0;
            if ((pos & 31) == 31 || pos == PH - 1) {
              if (pos == PH - 1)
#pragma unroll
                for (int i = (PH & 31); i < 32; ++i) val[i] = 0.0;
              warp_reduce_scatter32(val, lane);
              const int p0 = pos & ~31;
              if (p0 + lane < PH) out[12 + pass * PH + c_colpk[p0 + lane]] = val[0];
            }
          }
        }
      }
      if (!anyres)
        for (int i = lane; i < PH; i += 32) out[12 + PH + i] = 0.0;
    }
  }
#undef HYS
}


// ------------------------------------------------------------------------------------------
// assembly: gradient g, soft BSR (diag + edge blocks), body 12×12 blocks, block-Jacobi inverses
// ------------------------------------------------------------------------------------------
#ifdef TAC_CLOCKS   // per-section clock64 accumulators of k_pcg (tools/pcg_clocks.py; not in the product build)
__device__ unsigned long long g_clk[32];
#define CLK_INIT long long clk_t = clock64();
#define CLK_COUNT atomicAdd(&g_clk[15], 1ull);
#define CLKN(i) atomicAdd(&g_clk[i], 1ull);
#define CLKT(i) { const long long t_ = clock64(); atomicAdd(&g_clk[i], (unsigned long long)(t_ - clk_t)); atomicMax(&g_clk[i + 4], (unsigned long long)(t_ - clk_t)); clk_t = t_; }
#define CLKR clk_t = clock64();
#define CLK(i) if (threadIdx.x == 0) { const long long t_ = clock64(); atomicAdd(&g_clk[i], (unsigned long long)(t_ - clk_t)); clk_t = t_; }
extern "C" int tac_debug_clocks(unsigned long long* out) {
  cudaDeviceSynchronize();
  cudaMemcpyFromSymbol(out, g_clk, sizeof(g_clk));
  unsigned long long z[32] = {};
  return (int)cudaMemcpyToSymbol(g_clk, z, sizeof(g_clk));
}
#else
#define CLK_INIT
#define CLK(i)
#define CLK_COUNT ;
#define CLKN(i) ;
#define CLKT(i)
#define CLKR
#endif

__device__ void chol_inverse12(const double* A, double* Ainv, double* L /*144 scratch*/) {
  // single thread: Cholesky A = L Lᵀ then Ainv = L⁻ᵀ L⁻¹
  for (int i = 0; i < 144; ++i) L[i] = 0.0;
  for (int j = 0; j < 12; ++j) {
    double s = A[13 * j];
    for (int k = 0; k < j; ++k) s -= L[12 * j + k] * L[12 * j + k];
    double ljj = sqrt(fmax(s, 1e-300));
    L[13 * j] = ljj;
    for (int i = j + 1; i < 12; ++i) {
      double t = A[12 * i + j];
      for (int k = 0; k < j; ++k) t -= L[12 * i + k] * L[12 * j + k];
      L[12 * i + j] = t / ljj;
    }
  }
  for (int c = 0; c < 12; ++c) {
    double y[12];
    for (int i = 0; i < 12; ++i) {  // L y = e_c
      double t = (i == c) ? 1.0 : 0.0;
      for (int k = 0; k < i; ++k) t -= L[12 * i + k] * y[k];
      y[i] = t / L[13 * i];
    }
    for (int i = 11; i >= 0; --i) {  // Lᵀ x = y
      double t = y[i];
      for (int k = i + 1; k < 12; ++k) t -= L[12 * k + i] * y[k];
      y[i] = t / L[13 * i];
    }
    for (int i = 0; i < 12; ++i) Ainv[12 * i + c] = y[i];
  }
}

// the same factorisation and solves as chol_inverse12 (identical operation order per entry), spread
// over a warp: lanes i > j form column j of L from row dot products; lane c solves column c
__device__ void chol_inverse12_warp(const double* A, double* Ainv, double* L /*144 scratch*/, int lane) {
  for (int j = 0; j < 12; ++j) {
    if (lane == 0) {
      double s = A[13 * j];
      for (int k = 0; k < j; ++k) s -= L[12 * j + k] * L[12 * j + k];
      L[13 * j] = sqrt(fmax(s, 1e-300));
    }
    __syncwarp();
    if (lane > j && lane < 12) {
      double t = A[12 * lane + j];
      for (int k = 0; k < j; ++k) t -= L[12 * lane + k] * L[12 * j + k];
      L[12 * lane + j] = t / L[13 * j];
    }
    __syncwarp();
  }
  if (lane < 12) {
    const int c = lane;
    double y[12];
#pragma unroll
    for (int i = 0; i < 12; ++i) {  // L y = e_c
      double t = (i == c) ? 1.0 : 0.0;
#pragma unroll
      for (int k = 0; k < i; ++k) t -= L[12 * i + k] * y[k];
      y[i] = t / L[13 * i];
    }
#pragma unroll
    for (int i = 11; i >= 0; --i) {  // Lᵀ x = y
      double t = y[i];
#pragma unroll
      for (int k = i + 1; k < 12; ++k) t -= L[12 * k + i] * y[k];
      y[i] = t / L[13 * i];
    }
#pragma unroll
    for (int i = 0; i < 12; ++i) Ainv[12 * i + c] = y[i];
  }
  __syncwarp();
}

// elastic soft edge blocks, grid-parallel over (edge tile, env): one thread per soft edge {i < j} sums its
// tets' (i, j) block once (template list eblk, in order) and stores it and its transpose — into the
// sliced-ELL copy the streamed PCG reads (asm_ell) or the row-ordered blocks.  Split out of k_assemble_soft,
// where 256 threads per env walked the edges one after another (latency-bound dependent loads)
__global__ void __launch_bounds__(NTHREADS) k_asm_edges(Dev D, int env0, int force) {
  const int e = env_at(D, env0, blockIdx.y);
  const int sl = blockIdx.y;                   // slot in the assembly scratch (launch-local, < asm_envs)
  if (env_skip(D, e, force)) return;
  const int ei = blockIdx.x * blockDim.x + threadIdx.x;
  if (ei >= D.NEs) return;
  const double* tb = D.tetbuf + (size_t)sl * TETBUF * D.T;
  double* const He = D.asm_ell ? D.Hell + (size_t)e * D.ell_total : nullptr;
  {
    double B[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
    for (int j = D.eblk_ptr[ei]; j < D.eblk_ptr[ei + 1]; ++j) {
      int ent = D.eblk[j], t = ent >> 4, a = (ent >> 2) & 3, b = ent & 3;
#pragma unroll
      for (int r = 0; r < 3; ++r)
#pragma unroll
        for (int c = 0; c < 3; ++c) B[3 * r + c] += tb[(size_t)(12 + sym_idx(3 * a + r, 3 * b + c, 12)) * D.T + t];
    }
    const int qu = D.eup[ei], ql = D.elo[ei];
    if (He) {
      double* hu = He + D.ell_pos[qu];
      double* hl = He + D.ell_pos[ql];
#pragma unroll
      for (int r = 0; r < 3; ++r)
#pragma unroll
        for (int c = 0; c < 3; ++c) { hu[32 * (3 * r + c)] = B[3 * r + c]; hl[32 * (3 * c + r)] = B[3 * r + c]; }
    } else {
      double* hu = D.Ho + ((size_t)e * D.NNZ + qu) * 9;
      double* hl = D.Ho + ((size_t)e * D.NNZ + ql) * 9;
#pragma unroll
      for (int r = 0; r < 3; ++r)
#pragma unroll
        for (int c = 0; c < 3; ++c) { hu[3 * r + c] = B[3 * r + c]; hl[3 * c + r] = B[3 * r + c]; }
    }
  }
}

// soft part of the assembly (elastic edge and diagonal blocks, gradient, condensed contact terms,
// 3×3 block-Jacobi inverses); register-light, so it runs at higher occupancy than the body part
constexpr int ASM_SOFT_MAX = 320;
// MINB: 3 CTAs/SM (64 registers) for envs that fit one pass of ≤ 320 threads (C2: assemble 135 -> 123 ms / 20
// steps), 2 otherwise (C3 measured 1.63 -> 2.27 s / 10 steps at 3)
template <int MINB>
__global__ void __launch_bounds__(ASM_SOFT_MAX, MINB) k_assemble_soft(Dev D, int env0, int force) {
  const int e = env_at(D, env0, blockIdx.x);
  const int sl = blockIdx.x;                   // slot in the assembly scratch (launch-local, < asm_envs)
  if (env_skip(D, e, force)) return;
  __shared__ int shs[33];
  __shared__ int next_cv;
  extern __shared__ double dsm_asm[];   // contact-vertex list [V] ints
  EnvCtl& C = D.ctl[e];
  double* g = D.g + (size_t)e * D.n;
  const int* cptr = D.cptr + (size_t)e * (D.V + 1);
  CLK_INIT
  // the elastic edge blocks come from k_asm_edges (grid-parallel, launched before this kernel)
  double* const He = D.asm_ell ? D.Hell + (size_t)e * D.ell_total : nullptr;
  CLK(10)
  // ---- soft vertices: gradient, diagonal blocks, and the condensed contact terms of row v ----
  int* cpp = D.cpl_ptr + (size_t)e * (D.V + 1);
  int* cplv = D.cpl_v + (size_t)e * D.cpl_cap;
  int* cpld = D.cpl_d + (size_t)e * D.cpl_cap;
  double* cval = D.cpl_val + (size_t)e * 36 * D.cpl_cap;
  double* Hoe = D.Ho + (size_t)e * D.NNZ * 9;
  const int* rcnt = D.rcnt + (size_t)e * D.V;
  const double* srec = D.srec + (size_t)sl * 4 * D.act_cap * SREC;
  const int* snb = D.snb + (size_t)sl * 4 * D.act_cap * 2;
  const int* sbody = D.sbody + (size_t)sl * 4 * D.act_cap;
  int* cvl = reinterpret_cast<int*>(dsm_asm);        // [V] soft vertices with contact records
  double* accs = dsm_asm + (D.V + 3) / 2;             // [ngrp][maxrl][9] soft–soft block sums
  int cpl_run = 0, nct = 0;
  // phase 1 (thread per vertex): inertia, gravity, AL and elastic terms; body mask of the condensed
  // records; coupling offsets and the contact-vertex list by block scans (a grid-parallel split of the vertex
  // terms, like k_asm_edges, measured no faster)
  const double* q = D.q + (size_t)e * D.n;
  const double* qt = D.qt + (size_t)e * D.n;
  const double* tb = D.tetbuf + (size_t)sl * TETBUF * D.T;
  const double dt2 = D.dt * D.dt, rho = C.rho;
  const double* s_att = D.s_att + (size_t)e * D.NC * 3;
  const double* lam_att = D.lam_att + (size_t)e * D.NC * 3;
  for (int v0 = 0; v0 < D.V; v0 += blockDim.x) {
    const int v = v0 + threadIdx.x;
    unsigned bmask = 0u;
    int hasc = 0;
    if (v < D.V) {
      const double m = D.mass[v];
      v3 x = ld3(q + 3 * v), xt = ld3(qt + 3 * v);
      v3 gv = m * (x - xt) - (dt2 * m) * mk(D.grav[0], D.grav[1], D.grav[2]);
      double dg = m;
      int ci = D.att_of_vert[v];
      if (ci >= 0) {
        v3 r = x - ld3(s_att + 3 * ci);
        gv += (rho * m) * r - m * ld3(lam_att + 3 * ci);
        dg += rho * m;
      }
      double Hv[9] = {dg, 0, 0, 0, dg, 0, 0, 0, dg};
      for (int j = D.vdiag_ptr[v]; j < D.vdiag_ptr[v + 1]; ++j) {
        int ent = D.vdiag[j], t = ent >> 2, a = ent & 3;
        gv += mk(tb[(size_t)(3 * a) * D.T + t], tb[(size_t)(3 * a + 1) * D.T + t], tb[(size_t)(3 * a + 2) * D.T + t]);
        for (int r = 0; r < 3; ++r)
          for (int c = 0; c < 3; ++c) Hv[3 * r + c] += tb[(size_t)(12 + sym_idx(3 * a + r, 3 * a + c, 12)) * D.T + t];
      }
      const int j0 = cptr[v], j1 = cptr[v + 1];
      hasc = j1 > j0;
      for (int j = j0 + rcnt[v]; j < j1; ++j) { const int d = sbody[j]; if (d >= 0) bmask |= 1u << d; }
      st3(g + 3 * v, gv);
      double* hd = D.Hd + (size_t)e * D.V * 9;           // SoA [9][V]: SpMV diagonal (contact added in phase 2)
      double* ds = D.Dg_s + (size_t)e * D.V * 9;         // raw diagonal block (SoA) for LM re-inversion
      for (int i = 0; i < 9; ++i) { hd[(size_t)i * D.V + v] = Hv[i]; ds[(size_t)i * D.V + v] = Hv[i]; }
      if (!hasc) {
        const double sh = C.mu * m;                       // mass-scaled LM shift μ·m_v I (R14c)
        Hv[0] += sh; Hv[4] += sh; Hv[8] += sh;
        double Pi[9];
        inv33(Hv, Pi);
        double* ps = D.Pinv_s + (size_t)e * D.V * 9;     // SoA [9][V]
        for (int i = 0; i < 9; ++i) ps[(size_t)i * D.V + v] = Pi[i];
      }
    }
    int tot, totc;
    const int ex = block_excl_scan(__popc(bmask), shs, &tot);
    const int exc = block_excl_scan(hasc, shs, &totc);
    if (v < D.V) {
      cpp[v] = cpl_run + ex;
      if (hasc) cvl[nct + exc] = v;
      for (unsigned mm = bmask; mm; mm &= mm - 1) {
        const int d = __ffs(mm) - 1, pos = cpl_run + ex + __popc(bmask & ((1u << d) - 1u));
        cplv[pos] = v; cpld[pos] = d;
      }
    }
    cpl_run += tot;
    nct += totc;
  }
  __syncthreads();
  CLK(16)
  // phase 2 (8-lane group per contact vertex): sum the vertex's condensed records, field-parallel
  // (lane l8 owns fields l8 + 8i of [g 3 | H_ss 9 | C 36]); entries in vertex-sorted order
  {
    const int l8 = threadIdx.x & 7, grp = threadIdx.x >> 3;
    double* hd = D.Hd + (size_t)e * D.V * 9;
    double* ds = D.Dg_s + (size_t)e * D.V * 9;
    // dynamic assignment of contact vertices to 8-lane groups (a vertex is summed by one group in a
    // fixed record order, so results do not depend on the assignment)
    const unsigned gmask = 0xFFu << (threadIdx.x & 24);
    if (threadIdx.x == 0) next_cv = 0;
    __syncthreads();
    for (;;) {
      int ci = 0;
      if (l8 == 0) ci = atomicAdd(&next_cv, 1);
      ci = __shfl_sync(gmask, ci, threadIdx.x & 24);
      if (ci >= nct) break;
      const int v = cvl[ci];
      const int j0 = cptr[v], jr = j0 + rcnt[v], j1 = cptr[v + 1];
      unsigned bmask = 0u;
      for (int j = jr; j < j1; ++j) { const int d = sbody[j]; if (d >= 0) bmask |= 1u << d; }
      const int dlo = bmask ? __ffs(bmask) - 1 : -1;
      double aa[6] = {0, 0, 0, 0, 0, 0}, an[6] = {0, 0, 0, 0, 0, 0};
#pragma unroll 4
      for (int j = j0; j < j1; ++j) {
        const double* rec = srec + (size_t)j * SREC;
        const bool nr = j >= jr;
        const bool cp = nr && sbody[j] == dlo;
#pragma unroll
        for (int i = 0; i < 6; ++i) {
          const int f = l8 + 8 * i;
          const double val = rec[f];
          if (f < 12) { aa[i] += val; if (nr) an[i] += val; }
          else if (cp) an[i] += val;
        }
      }
      const int base = cpp[v];
#pragma unroll
      for (int i = 0; i < 6; ++i) {
        const int f = l8 + 8 * i;
        if (f < 3) g[3 * v + f] += aa[i];
        else if (f < 12) { hd[(size_t)(f - 3) * D.V + v] += an[i]; ds[(size_t)(f - 3) * D.V + v] += aa[i]; }
        else if (dlo >= 0) cval[(size_t)(f - 12) * D.cpl_cap + base] = an[i];
      }
      // further bodies of this vertex (rare), ascending
      for (unsigned mm = bmask & (bmask - 1u); mm; mm &= mm - 1) {
        const int d = __ffs(mm) - 1, pos = base + __popc(bmask & ((1u << d) - 1u));
        for (int f = 12 + l8; f < 48; f += 8) {
          double a = 0.0;
          for (int j = jr; j < j1; ++j)
            if (sbody[j] == d) a += srec[(size_t)j * SREC + f];
          cval[(size_t)(f - 12) * D.cpl_cap + pos] = a;
        }
      }
      // soft–soft contact blocks folded into row v's BSR blocks (lane l8 owns element l8, lane 0 also 8):
      // summed per block of row v in shared memory in record order, then one read-modify-write per
      // touched block (independent, so the global round trips overlap)
      if (D.maxrl <= 32) {
        const int r0 = D.rptr[v], rl = D.rptr[v + 1] - r0;
        double* acc = accs + (size_t)grp * D.maxrl * 9;
        for (int sl = 0; sl < rl; ++sl) { acc[9 * sl + l8] = 0.0; if (l8 == 0) acc[9 * sl + 8] = 0.0; }
        unsigned touched = 0u;
        for (int j = jr; j < j1; ++j)
          for (int nb = 0; nb < 2; ++nb) {
            const int jb = snb[2 * j + nb];
            if (jb < 0) continue;
            const int sl = jb - r0;
            touched |= 1u << sl;
            const double* rec = srec + (size_t)j * SREC + 48 + 9 * nb;
            acc[9 * sl + l8] += rec[l8];
            if (l8 == 0) acc[9 * sl + 8] += rec[8];
          }
        for (unsigned m = touched; m; m &= m - 1u) {
          const int sl = __ffs(m) - 1;
          const int hs = He ? 32 : 1;                     // element stride of the block's storage
          double* hb = He ? He + D.ell_pos[r0 + sl] : Hoe + (size_t)(r0 + sl) * 9;
          hb[hs * l8] += acc[9 * sl + l8];
          if (l8 == 0) hb[hs * 8] += acc[9 * sl + 8];
        }
      } else {
        for (int j = jr; j < j1; ++j)
          for (int nb = 0; nb < 2; ++nb) {
            const int jb = snb[2 * j + nb];
            if (jb < 0) continue;
            const int hs = He ? 32 : 1;
            double* hb = He ? He + D.ell_pos[jb] : Hoe + (size_t)jb * 9;
            const double* rec = srec + (size_t)j * SREC + 48 + 9 * nb;
            hb[hs * l8] += rec[l8];
            if (l8 == 0) hb[hs * 8] += rec[8];
          }
      }
    }
  }
  __syncthreads();
  CLK(17)
  // phase 3: block-Jacobi inverses of the contact vertices
  for (int ci = threadIdx.x; ci < nct; ci += blockDim.x) {
    const int v = cvl[ci];
    const double* ds = D.Dg_s + (size_t)e * D.V * 9;
    double Pv[9], Pi[9];
    for (int i = 0; i < 9; ++i) Pv[i] = ds[(size_t)i * D.V + v];
    const double sh = C.mu * D.mass[v];
    Pv[0] += sh; Pv[4] += sh; Pv[8] += sh;
    inv33(Pv, Pi);
    double* ps = D.Pinv_s + (size_t)e * D.V * 9;
    for (int i = 0; i < 9; ++i) ps[(size_t)i * D.V + v] = Pi[i];
  }
  if (threadIdx.x == 0) { cpp[D.V] = cpl_run; C.n_cpl = cpl_run; }
  CLK(11)
}

// body part of the assembly: inertia, orthogonality, gravity and AL terms of the DoF bodies, the
// pairs' body blocks (k_pairs_x partials) and the 12×12 block-Jacobi inverses
__global__ void __launch_bounds__(NTHREADS, 2) k_assemble_body(Dev D, int env0, int force) {
  const int e = env_at(D, env0, blockIdx.x);
  const int sl = blockIdx.x;                   // slot in the assembly scratch (launch-local, < asm_envs)
  if (env_skip(D, e, force)) return;
  __shared__ JacobiScratch JS[NTHREADS / 32];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  EnvCtl& C = D.ctl[e];
  const double* q = D.q + (size_t)e * D.n;
  const double* qt = D.qt + (size_t)e * D.n;
  double* g = D.g + (size_t)e * D.n;
  const double dt2 = D.dt * D.dt, rho = C.rho;
  CLK_INIT
  // ---- affine DoF bodies: warp per body ----
  for (int d = w; d < D.ND; d += nw) {
    const int b = D.dof_body[d];
    const double* y = q + 3 * D.V + 12 * d;
    const double* yt = qt + 3 * D.V + 12 * d;
    const double* M = D.My + (size_t)b * 144;
    const int ki = D.kin_of_body[b];
    const double* sk = ki >= 0 ? D.s_kin + ((size_t)e * D.NK + ki) * 12 : nullptr;
    const double* lk = ki >= 0 ? D.lam_kin + ((size_t)e * D.NK + ki) * 12 : nullptr;
    const double kv = dt2 * D.bkappa[b] * D.bvol[b];
    JacobiScratch& S = JS[w];
    // ortho 9×9 into the 12×12 scratch (zero padded), projected
    for (int i = lane; i < 144; i += 32) {
      int r = i / 12, c = i % 12;
      S.A[i] = (r < 9 && c < 9) ? ortho_hess_entry(y + 3, kv, r, c) : 0.0;
    }
    __syncwarp();
    if (!C.exact) jacobi12_psd(S, lane, 32);
    double gb = 0.0;
    if (lane < 12) {
      int al = lane;
      double acc = 0.0;
      for (int be = 0; be < 12; ++be) acc += M[12 * al + be] * (y[be] - yt[be]);
      if (ki >= 0) {
        double a2 = 0.0, a3 = 0.0;
        for (int be = 0; be < 12; ++be) { a2 += M[12 * al + be] * (y[be] - sk[be]); a3 += M[12 * al + be] * lk[be]; }
        acc += rho * a2 - a3;
      }
      if (al < 3) acc -= dt2 * D.bmass[b] * D.grav[al];
      else acc -= dt2 * D.grav[(al - 3) / 3] * D.bs1[3 * b + (al - 3) % 3];
      if (al >= 3) {
        double g9[9];
        ortho_grad(y + 3, kv, g9);
        acc += g9[al - 3];
      }
      gb = acc;
    }
    // body block Hb = M(1 + ρ[kin]) + ortho⁺
    double* Hb = D.Hb + ((size_t)e * D.ND + d) * 144;
    const double fac = 1.0 + (ki >= 0 ? rho : 0.0);
    for (int i = lane; i < 144; i += 32) {
      int r = i / 12, c = i % 12;
      double v = M[i] * fac;
      if (r >= 3 && c >= 3) v += S.A[12 * (r - 3) + (c - 3)];
      Hb[i] = v;
    }
    __syncwarp();
    if (lane < 12) g[3 * D.V + 12 * d + lane] = gb;      // pair terms added below
  }
  __syncthreads();
  // pair contributions to each body's gradient and diagonal block, from the per-chunk partials
  // (k_pairs_x / k_bpart_proj) summed in chunk order: the condensed pairs go into Hb (the SpMV's body
  // block), the residual pairs (applied matrix-free by the SpMV) only into the preconditioner block
  CLK(12)
  {
    const int nch = (C.n_act + 31) >> 5;
    const size_t nchunk = (size_t)(D.act_cap + 31) >> 5;
    const double* bp = D.bpart + (size_t)sl * nchunk * D.ND * BPART;
    for (int t = threadIdx.x; t < D.ND * 156; t += blockDim.x) {
      const int d = t / 156, i = t % 156;
      if (i < 144) {
        const int si = sym_idx(i / 12, i % 12, 12);
        double sc = 0.0, sr = 0.0;
#pragma unroll 4
        for (int ch = 0; ch < nch; ++ch) {
          const double* qq = bp + ((size_t)ch * D.ND + d) * BPART;
          sc += qq[12 + si];
          sr += qq[12 + PH + si];
        }
        double* Hb = D.Hb + ((size_t)e * D.ND + d) * 144;
        const double hv = Hb[i] + sc;
        Hb[i] = hv;
        D.Dg_b[((size_t)e * D.ND + d) * 144 + i] = hv + sr;
      } else {
        const int a = i - 144;
        double sg = 0.0;
#pragma unroll 4
        for (int ch = 0; ch < nch; ++ch) sg += bp[((size_t)ch * D.ND + d) * BPART + a];
        g[3 * D.V + 12 * d + a] += sg;
      }
    }
  }
  __syncthreads();
  for (int d = w; d < D.ND; d += nw) {
    double* T = JS[w].A;
    const double* Db = D.Dg_b + ((size_t)e * D.ND + d) * 144;
    const double* Mb = D.My + (size_t)D.dof_body[d] * 144;
    for (int i = lane; i < 144; i += 32) T[i] = Db[i] + C.mu * Mb[i];
    __syncwarp();
    chol_inverse12_warp(T, D.Pinv_b + ((size_t)e * D.ND + d) * 144, JS[w].Q, lane);
    __syncwarp();
  }
  CLK(13)
  if (threadIdx.x == 0) CLKN(14)
}

// ------------------------------------------------------------------------------------------
// SpMV y = H x with the contact terms condensed at assembly (k_assemble): soft BSR (elastic +
// soft–soft contact blocks) + 3×3 diagonals, body 12×12 (incl. same-body pair terms), 3×12
// soft–body coupling blocks, and the few residual pairs matrix-free through J_v (deterministic)
// ------------------------------------------------------------------------------------------
// Pass A1: residual pairs (one per lane): out = H_k x_local; soft-slot outputs go to their
// vertex-sorted position sout[spos]; DoF-body slots are pulled back through J_vᵀ and warp-reduced
// in a fixed order into per-warp partials part[w][d][12].  Pass A2: couplings (one per lane):
// C_vd x_d → cpl_out[c], C_vdᵀ x_v → part.  Pass B: soft rows (BSR + diagonal + contiguous sout
// and cpl_out ranges) and body rows (Hb x_b + Σ_w part[w][d]).  Deterministic for a fixed blockDim.
// env-resident copy of the condensed soft matrix in shared memory (k_pcg_r): upper edge blocks U
// (one per soft edge; the lower block is its transpose), SoA diagonal blocks, body blocks, the
// block-Jacobi inverses and the row/contribution index arrays
struct SmemMat {
  int lpr;                                        // soft-row lanes per row in the SpMV
  const double *U, *Hd, *Hb, *Ps, *Pb;
  double* cout;                                   // [3·ncpl] coupling outputs C_vd x_d (pass A2 → B)
  const int *rptr, *rcol, *rupx, *cptr, *rcnt, *cpp;
};

// SpMV pass A1 (residual pairs, matrix-free 12×12, one pair per lane), out of line: rare (two soft bodies or two
// DoF bodies in one pair) and register-heavy, so the PCG loop does not carry its registers
__device__ __forceinline__ void spmv_residual_inl(const Dev& D, int e, const double* x, double* part, const double* aH,
                                                 const int* aslot, const double* axb, const int* spos, double* sout,
                                                 const int* rl, int nres, int nb12, int lane, int w) {
  // pass A1: residual pairs, matrix-free 12×12 (one pair per lane)
  for (int base = 32 * w; base < nres; base += blockDim.x) {
    const int idx = base + lane;
    double out[12];
    int bd[4] = {-1, -1, -1, -1};
    v3 xbs[4];
    if (idx < nres) {
      const int k = rl[idx];
      double xl[12];
      const int4 code4 = reinterpret_cast<const int4*>(aslot)[k];
      const int codes[4] = {code4.x, code4.y, code4.z, code4.w};
      for (int s = 0; s < 4; ++s) {
        const int cd = codes[s];
        v3 u = mk(0, 0, 0);
        if (cd >= 0) u = ld3(x + 3 * cd);
        else if (cd != INT_MIN) {
          const int sl = -1 - cd;
          xbs[s] = ld3(axb + 12 * k + 3 * s);
          u = embed(x + 3 * D.V + 12 * sl, xbs[s]);
          bd[s] = sl;
        }
        xl[3 * s] = u.x; xl[3 * s + 1] = u.y; xl[3 * s + 2] = u.z;
      }
      const double* H = aH + (size_t)idx * PH;          // packed upper 12×12 (AoS), by residual index
#pragma unroll
      for (int r = 0; r < 12; ++r) out[r] = 0.0;
#pragma unroll
      for (int r = 0; r < 12; ++r)
#pragma unroll
        for (int c = r; c < 12; ++c) {
          const double h = H[sym_idx(r, c, 12)];
          out[r] += h * xl[c];
          if (c != r) out[c] += h * xl[r];
        }
      for (int s = 0; s < 4; ++s) {
        const int j = spos[4 * k + s];
        if (j >= 0) { double* o = sout + 3 * j; o[0] = out[3 * s]; o[1] = out[3 * s + 1]; o[2] = out[3 * s + 2]; }
      }
    } else {
      for (int r = 0; r < 12; ++r) out[r] = 0.0;
    }
    const bool touches = bd[0] >= 0 || bd[1] >= 0 || bd[2] >= 0 || bd[3] >= 0;
    if (__ballot_sync(0xffffffffu, touches) == 0u) continue;
    for (int d = 0; d < D.ND; ++d) {
      const bool mine = bd[0] == d || bd[1] == d || bd[2] == d || bd[3] == d;
      if (__ballot_sync(0xffffffffu, mine) == 0u) continue;
      double c[12];
#pragma unroll
      for (int i = 0; i < 12; ++i) c[i] = 0.0;
      if (mine)
        for (int s = 0; s < 4; ++s) {
          if (bd[s] != d) continue;
          for (int i = 0; i < 3; ++i) {
            const double oi = out[3 * s + i];
            c[i] += oi;
            c[3 + 3 * i] += oi * xbs[s].x; c[4 + 3 * i] += oi * xbs[s].y; c[5 + 3 * i] += oi * xbs[s].z;
          }
        }
#pragma unroll
      for (int i = 0; i < 12; ++i) c[i] = warp_sum(c[i]);
      if (lane == 0)
        for (int i = 0; i < 12; ++i) part[w * nb12 + 12 * d + i] += c[i];
    }
  }
}

__device__ __noinline__ void spmv_residual(const Dev& D, int e, const double* x, double* part, const double* aH, const int* aslot,
                                          const double* axb, const int* spos, double* sout, const int* rl, int nres, int nb12,
                                          int lane, int w) {
  spmv_residual_inl(D, e, x, part, aH, aslot, axb, spos, sout, rl, nres, nb12, lane, w);
}

// what: 1 = zero the body partials + barrier, 2 = pass A (+ barrier), 4 = pass B, 8 = final barrier.
// Returns this thread's partial Σ x_i y_i over the rows it wrote (for fused PCG dot products).
constexpr int SPMV_ALL = 15;
__device__ double spmv(const Dev& D, int e, const double* x, double* y, double* part /*smem [nw][ND][12]*/,
                       double mu = 0.0, const SmemMat* R = nullptr, int what = SPMV_ALL, int stream_lpr = 4, bool ell = false) {
  const EnvCtl& C = D.ctl[e];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const double* aH = D.act_H + (size_t)e * D.res_cap * PH;
  const int* aslot = D.act_slot + (size_t)e * 4 * D.act_cap;
  const double* axb = D.act_xb + (size_t)e * 12 * D.act_cap;
  const int* spos = D.spos + (size_t)e * 4 * D.act_cap;
  double* sout = D.sout + (size_t)e * 4 * D.act_cap * 3;
  const int* rl = D.res_list + (size_t)e * D.act_cap;
  const int nres = C.n_res, ncpl = C.n_cpl;
  const int nb12 = D.ND * 12;
  CLK_INIT
  double xy = 0.0;
  if (what & 1) {
    for (int i = threadIdx.x; i < nw * nb12; i += blockDim.x) part[i] = 0.0;
    __syncthreads();
  }
  CLK(0)
  if (what & 2) {
  if (nres > 0) {                      // the streamed kernel calls it out of line (registers); the resident inline
    if (R) spmv_residual_inl(D, e, x, part, aH, aslot, axb, spos, sout, rl, nres, nb12, lane, w);
    else spmv_residual(D, e, x, part, aH, aslot, axb, spos, sout, rl, nres, nb12, lane, w);
  }
  // pass A2: soft–body couplings (one per lane): soft output C_vd x_d → cpl_out[c] (summed by row v
  // in pass B), body output C_vdᵀ x_v warp-reduced per body into part[w][d]
  {
    const int* cplv = D.cpl_v + (size_t)e * D.cpl_cap;
    const int* cpld = D.cpl_d + (size_t)e * D.cpl_cap;
    const double* cval = D.cpl_val + (size_t)e * 36 * D.cpl_cap;
    double* cout = R ? R->cout : D.cpl_out + (size_t)e * 3 * D.cpl_cap;
    const size_t ccap = D.cpl_cap;
    for (int base = 32 * w; base < ncpl; base += blockDim.x) {
      const int c = base + lane;
      double ob[12];
#pragma unroll
      for (int i = 0; i < 12; ++i) ob[i] = 0.0;
      int bd = -1;
      if (c < ncpl) {
        const int v = cplv[c];
        bd = cpld[c];
        const v3 xv = ld3(x + 3 * v);
        const double* xb = x + 3 * D.V + 12 * bd;
        double so[3] = {0.0, 0.0, 0.0};
#pragma unroll
        for (int b = 0; b < 12; ++b) {
          const double xbb = xb[b];
          const double* cv = cval + (size_t)b * ccap + c;     // coupling blocks: streamed like the soft blocks
          const double c0 = R ? cv[0] : __ldcs(cv), c1 = R ? cv[12 * ccap] : __ldcs(cv + 12 * ccap),
                       c2 = R ? cv[24 * ccap] : __ldcs(cv + 24 * ccap);
          so[0] += c0 * xbb; so[1] += c1 * xbb; so[2] += c2 * xbb;
          ob[b] = c0 * xv.x + c1 * xv.y + c2 * xv.z;
        }
        cout[3 * c] = so[0]; cout[3 * c + 1] = so[1]; cout[3 * c + 2] = so[2];
      }
      if (__ballot_sync(0xffffffffu, bd >= 0) == 0u) continue;
      for (int d = 0; d < D.ND; ++d) {
        const bool mine = bd == d;
        if (__ballot_sync(0xffffffffu, mine) == 0u) continue;
#pragma unroll
        for (int i = 0; i < 12; ++i) {
          const double t = warp_sum(mine ? ob[i] : 0.0);
          if (lane == 0) part[w * nb12 + 12 * d + i] += t;
        }
      }
    }
  }
  CLK(1)
  __syncthreads();
  }
  CLK(2)
  if (!(what & 4)) return 0.0;
  const int* cptr = R ? R->cptr : D.cptr + (size_t)e * (D.V + 1);
  const int* rcnt = R ? R->rcnt : D.rcnt + (size_t)e * D.V;
  const int* cpp = R ? R->cpp : D.cpl_ptr + (size_t)e * (D.V + 1);
  const double* cout = R ? R->cout : D.cpl_out + (size_t)e * 3 * D.cpl_cap;
  const double* Hd = R ? R->Hd : D.Hd + (size_t)e * D.V * 9;       // SoA [9][V]
  const double* Ho = D.Ho + (size_t)e * D.NNZ * 9;
  const int* rptr = R ? R->rptr : D.rptr;
  // soft rows, streamed operator in sliced-ELL layout (written by the assembly, or converted once per k_pcg
  // launch): slot s of the sorted row order, warp = 32 consecutive slots, every block component load is 256
  // contiguous bytes
  if (ell && !R) {
    const double* He = D.Hell + (size_t)e * D.ell_total;
    const int nslot = 32 * D.ell_groups;
    for (int s0 = 0; s0 < nslot; s0 += blockDim.x) {
      const int slot = s0 + threadIdx.x;
      const int v = slot < nslot ? D.ell_row[slot] : -1;
      if (v < 0) continue;
      const int g = slot >> 5, l = slot & 31, len = D.ell_len[g];
      const double* hb = He + D.ell_vb[g] + l;
      const int* cb = D.ell_col + D.ell_cb[g] + l;
      v3 acc = mk(0, 0, 0);
      // the operator is read once per iteration: streaming loads (evict-first), so the per-env vectors, which
      // every iteration re-reads, keep their L2 lines
#pragma unroll 4
      for (int j = 0; j < len; ++j) {
        const v3 xu = ld3(x + 3 * cb[32 * j]);
        const double* B = hb + 288 * j;
        acc += mk(__ldcs(B) * xu.x + __ldcs(B + 32) * xu.y + __ldcs(B + 64) * xu.z,
                  __ldcs(B + 96) * xu.x + __ldcs(B + 128) * xu.y + __ldcs(B + 160) * xu.z,
                  __ldcs(B + 192) * xu.x + __ldcs(B + 224) * xu.y + __ldcs(B + 256) * xu.z);
      }
      const v3 xv = ld3(x + 3 * v);
      const size_t V = D.V;
      acc += mk(__ldcs(Hd + v) * xv.x + __ldcs(Hd + V + v) * xv.y + __ldcs(Hd + 2 * V + v) * xv.z,
                __ldcs(Hd + 3 * V + v) * xv.x + __ldcs(Hd + 4 * V + v) * xv.y + __ldcs(Hd + 5 * V + v) * xv.z,
                __ldcs(Hd + 6 * V + v) * xv.x + __ldcs(Hd + 7 * V + v) * xv.y + __ldcs(Hd + 8 * V + v) * xv.z);
      for (int j = cptr[v], j1r = cptr[v] + rcnt[v]; j < j1r; ++j) acc += ld3(sout + 3 * j);
      for (int j = cpp[v]; j < cpp[v + 1]; ++j) acc += ld3(cout + 3 * j);
      if (mu != 0.0) acc += (mu * D.mass[v]) * xv;
      st3(y + 3 * v, acc);
      xy += xv.x * acc.x + xv.y * acc.y + xv.z * acc.z;
    }
  } else
  // soft rows: lpr lanes per row (streamed operator: 4; resident: 1, measured best); lane q of the
  // group takes blocks j = rptr[v]+q, +lpr, ... (adjacent lanes read adjacent 72-byte blocks), then a
  // shuffle reduction; lane q==0 adds the diagonal block and the contiguous pair outputs and stores
  {
    const int lpr = R ? R->lpr : stream_lpr;          // lanes per row (1, 2 or 4)
    const int q = lane & (lpr - 1);
    const int rows_per_pass = blockDim.x / lpr;
    for (int v0 = 0; v0 < D.V; v0 += rows_per_pass) {
      const int v = v0 + threadIdx.x / lpr;
      const bool live = v < D.V;
      v3 acc = mk(0, 0, 0);
      if (live) {
        const int j1 = rptr[v + 1];
        if (R) {
#pragma unroll 4
          for (int j = rptr[v] + q; j < j1; j += lpr) {
            const int ux = R->rupx[j];
            const double* Bk = R->U + 9 * (ux >> 1);
            const v3 xu = ld3(x + 3 * R->rcol[j]);
            acc += (ux & 1) ? mul33T(Bk, xu) : mul33(Bk, xu);
          }
        } else {
#pragma unroll 4
          for (int j = rptr[v] + q; j < j1; j += lpr) acc += mul33(Ho + 9 * j, ld3(x + 3 * D.rcol[j]));
        }
      }
      for (int o = 1; o < lpr; o <<= 1) {
        acc.x += __shfl_xor_sync(0xffffffffu, acc.x, o);
        acc.y += __shfl_xor_sync(0xffffffffu, acc.y, o);
        acc.z += __shfl_xor_sync(0xffffffffu, acc.z, o);
      }
      if (live && q == 0) {
        const v3 xv = ld3(x + 3 * v);
        const size_t V = D.V;
        acc += mk(Hd[v] * xv.x + Hd[V + v] * xv.y + Hd[2 * V + v] * xv.z,
                  Hd[3 * V + v] * xv.x + Hd[4 * V + v] * xv.y + Hd[5 * V + v] * xv.z,
                  Hd[6 * V + v] * xv.x + Hd[7 * V + v] * xv.y + Hd[8 * V + v] * xv.z);
        for (int j = cptr[v], j1r = cptr[v] + rcnt[v]; j < j1r; ++j) acc += ld3(sout + 3 * j);
        for (int j = cpp[v]; j < cpp[v + 1]; ++j) acc += ld3(cout + 3 * j);
        if (mu != 0.0) acc += (mu * D.mass[v]) * xv;
        st3(y + 3 * v, acc);
        xy += xv.x * acc.x + xv.y * acc.y + xv.z * acc.z;
      }
    }
  }
  CLK(3)
  // body rows: taken by the highest thread indices (idle in the soft-row pass when V < blockDim)
  for (int i = blockDim.x - 1 - threadIdx.x; i < nb12; i += blockDim.x) {
    const int d = i / 12, row = i % 12;
    const double* Hb = (R ? R->Hb + (size_t)d * 144 : D.Hb + ((size_t)e * D.ND + d) * 144) + 12 * row;
    const double* xb = x + 3 * D.V + 12 * d;
    double sacc = 0.0;
    for (int c = 0; c < 12; ++c) sacc += Hb[c] * xb[c];
    if (mu != 0.0) {
      const double* Mr = D.My + (size_t)D.dof_body[d] * 144 + 12 * row;
      for (int c = 0; c < 12; ++c) sacc += mu * Mr[c] * xb[c];
    }
    for (int ww = 0; ww < nw; ++ww) sacc += part[ww * nb12 + i];
    y[3 * D.V + i] = sacc;
    xy += xb[row] * sacc;
  }
  if (what & 8) __syncthreads();
  CLK(4)
  return xy;
}

// block-Jacobi inverses of (diag blocks + μM) — LM retry inside k_pcg (R14c).  The 3×3 soft
// blocks are thread-parallel; warp 0 inverts the body blocks one by one (warp Cholesky) meanwhile.
// Outputs: ps [9][V] SoA and pb [ND][144] (global, or the resident shared-memory copies)
__device__ __forceinline__ void reinvert_precond_inl(const Dev& D, int e, double mu, double* ps, double* pb, double* scratch /*smem 144*/,
                                 double* T /*smem 144*/) {
  const double* ds = D.Dg_s + (size_t)e * D.V * 9;
  for (int v = threadIdx.x; v < D.V; v += blockDim.x) {
    double Pv[9], Pi[9];
    for (int i = 0; i < 9; ++i) Pv[i] = ds[(size_t)i * D.V + v];
    const double sh = mu * D.mass[v];
    Pv[0] += sh; Pv[4] += sh; Pv[8] += sh;
    inv33(Pv, Pi);
    for (int i = 0; i < 9; ++i) ps[(size_t)i * D.V + v] = Pi[i];
  }
  if (threadIdx.x < 32) {
    const int lane = threadIdx.x;
    for (int d = 0; d < D.ND; ++d) {
      const double* Db = D.Dg_b + ((size_t)e * D.ND + d) * 144;
      const double* Mb = D.My + (size_t)D.dof_body[d] * 144;
      for (int i = lane; i < 144; i += 32) T[i] = Db[i] + mu * Mb[i];
      __syncwarp();
      chol_inverse12_warp(T, pb + (size_t)d * 144, scratch, lane);
      __syncwarp();
    }
  }
  __syncthreads();
}
__device__ __noinline__ void reinvert_precond(const Dev& D, int e, double mu, double* ps, double* pb, double* scratch,
                                             double* T) {
  reinvert_precond_inl(D, e, mu, ps, pb, scratch, T);
}

__device__ void precond(const Dev& D, int e, const double* r, double* z, const SmemMat* R = nullptr) {
  const double* Ps = R ? R->Ps : D.Pinv_s + (size_t)e * D.V * 9;    // SoA [9][V]
  const size_t V = D.V;
  for (int v = threadIdx.x; v < D.V; v += blockDim.x) {
    const v3 rv = ld3(r + 3 * v);
    st3(z + 3 * v, mk(Ps[v] * rv.x + Ps[V + v] * rv.y + Ps[2 * V + v] * rv.z,
                      Ps[3 * V + v] * rv.x + Ps[4 * V + v] * rv.y + Ps[5 * V + v] * rv.z,
                      Ps[6 * V + v] * rv.x + Ps[7 * V + v] * rv.y + Ps[8 * V + v] * rv.z));
  }
  for (int i = threadIdx.x; i < 12 * D.ND; i += blockDim.x) {
    int d = i / 12, row = i % 12;
    const double* Pi = (R ? R->Pb + (size_t)d * 144 : D.Pinv_b + ((size_t)e * D.ND + d) * 144) + 12 * row;
    const double* rb = r + 3 * D.V + 12 * d;
    double s = 0.0;
    for (int c = 0; c < 12; ++c) s += Pi[c] * rb[c];
    z[3 * D.V + 12 * d + row] = s;
  }
  __syncthreads();
}

// ------------------------------------------------------------------------------------------
// block-Jacobi PCG: H p = −g from p₀ = 0, stop at rᵀz ≤ η² r₀ᵀz₀ or max_pcg; then the
// Newton convergence test ‖p‖_emb,∞ ≤ τ_N L_env and gᵀp.
// ------------------------------------------------------------------------------------------
__device__ void pcg_finish(const Dev& D, int e, double* p, double* red, double mu, bool bad, bool zero_g, int it_total,
                           double gp);
// PCG tolerance of this solve (reading R24): fixed η, or the Eisenstat–Walker forcing from the
// env's last accepted solve of the step: η = 0.9·r₀ᵀz₀ / (r₀ᵀz₀)_prev, ≥ 0.9·η_prev² when that exceeds 0.1,
// clamped to [η, η_max]; η_max for the first solve of a step.  Uniform across the block (rz0 is).
__device__ __forceinline__ double pcg_forcing(const Dev& D, const EnvCtl& C, double rz0) {
  if (!(D.eta_max > 0.0)) return D.eta;
  if (!C.ew_has) return D.eta_max;
  double eta = 0.9 * rz0 / C.ew_rz0;
  const double sg = 0.9 * C.ew_eta * C.ew_eta;
  if (sg > 0.1) eta = fmax(eta, sg);
  return fmin(fmax(eta, D.eta), D.eta_max);
}
// vsm = 1: the five PCG vectors live in shared memory (n small enough), p is copied out at the end
__device__ __noinline__ void pcg_finish_noinline(const Dev& D, int e, double* p, double* red, double mu, bool bad, bool zero_g,
                                                 int it_total, double gp);
__device__ void pcg_body(const Dev& D, int e, int vsm, double* dsmem, double* red, SmemMat* R, double* Rw_Ps, double* Rw_Pb,
                         int fused = 0, int stream_lpr = 4);

// 2 CTAs/SM (128 registers); a 3-CTA/SM budget (80 registers) was measured slower (C3 PCG 6.7 -> 9.1 s / 10
// steps: spills in the SpMV loop)
template <int MINB>
__global__ void __launch_bounds__(NTHREADS, MINB) k_pcg(Dev D, int env0, int force, int vsm, int fused, int lpr) {
  const int e = env_at(D, env0, blockIdx.x);
  if (env_skip(D, e, force)) return;
  __shared__ double red[32];
  extern __shared__ double dsmem[];     // [nw][ND][12] body partials, then (vsm) p, r, z, d, Ad
  pcg_body(D, e, vsm, dsmem, red, nullptr, nullptr, nullptr, fused, lpr);
}

// shared-memory bytes of k_pcg_r for this batch (0 if the env does not fit one CTA)
// env-resident PCG: one CTA (512 threads) per env with the condensed soft matrix, diagonal and body
// blocks, preconditioner and index arrays staged once into shared memory; only the (few) residual
// pairs and the soft–body couplings are read from global memory per iteration
__device__ __forceinline__ void pcg_r_body(const Dev& D, int env0, int force, int lpr) {
  const int e = env_at(D, env0, blockIdx.x);
  if (env_skip(D, e, force)) return;
  __shared__ double red[32];
  extern __shared__ double dsmem[];
  const int V = D.V, ND = D.ND, n = D.n, NNZ = D.NNZ;
  double* base = dsmem + ((blockDim.x / 32) * ND * 12 + 1) + 5 * (size_t)n;   // after bpart + vectors
  double* U = base;
  double* Hd = U + 9 * (size_t)D.NEs;
  double* Ps = Hd + 9 * (size_t)V;
  double* Pb = Ps + 9 * (size_t)V;
  double* Hb = Pb + 144 * (size_t)ND;
  double* couts = Hb + 144 * (size_t)ND;
  int* rptr = reinterpret_cast<int*>(couts + 3 * pcg_r_ncpl(D));
  int* cptr = rptr + V + 1;
  int* cpp = cptr + V + 1;
  int* rcnt = cpp + V + 1;
  int* rcol = rcnt + V;
  int* rupx = rcol + NNZ;
  const double* Ho = D.Ho + (size_t)e * NNZ * 9;
  for (int j = threadIdx.x; j < NNZ; j += blockDim.x) { rcol[j] = D.rcol[j]; rupx[j] = D.rupx[j]; }
  for (int v = threadIdx.x; v <= V; v += blockDim.x) {
    rptr[v] = D.rptr[v];
    cptr[v] = D.cptr[(size_t)e * (V + 1) + v];
    cpp[v] = D.cpl_ptr[(size_t)e * (V + 1) + v];
    if (v < V) rcnt[v] = D.rcnt[(size_t)e * V + v];
  }
  for (int i = threadIdx.x; i < 9 * V; i += blockDim.x) {
    Hd[i] = D.Hd[(size_t)e * V * 9 + i];
    Ps[i] = D.Pinv_s[(size_t)e * V * 9 + i];
  }
  for (int i = threadIdx.x; i < 144 * ND; i += blockDim.x) {
    Pb[i] = D.Pinv_b[(size_t)e * ND * 144 + i];
    Hb[i] = D.Hb[(size_t)e * ND * 144 + i];
  }
  __syncthreads();
  for (int i = threadIdx.x; i < 9 * D.NEs; i += blockDim.x)    // upper edge blocks (72-byte runs of Ho)
    U[i] = Ho[9 * (size_t)D.eup[i / 9] + i % 9];
  __syncthreads();
  SmemMat R{lpr, U, Hd, Hb, Ps, Pb, couts, rptr, rcol, rupx, cptr, rcnt, cpp};
  pcg_body(D, e, 1, dsmem, red, &R, Ps, Pb);
}
// the env-resident PCG at two register budgets: ≤ 384 threads (C2: 168 registers per thread, 256 B of
// spills) and ≤ 512 threads (128 registers)
__global__ void __launch_bounds__(384, 1) k_pcg_r(Dev D, int env0, int force, int lpr) { pcg_r_body(D, env0, force, lpr); }
__global__ void __launch_bounds__(PCG_R_THREADS, 1) k_pcg_r512(Dev D, int env0, int force, int lpr) {
  pcg_r_body(D, env0, force, lpr);
}

__device__ void pcg_body(const Dev& D, int e, int vsm, double* dsmem, double* red, SmemMat* R, double* Rw_Ps, double* Rw_Pb,
                         int fused, int stream_lpr) {
  double* bpart = dsmem;
  EnvCtl& C = D.ctl[e];
  const int n = D.n;
  const double* g = D.g + (size_t)e * n;
  double* const p_out = D.p + (size_t)e * n;
  double *p, *r, *z, *d, *Ad;
  if (vsm == 1) {
    double* base = dsmem + ((blockDim.x / 32) * D.ND * 12 + 1);
    p = base; r = base + n; z = base + 2 * n; d = base + 3 * n; Ad = base + 4 * n;
  } else {
    p = p_out; r = D.r + (size_t)e * n; z = D.z + (size_t)e * n; d = D.dd + (size_t)e * n; Ad = D.Ad + (size_t)e * n;
    if (vsm == 2) d = dsmem + ((blockDim.x / 32) * D.ND * 12 + 1);   // the SpMV's gathered vector on chip
  }
  // hessian_mode 2 (reading R14c): solve (H + μM) p = −g; on negative curvature or a non-descent
  // direction raise μ ← max(μ₀, 10μ), re-invert the block-Jacobi blocks and restart (same launch)
  double mu = C.mu;
  bool bad = false;
  int it_total = 0;
  double gp = 0.0;
  bool zero_g = false;
  double rz0_used = 0.0, eta_used = 0.0;
  __shared__ double chol_scratch[144], chol_T[144];
  // streamed operator: the soft blocks of this env in sliced-ELL layout, once per launch
  const bool ell = !R && D.ell_groups > 0;
  if (ell && !D.asm_ell) {                    // row-ordered blocks → sliced ELL (when the assembly did not)
    double* He = D.Hell + (size_t)e * D.ell_total;
    const double* Ho = D.Ho + (size_t)e * D.NNZ * 9;
    for (int q = threadIdx.x; q < D.NNZ; q += blockDim.x) {
      const long long b = D.ell_pos[q];
#pragma unroll
      for (int c = 0; c < 9; ++c) He[b + 32 * c] = Ho[9 * (size_t)q + c];
    }
    __syncthreads();
  }
  for (int attempt = 0;; ++attempt) {
    if (attempt > 0) {
      if (R) reinvert_precond_inl(D, e, mu, Rw_Ps, Rw_Pb, chol_scratch, chol_T);  // resident copies (inline)
      else reinvert_precond(D, e, mu, D.Pinv_s + (size_t)e * D.V * 9, D.Pinv_b + (size_t)e * D.ND * 144, chol_scratch, chol_T);
    }
    for (int i = threadIdx.x; i < n; i += blockDim.x) { p[i] = 0.0; r[i] = -g[i]; }
    __syncthreads();
    precond(D, e, r, z, R);
    double part = 0.0;
    for (int i = threadIdx.x; i < n; i += blockDim.x) { d[i] = z[i]; part += r[i] * z[i]; }
    double rz = block_sum(part, red);
    const double rz0 = rz, eta_k = pcg_forcing(D, C, rz0), stop = eta_k * eta_k * rz0;
    rz0_used = rz0; eta_used = eta_k;
    zero_g = rz0 == 0.0;                                 // g = 0: p = 0 is the (converged) answer
    int it = 0;
    bad = !(rz0 == rz0);
    if (R || fused) {
      // fused iteration (resident or streamed operator), 4 barriers: [pass A | B2 | pass B + dᵀAd partials | B3 | α, p/r update,
      // block-Jacobi z and rᵀz partials per vertex / body | B4 | β, d update | B1].  Per-warp partials in
      // red[0..15] (dᵀAd) and red[16..31] (rᵀz), summed in warp order by every thread (deterministic)
      const int lane = threadIdx.x & 31, wi = threadIdx.x >> 5, nwp = blockDim.x >> 5;
      const int V = D.V, nb12 = 12 * D.ND;
      for (int i = threadIdx.x; i < nwp * nb12; i += blockDim.x) bpart[i] = 0.0;
      __syncthreads();
      while (!bad && it < D.max_pcg && rz > stop) {
        CLK_INIT
        double loc = spmv(D, e, d, Ad, bpart, mu, R, 2 | 4, stream_lpr, ell);
        loc = warp_sum(loc);
        if (lane == 0) red[wi] = loc;
        CLK(5)
        __syncthreads();                                  // B3
        CLK(6)
        double dAd = 0.0;
        for (int k = 0; k < nwp; ++k) dAd += red[k];
        if (!(dAd > 0.0)) { bad = true; __syncthreads(); break; }   // uniform; red[] reads done
        const double alpha = rz / dAd;
        double loc2 = 0.0;
        // two vertices per thread and pass, every load issued before the stores (r, p, z may alias the loaded
        // arrays as far as the compiler knows, so it would not hoist the next vertex's loads itself)
        const double* Ps = R ? R->Ps : D.Pinv_s + (size_t)e * V * 9;
        for (int v0 = threadIdx.x; v0 < V; v0 += 2 * blockDim.x) {
          const int v1 = v0 + blockDim.x;
          const bool h1 = v1 < V;
          v3 rr[2], aa[2], dd[2], pp[2];
          double P[2][9];
#pragma unroll
          for (int k = 0; k < 2; ++k) {
            const int v = k ? (h1 ? v1 : v0) : v0;
            rr[k] = ld3(r + 3 * v); aa[k] = ld3(Ad + 3 * v); dd[k] = ld3(d + 3 * v); pp[k] = ld3(p + 3 * v);
#pragma unroll
            for (int i = 0; i < 9; ++i) P[k][i] = R ? Ps[(size_t)i * V + v] : __ldcs(Ps + (size_t)i * V + v);
          }
#pragma unroll
          for (int k = 0; k < 2; ++k) {
            if (k == 1 && !h1) break;
            const int v = k ? v1 : v0;
            const v3 rv = mk(rr[k].x - alpha * aa[k].x, rr[k].y - alpha * aa[k].y, rr[k].z - alpha * aa[k].z);
            st3(p + 3 * v, mk(pp[k].x + alpha * dd[k].x, pp[k].y + alpha * dd[k].y, pp[k].z + alpha * dd[k].z));
            st3(r + 3 * v, rv);
            const double* Q = P[k];
            const v3 zv = mk(Q[0] * rv.x + Q[1] * rv.y + Q[2] * rv.z, Q[3] * rv.x + Q[4] * rv.y + Q[5] * rv.z,
                             Q[6] * rv.x + Q[7] * rv.y + Q[8] * rv.z);
            st3(z + 3 * v, zv);
            loc2 += rv.x * zv.x + rv.y * zv.y + rv.z * zv.z;
          }
        }
        for (int db = nwp - 1 - wi; db >= 0 && db < D.ND; db += nwp) {   // body db (last warps): lanes 0..11 own its rows
          const int o = 3 * V + 12 * db;
          if (lane < 12) {
            p[o + lane] += alpha * d[o + lane];
            r[o + lane] -= alpha * Ad[o + lane];
          }
          __syncwarp();
          if (lane < 12) {
            const double* Pi = (R ? R->Pb : D.Pinv_b + (size_t)e * D.ND * 144) + (size_t)db * 144 + 12 * lane;
            double zz = 0.0;
            for (int c = 0; c < 12; ++c) zz += Pi[c] * r[o + c];
            z[o + lane] = zz;
            loc2 += r[o + lane] * zz;
          }
          __syncwarp();
        }
        for (int i = threadIdx.x; i < nwp * nb12; i += blockDim.x) bpart[i] = 0.0;   // read before B3
        loc2 = warp_sum(loc2);
        if (lane == 0) red[16 + wi] = loc2;
        CLK(7)
        __syncthreads();                                  // B4
        CLK(8)
        double rzn = 0.0;
        for (int k = 0; k < nwp; ++k) rzn += red[16 + k];
        const double beta = rzn / rz;
        for (int i = threadIdx.x; i < n; i += blockDim.x) d[i] = z[i] + beta * d[i];
        __syncthreads();                                  // B1
        CLK(9)
        if (threadIdx.x == 0) CLK_COUNT
        rz = rzn;
        ++it;
        if (!(rz == rz)) bad = true;
      }
    }
    while (!R && !fused && !bad && it < D.max_pcg && rz > stop) {
      spmv(D, e, d, Ad, bpart, mu, R, SPMV_ALL, 4, ell);
      CLK_INIT
      part = 0.0;
      for (int i = threadIdx.x; i < n; i += blockDim.x) part += d[i] * Ad[i];
      double dAd = block_sum(part, red);
      CLK(5)
      if (!(dAd > 0.0)) { bad = true; break; }          // not SPD along d (uniform across the block)
      double alpha = rz / dAd;
      for (int i = threadIdx.x; i < n; i += blockDim.x) { p[i] += alpha * d[i]; r[i] -= alpha * Ad[i]; }
      __syncthreads();
      CLK(6)
      precond(D, e, r, z, R);
      CLK(7)
      part = 0.0;
      for (int i = threadIdx.x; i < n; i += blockDim.x) part += r[i] * z[i];
      double rzn = block_sum(part, red);
      CLK(8)
      double beta = rzn / rz;
      for (int i = threadIdx.x; i < n; i += blockDim.x) d[i] = z[i] + beta * d[i];
      __syncthreads();
      CLK(9)
      if (threadIdx.x == 0) CLK_COUNT
      rz = rzn;
      ++it;
      if (!(rz == rz)) bad = true;
    }
    it_total += it;
    part = 0.0;
    for (int i = threadIdx.x; i < n; i += blockDim.x) part += g[i] * p[i];
    gp = block_sum(part, red);
    if (D.hmode != 2 || (!bad && (gp < 0.0 || zero_g)) || mu > 1e12) break;
    mu = fmax(D.lm_mu0, 10.0 * mu);
  }
  if (vsm == 1) {
    for (int i = threadIdx.x; i < n; i += blockDim.x) p_out[i] = p[i];
    __syncthreads();
    p = p_out;
  }
  if (threadIdx.x == 0 && !bad && rz0_used > 0.0) { C.ew_rz0 = rz0_used; C.ew_eta = eta_used; C.ew_has = 1; }
  if (R) pcg_finish(D, e, p, red, mu, bad, zero_g, it_total, gp);
  else pcg_finish_noinline(D, e, p, red, mu, bad, zero_g, it_total, gp);   // streamed: out of line (registers)
}

// end of a PCG launch (block-level, one CTA per env): embedded ∞-norm of the direction, step cap
// (R17c), Newton convergence test (R14) and the per-env statistics
__device__ void pcg_finish(const Dev& D, int e, double* p, double* red, double mu, bool bad, bool zero_g, int it_total,
                           double gp) {
  EnvCtl& C = D.ctl[e];
  const int n = D.n;
  // reading R14d: under an LM shift (μ > 0) the step no longer measures convergence; the env is
  // converged when the mass-scaled gradient step M⁻¹g is below τ_N·L_env (embedded ∞-norm)
  const double mu_used = D.hmode == 2 ? mu : 0.0;
  double gm = 1.0 / 0.0;
  if (mu_used > 0.0 && !bad) {
    const double* g = D.g + (size_t)e * n;
    double* mg = D.Ad + (size_t)e * n;                  // PCG scratch, free after the solve
    for (int i = threadIdx.x; i < 3 * D.V; i += blockDim.x) mg[i] = g[i] / D.mass[i / 3];
    for (int i = threadIdx.x; i < 12 * D.ND; i += blockDim.x) {
      const int d = i / 12, row = i % 12;
      const double* Mi = D.MyInv + (size_t)D.dof_body[d] * 144 + 12 * row;
      const double* gb = g + 3 * D.V + 12 * d;
      double t = 0.0;
      for (int c = 0; c < 12; ++c) t += Mi[c] * gb[c];
      mg[3 * D.V + i] = t;
    }
    __syncthreads();
    gm = embedded_inf_norm(D, e, mg, red);
    __syncthreads();
  }
  double pm = embedded_inf_norm(D, e, p, red);
  // step cap (reading R17c): scale p to max_step·L_env if longer (direction unchanged)
  const double cap = D.max_step * C.L;
  if (pm > cap && pm == pm) {
    const double sc = cap / pm;
    for (int i = threadIdx.x; i < n; i += blockDim.x) p[i] *= sc;
    __syncthreads();
    gp *= sc;
  }
  if (threadIdx.x == 0) {
    const bool exact_failed = D.hmode == 1 && C.exact && (bad || !(gp < 0.0) || !(pm == pm));
    C.pcg += it_total;
    C.pcg_total += it_total;
    // algorithmic bytes per PCG iteration of the condensed operator (SURVEY §8(d) model with the
    // contact condensation): 72(V+E_s) + 4E_s [soft BSR] + 640·P_res [residual pairs]
    // + 296·N_cpl [3×12 couplings + ids] + 624·ND [body blocks] + 48V + 624·ND [preconditioner] + 96n
    const double bpi = 72.0 * (D.V + D.NEs) + 4.0 * D.NEs + 640.0 * C.n_res + 296.0 * C.n_cpl + 1248.0 * D.ND +
                       48.0 * D.V + 96.0 * D.n;
    C.pcg_bytes += bpi * it_total;
    C.gp = gp;
    C.pnorm = pm;
    if (e == D.trace_env && D.trace) {                   // diagnostic trace (tac_debug_trace)
      const int r = *D.trace_n;
      if (r < D.trace_cap) {
        double* t = D.trace + 10 * (size_t)r;
        t[0] = C.newton; t[1] = it_total; t[2] = D.hmode == 2 ? mu : 0.0; t[3] = pm; t[4] = gm; t[5] = gp;
        t[6] = 0.0; t[7] = 0.0; t[8] = 0.0; t[9] = 0.0;
      }
    }
    if (exact_failed) {
      C.xfail = 1;                                        // retry projected next pass (not counted)
    } else {
      C.newton += 1;
      C.mu_used = mu_used;
      if (D.hmode == 2) C.mu = (mu * 0.1 >= D.lm_mu0) ? mu * 0.1 : 0.0;
      if (bad || !(pm == pm) || !(gp < 0.0 || zero_g)) { C.phase = PHASE_FAILED; C.status = ENV_NONFINITE; }
      else C.inner_conv = ((pm <= D.tolN * C.L && mu_used == 0.0) || gm <= D.tolN * C.L) ? 1 : 0;
    }
  }
}

__device__ __noinline__ void pcg_finish_noinline(const Dev& D, int e, double* p, double* red, double mu, bool bad, bool zero_g,
                                                 int it_total, double gp) {
  pcg_finish(D, e, p, red, mu, bad, zero_g, it_total, gp);
}
}  // namespace tac
#include "pcg_cluster.cuh"
namespace tac {

__global__ void __launch_bounds__(NTHREADS) k_spmv(Dev D, int env0, const double* x, double* y) {
  const int e = env_at(D, env0, blockIdx.x);
  extern __shared__ double part[];
  spmv(D, e, x, y, part, 0.0, nullptr, SPMV_ALL, 4, D.asm_ell != 0);
}

// ------------------------------------------------------------------------------------------
// additive CCD (reading R16): α_max = min(1, min over C′ of ACCD)
// ------------------------------------------------------------------------------------------
__device__ double accd_pair(int kind, v3* X, v3* Pd, double s, double tc, int max_iters) {
  v3 mean = 0.25 * (Pd[0] + Pd[1] + Pd[2] + Pd[3]);
  double n[4];
  for (int i = 0; i < 4; ++i) { Pd[i] = Pd[i] - mean; n[i] = sqrt(dot(Pd[i], Pd[i])); }
  double lp = kind == 0 ? n[0] + fmax(n[1], fmax(n[2], n[3])) : fmax(n[0], n[1]) + fmax(n[2], n[3]);
  if (lp == 0.0) return 1.0;
  // the first advance t_l = (1−s)·d/l_p already exceeds t_c when the box distance does: ACCD returns 1
  if ((1.0 - s) * prim_box_dist(kind, X) > tc * lp * (1.0 + 1e-10)) return 1.0;
  double d2;
  classify(kind, X, &d2);
  double d = sqrt(d2);
  double g = s * d, t = 0.0, tl = (1.0 - s) * d / lp;
  int it = 0;
  while (true) {
    for (int i = 0; i < 4; ++i) X[i] = X[i] + tl * Pd[i];
    classify(kind, X, &d2);
    d = sqrt(d2);
    if (t > 0.0 && d < g) break;
    t += tl;
    if (t > tc) return 1.0;
    tl = (1.0 - s) * d / lp;
    if (++it >= max_iters) break;
  }
  return t;
}

__global__ void __launch_bounds__(NTHREADS, 2) k_ccd(Dev D, int env0, int force) {
  const int e = env_at(D, env0, blockIdx.x);
  EnvCtl& C = D.ctl[e];
  if (!force && (C.phase != PHASE_ACTIVE || C.inner_conv || C.xfail)) return;
  __shared__ double red[32];
  const double* P = D.P + (size_t)e * D.NVall * 3;
  const double* Pd = D.Pd + (size_t)e * D.NVall * 3;
  const int* ca = D.cand_a + (size_t)e * D.cand_cap;
  const int* cb = D.cand_b + (size_t)e * D.cand_cap;
  double amin = 1.0;
  // candidates handed to warps 32 at a time (dynamic balance; the minimum is order-independent)
  __shared__ int next_k;
  if (threadIdx.x == 0) next_k = 0;
  __syncthreads();
  const int nck = C.ncand;
  for (;;) {
    int kb = 0;
    if ((threadIdx.x & 31) == 0) kb = atomicAdd(&next_k, 32);
    kb = __shfl_sync(0xffffffffu, kb, 0);
    if (kb >= nck) break;
    const int k = kb + (threadIdx.x & 31);
    if (k >= nck) continue;
    int kind = (ca[k] >> 30) & 1, a = ca[k] & ((1 << 30) - 1), b = cb[k], vid[4];
    pair_vids(D, kind, a, b, vid);
    v3 X[4], Q[4];
    for (int s = 0; s < 4; ++s) { X[s] = ld3(P + 3 * vid[s]); Q[s] = ld3(Pd + 3 * vid[s]); }
    amin = fmin(amin, accd_pair(kind, X, Q, D.accd_s, 1.0, D.max_accd));
  }
  amin = block_min(amin, red);
  if (threadIdx.x == 0) C.alpha_ccd = fmin(1.0, amin);
}

// ------------------------------------------------------------------------------------------
// energy at q + α p (line search): six deterministic block sums
// ------------------------------------------------------------------------------------------
// six deterministic block sums in one pass (2 barriers): per-warp partials → red6[6][32] → warp sums
constexpr int NTERMS = 7;                 // inertia, elastic, ortho, gravity, barrier, AL, friction
__device__ __forceinline__ void block_sum_terms(double* v, double* red) {   // red: [NTERMS][32]
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
#pragma unroll
  for (int i = 0; i < NTERMS; ++i) v[i] = warp_sum(v[i]);
  __syncthreads();
  if (lane == 0)
#pragma unroll
    for (int i = 0; i < NTERMS; ++i) red[32 * i + wid] = v[i];
  __syncthreads();
#pragma unroll
  for (int i = 0; i < NTERMS; ++i) v[i] = warp_sum(lane < nw ? red[32 * i + lane] : 0.0);
}

// Energy terms at q + αp.  lmode 0: barrier over every candidate of C′; 1: the same, and build the
// line-search list lsl of candidates that can be active for some α ∈ [0, K_eff·α_ccd] —
// d(0) − α_ccd·(max_A ‖Pd‖ + max_B ‖Pd‖) < d̂ (a primitive distance moves at most by the largest vertex
// displacement of each side) — in candidate order; 2: barrier over the list only (exact: the other
// candidates have d > d̂ at every trial α of this line search)
__device__ void energy_terms(const Dev& D, int e, double alpha, double* red, double* terms, int* inverted,
                             int lmode = 0, int* lsl = nullptr, int* nls = nullptr, int* sh = nullptr) {
  const EnvCtl& C = D.ctl[e];
  const double* q = D.q + (size_t)e * D.n;
  const double* p = D.p + (size_t)e * D.n;
  const double* qt = D.qt + (size_t)e * D.n;
  const double dt2 = D.dt * D.dt, rho = C.rho;
  const v3 G = mk(D.grav[0], D.grav[1], D.grav[2]);
  double ein = 0, eel = 0, eor = 0, egr = 0, eba = 0, eal = 0;
  int inv = 0;
  const double* s_att = D.s_att + (size_t)e * D.NC * 3;
  const double* lam_att = D.lam_att + (size_t)e * D.NC * 3;
  for (int v = threadIdx.x; v < D.V; v += blockDim.x) {
    double m = D.mass[v];
    v3 x = ld3(q + 3 * v) + alpha * ld3(p + 3 * v);
    v3 dx = x - ld3(qt + 3 * v);
    ein += 0.5 * m * dot(dx, dx);
    egr -= dt2 * m * dot(G, x);
    int ci = D.att_of_vert[v];
    if (ci >= 0) {
      v3 r = x - ld3(s_att + 3 * ci);
      eal += 0.5 * rho * m * dot(r, r) - m * dot(ld3(lam_att + 3 * ci), r);
    }
  }
  for (int t = threadIdx.x; t < D.T; t += blockDim.x) {
    int4 tv = reinterpret_cast<const int4*>(D.tets)[t];
    int ids[4] = {tv.x, tv.y, tv.z, tv.w};
    v3 x[4];
    for (int i = 0; i < 4; ++i) x[i] = ld3(q + 3 * ids[i]) + alpha * ld3(p + 3 * ids[i]);
    bool bad = false;
    double psi = nh_energy(x, D.Dmi + 9 * t, D.mu[t], D.lam[t], &bad);
    if (bad) inv = 1; else eel += dt2 * D.vol[t] * psi;
  }
  // affine DoF bodies: warp per body, lane i < 12 owns DoF i (row i of M^y); products through shuffles
  {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nwb = blockDim.x >> 5;
    for (int d = wid; d < D.ND; d += nwb) {
      const int b = D.dof_body[d];
      const int i = lane < 12 ? lane : 11;
      const size_t o = 3 * (size_t)D.V + 12 * (size_t)d + i;
      const double yi = q[o] + alpha * p[o];
      const double dyi = yi - qt[o];
      const double* Mrow = D.My + (size_t)b * 144 + 12 * i;
      double t = 0.0;
#pragma unroll
      for (int j = 0; j < 12; ++j) t += Mrow[j] * __shfl_sync(0xffffffffu, dyi, j);
      const double s = warp_sum(lane < 12 ? dyi * t : 0.0);
      const int ki = D.kin_of_body[b];
      double a1 = 0.0, a2 = 0.0;
      if (ki >= 0) {
        const double ri = yi - D.s_kin[((size_t)e * D.NK + ki) * 12 + i];
        const double li = D.lam_kin[((size_t)e * D.NK + ki) * 12 + i];
        double Mr = 0.0;
#pragma unroll
        for (int j = 0; j < 12; ++j) Mr += Mrow[j] * __shfl_sync(0xffffffffu, ri, j);
        a1 = warp_sum(lane < 12 ? ri * Mr : 0.0);
        a2 = warp_sum(lane < 12 ? li * Mr : 0.0);
      }
      double yv[12];
#pragma unroll
      for (int j = 0; j < 12; ++j) yv[j] = __shfl_sync(0xffffffffu, yi, j);
      if (lane == 0) {
        ein += 0.5 * s;
        const v3 As1 = mul33(yv + 3, ld3(D.bs1 + 3 * b));
        egr -= dt2 * dot(G, D.bmass[b] * mk(yv[0], yv[1], yv[2]) + As1);
        eor += ortho_energy(yv + 3, dt2 * D.bkappa[b] * D.bvol[b]);
        if (ki >= 0) eal += 0.5 * rho * a1 - a2;
      }
    }
  }
  // barrier over candidates active at the trial point
  const double* P = D.P + (size_t)e * D.NVall * 3;
  const double* Pd = D.Pd + (size_t)e * D.NVall * 3;
  const int* ca = D.cand_a + (size_t)e * D.cand_cap;
  const int* cb = D.cand_b + (size_t)e * D.cand_cap;
  const double dh2 = D.dhat * D.dhat;
  const int ncl = lmode == 2 ? *nls : C.ncand;
  const int ncl_r = (ncl + blockDim.x - 1) / blockDim.x * blockDim.x;   // tile-aligned (list scan)
  int run = 0;
  for (int kk = threadIdx.x; kk < ncl_r; kk += blockDim.x) {
    int keep = 0;
    const int k = lmode == 2 ? (kk < ncl ? lsl[kk] : 0) : kk;
    if (kk < ncl) {
      int kind = (ca[k] >> 30) & 1, a = ca[k] & ((1 << 30) - 1), b = cb[k], vid[4];
      pair_vids(D, kind, a, b, vid);
      v3 X[4];
      const double aK = alpha == 0.0 ? 0.0 : alpha / C.Keff;   // Pd holds K_eff·(displacement of p)
      for (int s = 0; s < 4; ++s) X[s] = ld3(P + 3 * vid[s]) + aK * ld3(Pd + 3 * vid[s]);
      double reach = 0.0;              // lmode 1: α_ccd·(max_A ‖Pd‖ + max_B ‖Pd‖)
      if (lmode == 1) {
        double mA = 0.0, mB = 0.0;
        const int na = kind == 0 ? 1 : 2;
        for (int s = 0; s < 4; ++s) {
          const v3 u = ld3(Pd + 3 * vid[s]);
          const double l = sqrt(dot(u, u));
          if (s < na) mA = fmax(mA, l); else mB = fmax(mB, l);
        }
        reach = C.alpha_ccd * (mA + mB);
      }
      // box-distance lower bound: neither active now nor (lmode 1) reachable within this search
      double d2 = dh2 * 4.0;
      if (prim_box_dist(kind, X) - reach < D.dhat * (1.0 + 1e-9)) {
        classify(kind, X, &d2);
        if (lmode == 1) keep = sqrt(d2) - reach < D.dhat * (1.0 + 1e-9);
      }
      if (d2 < dh2) {
        double B, B1, B2;
        barrier_s(d2, D.dhat, &B, &B1, &B2);
        double m = 1.0;
        if (kind == 1 && D.mollify) {
          v3 n = cross(X[1] - X[0], X[3] - X[2]);
          double m1, m2;
          mollifier(dot(n, n), pair_eps(D, kind, a, b), &m, &m1, &m2);
        }
        eba += dt2 * D.kappa * pair_area(D, kind, a, b) * m * B;
      }
    }
    if (lmode == 1) {
      int tot;
      const int ex = block_excl_scan(keep, sh, &tot);
      if (keep) lsl[run + ex] = k;
      run += tot;
    }
  }
  if (lmode == 1 && threadIdx.x == 0) *nls = run;
  // lagged friction pairs at the trial positions (reading R20)
  double efr = 0.0;
  if (D.mu_f > 0.0) {
    const int nfr = C.n_fr, nb = C.n_act - C.n_fr;
    const int* fv = D.fr_vid + (size_t)e * D.act_cap * 4;
    const double aK = alpha == 0.0 ? 0.0 : alpha / C.Keff;
    const double eps = D.eps_v * D.dt;
    for (int k = threadIdx.x; k < nfr; k += blockDim.x) {
      const int4 vv = reinterpret_cast<const int4*>(fv)[k];
      const int ids[4] = {vv.x, vv.y, vv.z, vv.w};
      v3 X[4];
      for (int s2 = 0; s2 < 4; ++s2) X[s2] = ld3(P + 3 * ids[s2]) + aK * ld3(Pd + 3 * ids[s2]);
      efr += friction_energy(D.fr_dat + ((size_t)e * D.act_cap + k) * 16, X, eps);
    }
    (void)nb;
  }
  double v7[NTERMS] = {ein, eel, eor, egr, eba, eal, efr};
  block_sum_terms(v7, red);
  for (int i = 0; i < NTERMS; ++i) terms[i] = v7[i];
  *inverted = __syncthreads_or(inv);
}

__global__ void __launch_bounds__(NTHREADS, 2) k_energy(Dev D, int env0, double alpha) {
  const int e = env_at(D, env0, blockIdx.x);
  __shared__ double red[NTERMS * 32];
  double t[NTERMS];
  int inv;
  energy_terms(D, e, alpha, red, t, &inv);
  if (threadIdx.x == 0) {
    double* out = D.eterm + (size_t)e * 8;
    for (int i = 0; i < NTERMS; ++i) out[i] = t[i];
    out[1] = inv ? 1.0 / 0.0 : out[1];
    out[7] = inv;
  }
}

// backtracking line search from α = min(1, α_ccd); Armijo c
template <int MINB>
__global__ void __launch_bounds__(NTHREADS, MINB) k_linesearch(Dev D, int env0) {
  const int e = env_at(D, env0, blockIdx.x);
  EnvCtl& C = D.ctl[e];
  if (C.phase != PHASE_ACTIVE || C.inner_conv || C.xfail) return;
  __shared__ double red[NTERMS * 32];
  __shared__ int sh[33], nls;
  int* lsl = D.lsl + (size_t)e * D.cand_cap;
  double t[NTERMS];
  int inv;
  energy_terms(D, e, 0.0, red, t, &inv, 1, lsl, &nls, sh);
  __syncthreads();
  const double E0 = t[0] + t[1] + t[2] + t[3] + t[4] + t[5] + t[6];
  const double alpha_max = C.Keff * C.alpha_ccd;  // ACCD bound along K_eff·p, in units of p
  double alpha = fmin(1.0, alpha_max);
  const double gp = C.gp;
  int bt = 0;
  bool ok = false;
  double E1 = E0;
  while (true) {
    energy_terms(D, e, alpha, red, t, &inv, 2, lsl, &nls);
    if (!inv) {
      E1 = t[0] + t[1] + t[2] + t[3] + t[4] + t[5] + t[6];
      if (E1 <= E0 + D.armijo * alpha * gp) { ok = true; break; }
    }
    alpha *= 0.5;
    ++bt;
    if (alpha < 1e-10) break;
  }
  // expansion (reading R17b): after a full step keep doubling α while the energy keeps decreasing,
  // Armijo holds and α stays under the ACCD bound of the K-times longer sweep
  if (ok && alpha == 1.0 && C.Keff > 1.0) {
    while (2.0 * alpha <= alpha_max) {
      energy_terms(D, e, 2.0 * alpha, red, t, &inv, 2, lsl, &nls);
      if (inv) break;
      const double E2 = t[0] + t[1] + t[2] + t[3] + t[4] + t[5] + t[6];
      if (!(E2 < E1) || !(E2 <= E0 + D.armijo * 2.0 * alpha * gp)) break;
      alpha *= 2.0;
      E1 = E2;
    }
  }
  if (ok) {
    double* q = D.q + (size_t)e * D.n;
    const double* p = D.p + (size_t)e * D.n;
    for (int i = threadIdx.x; i < D.n; i += blockDim.x) q[i] += alpha * p[i];
  }
  if (threadIdx.x == 0) {
    C.ls_bt += bt;
    if (!ok) { C.phase = PHASE_FAILED; C.status = ENV_NEWTON_STALL; }
    else { C.alpha_min = fmin(C.alpha_min, alpha); C.alpha = alpha; C.energy = E1; }
    if (e == D.trace_env && D.trace) {
      const int r = *D.trace_n;
      if (r < D.trace_cap) {
        double* t = D.trace + 10 * (size_t)r;
        t[6] = ok ? alpha : -alpha; t[7] = E0; t[8] = E1; t[9] = bt;
        *D.trace_n = r + 1;
      }
    }
    C.ls_E0 = E0; C.ls_E1 = E1;
  }
}

// ------------------------------------------------------------------------------------------
// Newton / AL control (readings R13-R14): AL update when the inner solve has converged
// ------------------------------------------------------------------------------------------
__global__ void __launch_bounds__(NTHREADS) k_control(Dev D, int env0) {
  const int e = env_at(D, env0, blockIdx.x);
  EnvCtl& C = D.ctl[e];
  if (C.phase != PHASE_ACTIVE) return;
  __shared__ double red[32];
  if (C.overflow) {
    if (threadIdx.x == 0) { C.phase = PHASE_FAILED; C.status = ENV_CAPACITY; }
    return;
  }
  if (C.fault) {                                           // test-only fault injection (tac_debug_inject_fault)
    __syncthreads();
    if (threadIdx.x == 0) { C.phase = PHASE_FAILED; C.status = C.fault; C.fault = 0; }
    return;
  }
  double* q = D.q + (size_t)e * D.n;
  // exact-Hessian-first schedule (reading R14b): a failed exact attempt backs off 2, 4, .. 64
  // projected iterations; a successful one resets the back-off
  if (threadIdx.x == 0) {
    if (C.xfail) {
      C.nfail += 1;
      C.hold = min(1 << min(C.nfail, 20), D.hold_cap);
      C.exact = 0;
      C.xfail = 0;
    } else if (!C.exact) {
      if (C.hold > 0) C.hold -= 1;
      if (C.hold == 0 && D.hmode == 1) C.exact = 1;
    } else {
      C.nfail = 0;
    }
  }
  __syncthreads();
  if (C.inner_conv) {
    const double* s_att = D.s_att + (size_t)e * D.NC * 3;
    double res = 0.0;
    for (int c = threadIdx.x; c < D.NC; c += blockDim.x) {
      v3 r = ld3(q + 3 * D.att_vert[c]) - ld3(s_att + 3 * c);
      res = fmax(res, sqrt(dot(r, r)));
    }
    for (int i = threadIdx.x; i < D.NKV; i += blockDim.x) {
      int gv = D.kin_vlist[i], b = D.vert_aff[gv], ki = D.kin_of_body[b], d = D.dof_slot[b];
      const double* y = q + 3 * D.V + 12 * d;
      const double* sk = D.s_kin + ((size_t)e * D.NK + ki) * 12;
      double dy[12];
      for (int j = 0; j < 12; ++j) dy[j] = y[j] - sk[j];
      v3 u = embed(dy, ld3(D.vert_xbar + 3 * gv));
      res = fmax(res, sqrt(dot(u, u)));
    }
    res = block_max(res, red);
    __syncthreads();
    const bool done = res <= D.tolAL * C.L;
    const int rounds = C.al_rounds + 1;
    if (e == D.trace_env && D.trace) {                       // diagnostic trace row of the AL round end
      __shared__ int arg;                                    // which constraint attains the max residual
      if (threadIdx.x == 0) arg = -1;
      __syncthreads();
      for (int c = threadIdx.x; c < D.NC; c += blockDim.x) {
        v3 r = ld3(q + 3 * D.att_vert[c]) - ld3(s_att + 3 * c);
        if (sqrt(dot(r, r)) == res) atomicMax(&arg, c);
      }
      for (int i = threadIdx.x; i < D.NKV; i += blockDim.x) {
        int gv = D.kin_vlist[i], b = D.vert_aff[gv], ki = D.kin_of_body[b], d = D.dof_slot[b];
        const double* y = q + 3 * D.V + 12 * d;
        const double* sk = D.s_kin + ((size_t)e * D.NK + ki) * 12;
        double dy[12];
        for (int j = 0; j < 12; ++j) dy[j] = y[j] - sk[j];
        v3 u = embed(dy, ld3(D.vert_xbar + 3 * gv));
        if (sqrt(dot(u, u)) == res) atomicMax(&arg, (1 << 24) + gv);
      }
      __syncthreads();
      const int r = *D.trace_n;
      if (threadIdx.x == 0 && r < D.trace_cap) {
        double* t = D.trace + 10 * (size_t)r;
        t[0] = -1.0; t[1] = rounds; t[2] = C.rho; t[3] = res; t[4] = D.tolAL * C.L; t[5] = C.newton;
        t[6] = arg >> 24; t[7] = arg & 0xffffff;
        t[8] = (arg >> 24) ? D.vert_aff[arg & 0xffffff] : (arg >= 0 ? D.att_vert[arg] : -1); t[9] = 0.0;
        *D.trace_n = r + 1;
      }
      __syncthreads();
    }
    __syncthreads();
    if (done) {
      if (threadIdx.x == 0) { C.residual = res; C.al_rounds = rounds; C.phase = PHASE_DONE; C.inner_conv = 0; }
      return;
    }
    if (rounds >= D.max_al) {
      if (threadIdx.x == 0) { C.residual = res; C.al_rounds = rounds; C.phase = PHASE_FAILED; C.status = ENV_AL_INFEASIBLE; }
      return;
    }
    double rho = C.rho;
    if (res > 0.5 * C.r_prev) rho *= 2.0;
    double* lam_att = D.lam_att + (size_t)e * D.NC * 3;
    for (int c = threadIdx.x; c < D.NC; c += blockDim.x) {
      v3 r = ld3(q + 3 * D.att_vert[c]) - ld3(s_att + 3 * c);
      st3(lam_att + 3 * c, ld3(lam_att + 3 * c) - rho * r);
    }
    for (int i = threadIdx.x; i < D.NK * 12; i += blockDim.x) {
      int ki = i / 12, j = i % 12, b = D.kin_body[ki], d = D.dof_slot[b];
      double r = q[3 * D.V + 12 * d + j] - D.s_kin[((size_t)e * D.NK + ki) * 12 + j];
      D.lam_kin[((size_t)e * D.NK + ki) * 12 + j] -= rho * r;
    }
    __syncthreads();
    if (threadIdx.x == 0) { C.rho = rho; C.r_prev = res; C.residual = res; C.al_rounds = rounds; C.inner_conv = 0; }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    if (C.phase == PHASE_ACTIVE && C.newton >= D.max_newton) { C.phase = PHASE_FAILED; C.status = ENV_NEWTON_STALL; }
    if (C.phase == PHASE_ACTIVE) mark_active(D, e);
  }
}

// ------------------------------------------------------------------------------------------
// step begin / end
// ------------------------------------------------------------------------------------------
// step setup of one env (block-level): x̃ = xⁿ + Δt ẋⁿ, targets s^y = yk (this step's kinematic
// targets [NK][12]) and s^x of ∂⁻G from the mount links, AL reset, per-step counters
__device__ void begin_env(const Dev& D, int e, const double* yk) {
  EnvCtl& C = D.ctl[e];
  double* q = D.q + (size_t)e * D.n;
  double* qn = D.qn + (size_t)e * D.n;
  double* qt = D.qt + (size_t)e * D.n;
  const double* vel = D.vel + (size_t)e * D.n;
  for (int i = threadIdx.x; i < D.n; i += blockDim.x) { qn[i] = q[i]; qt[i] = q[i] + D.dt * vel[i]; }
  for (int i = threadIdx.x; i < D.NK * 12; i += blockDim.x) {
    D.s_kin[(size_t)e * D.NK * 12 + i] = yk[i];
    D.lam_kin[(size_t)e * D.NK * 12 + i] = 0.0;
  }
  for (int c = threadIdx.x; c < D.NC; c += blockDim.x) {
    int b = D.att_body[c], ki = D.kin_of_body[b];
    const double* y = ki >= 0 ? yk + 12 * ki : body_y(D, e, b);
    st3(D.s_att + ((size_t)e * D.NC + c) * 3, embed(y, ld3(D.att_local + 3 * c)));
    st3(D.lam_att + ((size_t)e * D.NC + c) * 3, mk(0, 0, 0));
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    C.phase = PHASE_ACTIVE; C.status = ENV_OK; C.inner_conv = 0; C.newton = 0; C.pcg = 0; C.ls_bt = 0;
    C.al_rounds = 0; C.n_act = 0; C.overflow = 0; C.alpha_ccd = 1.0; C.alpha_min = 1.0;  // (ncand: reusable list)
    C.rho = D.rho0; C.r_prev = 1.0 / 0.0; C.energy = 0.0; C.residual = 0.0; C.gp = 0.0; C.pnorm = 0.0; C.alpha = 1.0;
    C.exact = D.hmode >= 1 ? 1 : 0; C.hold = 0; C.nfail = 0; C.xfail = 0; C.Keff = 1.0; C.mu = 0.0;
    C.ew_has = 0; C.ew_rz0 = 0.0; C.ew_eta = 0.0;
    C.n_fr = 0; C.fr_frozen = 0;
  }
  __syncthreads();
}

__global__ void __launch_bounds__(NTHREADS) k_begin(Dev D, int env0) {
  const int e = env_at(D, env0, blockIdx.x);
  EnvCtl& C = D.ctl[e];
  if (C.disabled) { if (threadIdx.x == 0) { C.phase = PHASE_IDLE; C.status = ENV_DISABLED; } return; }
  begin_env(D, e, D.ykin + (size_t)e * D.NK * 12);
}

// end of a step (block-level): ẋ = (xⁿ⁺¹ − xⁿ)/Δt, or rollback to xⁿ and disable on failure
__device__ void end_env(const Dev& D, int e) {
  EnvCtl& C = D.ctl[e];
  double* q = D.q + (size_t)e * D.n;
  const double* qn = D.qn + (size_t)e * D.n;
  double* vel = D.vel + (size_t)e * D.n;
  const bool ok = C.phase == PHASE_DONE;
  __syncthreads();
  for (int i = threadIdx.x; i < D.n; i += blockDim.x) {
    if (ok) vel[i] = (q[i] - qn[i]) / D.dt;
    else q[i] = qn[i];
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    if (!ok) {
      if (C.phase == PHASE_ACTIVE) C.status = ENV_NEWTON_STALL;
      C.phase = PHASE_FAILED;
      C.disabled = 1;
    }
  }
  __syncthreads();
}

__global__ void __launch_bounds__(NTHREADS) k_end(Dev D, int env0) {
  const int e = env_at(D, env0, blockIdx.x);
  if (D.ctl[e].phase == PHASE_IDLE) return;
  end_env(D, e);
}

// ------------------------------------------------------------------------------------------
// state I/O helpers, validation, readout
// ------------------------------------------------------------------------------------------
__global__ void k_scatter_y(Dev D, int env0, int which /*0: y→ystat+q, 1: ydot→vel, 2: zero vel bodies*/) {
  const int e = env_at(D, env0, blockIdx.x);
  const double* st = D.ystage + (size_t)e * D.NA * 12;
  for (int i = threadIdx.x; i < D.NA * 12; i += blockDim.x) {
    int b = i / 12, j = i % 12, s = D.dof_slot[b];
    if (which == 0) {
      D.ystat[(size_t)e * D.NA * 12 + i] = st[i];
      if (s >= 0) D.q[(size_t)e * D.n + 3 * D.V + 12 * s + j] = st[i];
    } else if (s >= 0) {
      D.vel[(size_t)e * D.n + 3 * D.V + 12 * s + j] = which == 1 ? st[i] : 0.0;
    }
  }
}
__global__ void k_gather_y(Dev D, int env0, int which /*0: y, 1: ydot*/) {
  const int e = env_at(D, env0, blockIdx.x);
  double* st = D.ystage + (size_t)e * D.NA * 12;
  for (int i = threadIdx.x; i < D.NA * 12; i += blockDim.x) {
    int b = i / 12, j = i % 12, s = D.dof_slot[b];
    if (which == 0) st[i] = s >= 0 ? D.q[(size_t)e * D.n + 3 * D.V + 12 * s + j] : D.ystat[(size_t)e * D.NA * 12 + i];
    else st[i] = s >= 0 ? D.vel[(size_t)e * D.n + 3 * D.V + 12 * s + j] : 0.0;
  }
}

// after set_state: L_env (bbox diagonal of all vertices), inversion and contact-distance checks
__global__ void __launch_bounds__(NTHREADS) k_validate(Dev D, int env0) {
  const int e = env_at(D, env0, blockIdx.x);
  EnvCtl& C = D.ctl[e];
  __shared__ double red[32];
  const double* P = D.P + (size_t)e * D.NVall * 3;
  double lo[3] = {1e300, 1e300, 1e300}, hi[3] = {-1e300, -1e300, -1e300};
  for (int gv = threadIdx.x; gv < D.NVall; gv += blockDim.x)
    for (int c = 0; c < 3; ++c) { lo[c] = fmin(lo[c], P[3 * gv + c]); hi[c] = fmax(hi[c], P[3 * gv + c]); }
  double L2 = 0.0;
  for (int c = 0; c < 3; ++c) {
    double l = block_min(lo[c], red), h = block_max(hi[c], red);
    L2 += (h - l) * (h - l);
  }
  const double* q = D.q + (size_t)e * D.n;
  int bad = 0;
  for (int t = threadIdx.x; t < D.T; t += blockDim.x) {
    int4 tv = reinterpret_cast<const int4*>(D.tets)[t];
    v3 x[4] = {ld3(q + 3 * tv.x), ld3(q + 3 * tv.y), ld3(q + 3 * tv.z), ld3(q + 3 * tv.w)};
    double F[9];
    deformation_gradient(x, D.Dmi + 9 * t, F);
    if (!(det33(F) > 0.0)) bad = 1;
  }
  const int* ca = D.cand_a + (size_t)e * D.cand_cap;
  const int* cb = D.cand_b + (size_t)e * D.cand_cap;
  for (int k = threadIdx.x; k < C.ncand; k += blockDim.x) {
    int kind = (ca[k] >> 30) & 1, a = ca[k] & ((1 << 30) - 1), b = cb[k], vid[4];
    pair_vids(D, kind, a, b, vid);
    v3 X[4];
    for (int s = 0; s < 4; ++s) X[s] = ld3(P + 3 * vid[s]);
    double d2;
    classify(kind, X, &d2);
    if (!(d2 > 0.0)) bad = 1;
  }
  bad = __syncthreads_or(bad);
  if (threadIdx.x == 0) {
    C.L = sqrt(L2);
    if (C.overflow) { C.status = ENV_CAPACITY; C.disabled = 1; C.phase = PHASE_IDLE; }
    else if (bad) { C.status = ENV_BAD_STATE; C.disabled = 1; C.phase = PHASE_IDLE; }
    else { C.status = ENV_OK; C.disabled = 0; C.phase = PHASE_IDLE; }
    C.overflow = 0;
  }
}

// gel-surface readout of one env into caller buffers (block-level); R18 / P:L153
__device__ void readout_env(const Dev& D, int e, double* oc, double* om, double* of) {
  const double* q = D.q + (size_t)e * D.n;
  auto delta = [&](int v, int pad) -> v3 {
    int b = D.pad_mount[pad];
    const double* T = D.pad_T + 12 * pad;
    v3 x = ld3(q + 3 * v), loc;
    if (b >= 0) {
      const double* y = body_y(D, e, b);
      double Ai[9];
      inv33(y + 3, Ai);
      loc = mul33(Ai, x - mk(y[0], y[1], y[2]));
    } else loc = x;
    return mul33T(T + 3, loc - ld3(T)) - ld3(D.Xrest + 3 * v);
  };
  for (int i = threadIdx.x; i < D.NCOAT; i += blockDim.x) st3(oc + 3 * i, delta(D.coat_vert[i], D.coat_pad[i]));
  for (int i = threadIdx.x; i < D.NMARK; i += blockDim.x) {
    v3 pos = mk(0, 0, 0), fl = mk(0, 0, 0);
    for (int j = 0; j < 3; ++j) {
      int v = D.mark_tri[3 * i + j];
      double a = D.mark_bary[3 * i + j];
      pos += a * ld3(q + 3 * v);
      fl += a * delta(v, D.mark_pad[i]);
    }
    st3(om + 3 * i, pos);
    st3(of + 3 * i, fl);
  }
}

__global__ void k_readout(Dev D, int env0) {
  const int e = env_at(D, env0, blockIdx.x);
  readout_env(D, e, D.out_coat + (size_t)e * D.NCOAT * 3, D.out_mpos + (size_t)e * D.NMARK * 3,
              D.out_mflow + (size_t)e * D.NMARK * 3);
}

// ------------------------------------------------------------------------------------------
// scheduled multi-step mode: each env advances through its own step sequence; an env that finished
// step k (DONE/FAILED) is finalised, read out into the per-step buffers and immediately starts step
// k+1 with its scheduled targets, so converged envs do not wait for the slowest env
// ------------------------------------------------------------------------------------------
__global__ void __launch_bounds__(NTHREADS) k_begin_sched(Dev D, int env0, const double* sched) {
  const int e = env_at(D, env0, blockIdx.x);
  EnvCtl& C = D.ctl[e];
  if (threadIdx.x == 0) C.step = 0;
  if (C.disabled) { if (threadIdx.x == 0) { C.phase = PHASE_IDLE; C.status = ENV_DISABLED; } return; }
  begin_env(D, e, sched + (size_t)e * D.NK * 12);
}

__global__ void __launch_bounds__(NTHREADS) k_advance(Dev D, int env0, const double* sched, int nsteps, double* oc,
                                                      double* om, double* of) {
  const int e = env_at(D, env0, blockIdx.x);
  EnvCtl& C = D.ctl[e];
  const int ph = C.phase;
  if (ph != PHASE_DONE && ph != PHASE_FAILED) return;
  end_env(D, e);
  const int k = C.step;
  if (oc) {
    readout_env(D, e, oc + ((size_t)k * D.E + e) * D.NCOAT * 3, om + ((size_t)k * D.E + e) * D.NMARK * 3,
                of + ((size_t)k * D.E + e) * D.NMARK * 3);
  }
  __syncthreads();
  if (ph == PHASE_DONE && k + 1 < nsteps) {
    begin_env(D, e, sched + ((size_t)(k + 1) * D.E + e) * D.NK * 12);
    if (threadIdx.x == 0) { C.step = k + 1; mark_active(D, e); }
  } else if (threadIdx.x == 0) {
    C.step = k + 1;
    if (ph == PHASE_DONE) C.phase = PHASE_IDLE;   // schedule finished (failures stay FAILED/disabled)
  }
}

// ------------------------------------------------------------------------------------------
// depth and normal maps of the deformed coated surface (reading R22): one CTA per (env, pad);
// the pad's coated vertices are brought to its sensor frame, the coated triangles binned into 16×16-pixel
// cells (lists sorted by triangle → deterministic sums), then each pixel takes the max depth and the
// summed area vector over the covering triangles of its cell
// ------------------------------------------------------------------------------------------
constexpr int DEPTH_THREADS = 256;
constexpr int DEPTH_CELL = 16;
__global__ void __launch_bounds__(DEPTH_THREADS) k_depth(Dev D, int env0, int H, int W, int ent_cap, double* depth,
                                                          double* normal) {
  const int el = blockIdx.x / D.npads, p = blockIdx.x % D.npads, e = env0 + el;
  extern __shared__ double dsm_depth[];
  const int c0 = D.coat_ptr[p], nc = D.coat_ptr[p + 1] - c0;
  const int t0 = D.ct_ptr[p], nt = D.ct_ptr[p + 1] - t0;
  const int ncx = (W + DEPTH_CELL - 1) / DEPTH_CELL, ncy = (H + DEPTH_CELL - 1) / DEPTH_CELL, ncell = ncx * ncy;
  double* X = dsm_depth;                                    // [nc][3] sensor-frame deformed positions
  int* cnt = reinterpret_cast<int*>(X + 3 * (size_t)nc);    // [ncell + 1]
  int* cur = cnt + ncell + 1;                               // [ncell]
  int* ent = cur + ncell;                                   // [ent_cap] triangle index (local)
  __shared__ int sh[33], ovf;
  const double* q = D.q + (size_t)e * D.n;
  const double* T = D.pad_T + 12 * p;
  const int mb = D.pad_mount[p];
  double Ai[9] = {1, 0, 0, 0, 1, 0, 0, 0, 1};
  v3 tl = mk(0, 0, 0);
  if (mb >= 0) {
    const double* y = body_y(D, e, mb);
    inv33(y + 3, Ai);
    tl = mk(y[0], y[1], y[2]);
  }
  for (int i = threadIdx.x; i < nc; i += blockDim.x) {
    const int v = D.coat_vert[c0 + i];
    const v3 loc = mb >= 0 ? mul33(Ai, ld3(q + 3 * v) - tl) : ld3(q + 3 * v);
    st3(X + 3 * i, mul33T(T + 3, loc - ld3(T)));
  }
  const double* cam = D.cam + 5 * p;
  const double x0 = cam[0], y0 = cam[2], dx = (cam[1] - cam[0]) / (W - 1), dy = (cam[3] - cam[2]) / (H - 1), zref = cam[4];
  for (int i = threadIdx.x; i <= ncell; i += blockDim.x) cnt[i] = 0;
  if (threadIdx.x == 0) ovf = 0;
  __syncthreads();
  const int* tri = D.ct_tri + 3 * (size_t)t0;
  // pixel-index range of a triangle's projected bounding box (pixels whose centre can be covered)
  auto prange = [&](int t, int* j0, int* j1, int* i0, int* i1) {
    const int a = tri[3 * t] - c0, b = tri[3 * t + 1] - c0, c = tri[3 * t + 2] - c0;
    const double xl = fmin(X[3 * a], fmin(X[3 * b], X[3 * c])), xh = fmax(X[3 * a], fmax(X[3 * b], X[3 * c]));
    const double yl = fmin(X[3 * a + 1], fmin(X[3 * b + 1], X[3 * c + 1])), yh = fmax(X[3 * a + 1], fmax(X[3 * b + 1], X[3 * c + 1]));
    const double px = 1e-7 * (xh - xl + dx), py = 1e-7 * (yh - yl + dy);   // margin ≫ the coverage tolerance
    *j0 = max(0, (int)ceil((xl - px - x0) / dx)); *j1 = min(W - 1, (int)floor((xh + px - x0) / dx));
    *i0 = max(0, (int)ceil((yl - py - y0) / dy)); *i1 = min(H - 1, (int)floor((yh + py - y0) / dy));
  };
  for (int t = threadIdx.x; t < nt; t += blockDim.x) {
    int j0, j1, i0, i1;
    prange(t, &j0, &j1, &i0, &i1);
    if (j0 > j1 || i0 > i1) continue;
    for (int cy = i0 / DEPTH_CELL; cy <= i1 / DEPTH_CELL; ++cy)
      for (int cx = j0 / DEPTH_CELL; cx <= j1 / DEPTH_CELL; ++cx) atomicAdd(&cnt[cy * ncx + cx], 1);
  }
  __syncthreads();
  {
    const int per = (ncell + blockDim.x - 1) / blockDim.x, b0 = threadIdx.x * per;
    int sum = 0;
    for (int i = 0; i < per && b0 + i < ncell; ++i) sum += cnt[b0 + i];
    int tot;
    int run = block_excl_scan(sum, sh, &tot);
    for (int i = 0; i < per && b0 + i < ncell; ++i) { const int c = cnt[b0 + i]; cnt[b0 + i] = run; cur[b0 + i] = run; run += c; }
    __syncthreads();
    if (threadIdx.x == 0) { cnt[ncell] = tot; if (tot > ent_cap) ovf = 1; }
    __syncthreads();
  }
  const bool brute = ovf != 0;                             // too many entries: every pixel tests every triangle
  if (!brute) {
    for (int t = threadIdx.x; t < nt; t += blockDim.x) {
      int j0, j1, i0, i1;
      prange(t, &j0, &j1, &i0, &i1);
      if (j0 > j1 || i0 > i1) continue;
      for (int cy = i0 / DEPTH_CELL; cy <= i1 / DEPTH_CELL; ++cy)
        for (int cx = j0 / DEPTH_CELL; cx <= j1 / DEPTH_CELL; ++cx) ent[atomicAdd(&cur[cy * ncx + cx], 1)] = t;
    }
    __syncthreads();
    for (int c = threadIdx.x; c < ncell; c += blockDim.x)            // ascending triangle order per cell
      for (int i = cnt[c] + 1; i < cnt[c + 1]; ++i) {
        const int key = ent[i];
        int j = i - 1;
        while (j >= cnt[c] && ent[j] > key) { ent[j + 1] = ent[j]; --j; }
        ent[j + 1] = key;
      }
    __syncthreads();
  }
  const size_t plane = (size_t)H * W, base = ((size_t)el * D.npads + p) * plane;
  for (int px = threadIdx.x; px < H * W; px += blockDim.x) {
    const int i = px / W, j = px % W;
    const double cxp = x0 + j * dx, cyp = y0 + i * dy;
    const int cell = (i / DEPTH_CELL) * ncx + (j / DEPTH_CELL);
    const int k0 = brute ? 0 : cnt[cell], k1 = brute ? nt : cnt[cell + 1];
    double best = -1.0 / 0.0;
    v3 nsum = mk(0, 0, 0);
    bool any = false;
    for (int k = k0; k < k1; ++k) {
      const int t = brute ? k : ent[k];
      const int a = tri[3 * t] - c0, b = tri[3 * t + 1] - c0, c = tri[3 * t + 2] - c0;
      const v3 A = ld3(X + 3 * a), B = ld3(X + 3 * b), Cc = ld3(X + 3 * c);
      const double ar = (B.x - A.x) * (Cc.y - A.y) - (B.y - A.y) * (Cc.x - A.x);
      if (ar == 0.0) continue;
      const double wa = ((B.x - cxp) * (Cc.y - cyp) - (B.y - cyp) * (Cc.x - cxp)) / ar;
      const double wb = ((Cc.x - cxp) * (A.y - cyp) - (Cc.y - cyp) * (A.x - cxp)) / ar;
      const double wc = ((A.x - cxp) * (B.y - cyp) - (A.y - cyp) * (B.x - cxp)) / ar;
      if (wa < -1e-9 || wb < -1e-9 || wc < -1e-9) continue;
      any = true;
      best = fmax(best, zref - (wa * A.z + wb * B.z + wc * Cc.z));
      v3 av = cross(B - A, Cc - A);
      if (av.z < 0.0) av = -av;
      nsum += av;
    }
    if (depth) depth[base + px] = any ? best : 0.0 / 0.0;
    if (normal) {
      const double ln = sqrt(dot(nsum, nsum));
      st3(normal + 3 * (base + px), any && ln > 0.0 ? (1.0 / ln) * nsum : mk(0, 0, 0));
    }
  }
}

// ------------------------------------------------------------------------------------------
// forward kinematics / action compilation: one thread per (env, link); each thread
// multiplies the homogeneous transforms from the root to its link (depth ≤ n_links) — no inter-thread
// dependencies, deterministic
// ------------------------------------------------------------------------------------------
struct Xf { double t[3], R[9]; };
__device__ __forceinline__ Xf xf_load(const double* y) {
  Xf a;
  for (int i = 0; i < 3; ++i) a.t[i] = y[i];
  for (int i = 0; i < 9; ++i) a.R[i] = y[3 + i];
  return a;
}
__device__ __forceinline__ Xf xf_mul(const Xf& a, const Xf& b) {   // a ∘ b: x ↦ a.t + a.R (b.t + b.R x)
  Xf c;
  for (int i = 0; i < 3; ++i) {
    c.t[i] = a.t[i] + a.R[3 * i] * b.t[0] + a.R[3 * i + 1] * b.t[1] + a.R[3 * i + 2] * b.t[2];
    for (int j = 0; j < 3; ++j) c.R[3 * i + j] = a.R[3 * i] * b.R[j] + a.R[3 * i + 1] * b.R[3 + j] + a.R[3 * i + 2] * b.R[6 + j];
  }
  return c;
}
__device__ __forceinline__ Xf xf_rot(const double* a, double th) {   // Rodrigues: cos θ I + sin θ [a]× + (1 − cos θ) a aᵀ
  Xf r;
  const double c = cos(th), s = sin(th), k = 1.0 - c;
  r.t[0] = r.t[1] = r.t[2] = 0.0;
  r.R[0] = c + k * a[0] * a[0]; r.R[1] = k * a[0] * a[1] - s * a[2]; r.R[2] = k * a[0] * a[2] + s * a[1];
  r.R[3] = k * a[1] * a[0] + s * a[2]; r.R[4] = c + k * a[1] * a[1]; r.R[5] = k * a[1] * a[2] - s * a[0];
  r.R[6] = k * a[2] * a[0] - s * a[1]; r.R[7] = k * a[2] * a[1] + s * a[0]; r.R[8] = c + k * a[2] * a[2];
  return r;
}
// joint frame of link i of env e (walks the ancestors; chains are shallow)
__device__ Xf fk_joint_frame(const Dev& D, int e, const double* q, int i) {
  int path[32], depth = 0;
  for (int l = i; l >= 0 && depth < 32; l = D.ch_parent[l]) path[depth++] = l;
  Xf T = xf_load(D.ch_base + (size_t)e * 12);
  for (int d = depth - 1; d >= 0; --d) {
    const int l = path[d];
    T = xf_mul(T, xf_load(D.ch_origin + 12 * (size_t)l));
    const int j = D.ch_joint[l];
    if (j >= 0) T = xf_mul(T, xf_rot(D.ch_axis + 3 * (size_t)l, q[j]));
  }
  return T;
}
__global__ void k_fk(Dev D, int env0, int ne, const double* q /*[ne][n_joints]*/) {
  const int gid = blockIdx.x * blockDim.x + threadIdx.x;
  if (gid >= ne * D.n_links) return;
  const int el = gid / D.n_links, i = gid % D.n_links, e = env0 + el;
  const Xf T = xf_mul(fk_joint_frame(D, e, q + (size_t)el * D.n_joints, i), xf_load(D.ch_body + 12 * (size_t)i));
  double* out = D.ykin + ((size_t)e * D.NK + D.ch_kin[i]) * 12;
  for (int k = 0; k < 3; ++k) out[k] = T.t[k];
  for (int k = 0; k < 9; ++k) out[3 + k] = T.R[k];
}

// ------------------------------------------------------------------------------------------
// host launchers
// ------------------------------------------------------------------------------------------
// per-device state: the __constant__ tables and the dynamic-shared-memory attributes exist once per
// device (CUDA keeps module state per device), so both are tracked per device id
constexpr int MAX_DEVICES = 64;
static int cur_device() {
  int d = 0;
  cudaGetDevice(&d);
  return (d >= 0 && d < MAX_DEVICES) ? d : 0;
}
static bool g_tables_ready[MAX_DEVICES] = {};
cudaError_t init_tables() {
  const int dev = cur_device();
  if (g_tables_ready[dev]) return cudaSuccess;
  unsigned char r[PH], c[PH];
  for (int i = 0; i < 12; ++i)
    for (int j = i; j < 12; ++j) { int k = sym_idx(i, j, 12); r[k] = (unsigned char)i; c[k] = (unsigned char)j; }
  unsigned char cp[PH];
  for (int be = 0; be < 12; ++be)
    for (int al = 0; al <= be; ++al) cp[be * (be + 1) / 2 + al] = (unsigned char)sym_idx(al, be, 12);
  cudaError_t err = cudaMemcpyToSymbol(c_unpack_r, r, PH);
  if (err == cudaSuccess) err = cudaMemcpyToSymbol(c_colpk, cp, PH);
  if (err == cudaSuccess) err = cudaMemcpyToSymbol(c_unpack_c, c, PH);
  if (err == cudaSuccess) g_tables_ready[dev] = true;
  return err;
}

// raise a kernel's dynamic shared-memory limit to `bytes` on the current device (cached per device
// and kernel); false if the device cannot give that much
template <class K>
static bool ensure_smem(K kernel, size_t* cache /*[MAX_DEVICES]*/, size_t bytes) {
  const int dev = cur_device();
  if (bytes <= 48 * 1024 || bytes <= cache[dev]) return true;
  if (cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  cache[dev] = bytes;
  return true;
}

void launch_positions(const Dev& D, int env0, int ne, int with_p, int force, cudaStream_t s) {
  k_positions<<<ne, NTHREADS, 0, s>>>(D, env0, with_p, force);
}
void launch_broad(const Dev& D, int env0, int ne, int swept, int force, cudaStream_t s) {
  k_broad<<<ne, BROAD_THREADS, 0, s>>>(D, env0, swept, force);
}
void launch_narrow(const Dev& D, int env0, int ne, int force, cudaStream_t s) {
  size_t smem = (size_t)(2 * D.V + 1) * sizeof(int);
  // 3 CTAs/SM measured faster than 2 (C3 narrow 280 -> 240 ms / 10 steps); TAC_NARROW_MINB=2 restores 128 registers
  static const int minb = getenv("TAC_NARROW_MINB") ? atoi(getenv("TAC_NARROW_MINB")) : 3;
  if (minb == 3) k_narrow<3><<<ne, NTHREADS, smem, s>>>(D, env0, force);
  else k_narrow<2><<<ne, NTHREADS, smem, s>>>(D, env0, force);
}
void launch_tets(const Dev& D, int env0, int ne, int force, cudaStream_t s) {
  dim3 grid((D.T + NTHREADS - 1) / NTHREADS, ne);
  if (D.T == 0) return;
  if (D.hmode == 2 && !force) k_tets_x<<<grid, NTHREADS, 0, s>>>(D, env0, force);
  else k_tets<<<grid, NTHREADS, 0, s>>>(D, env0, force);
}
void launch_pairs(const Dev& D, int env0, int ne, int force, cudaStream_t s) {
  // hessian_mode 2 (R14c) keeps every env on exact Hessians; modes 0/1 (and debug evaluations,
  // force = 1) may hold projected envs, which the warp-Jacobi kernel serves
  if (D.hmode != 2 || force) {
    dim3 grid(std::min((D.act_cap + PAIRS_PER_CTA - 1) / PAIRS_PER_CTA, PAIR_GRID_X), ne);
    k_pairs<<<grid, PAIR_WARPS * 32, 0, s>>>(D, env0, force);
    k_bpart_proj<<<dim3((D.act_cap + 31) / 32, ne), 256, 0, s>>>(D, env0, force);
  }
  if (D.hmode != 0 || force) {
    dim3 grid(std::min((D.act_cap + 127) / 128, 8), ne);
    k_pairs_x<<<grid, 128, 0, s>>>(D, env0, force);
  }
}
void launch_assemble(const Dev& D, int env0, int ne, int force, cudaStream_t s) {
  // threads: one per soft vertex in a single pass when V ≤ 320 (rounded to warps), else 256
  const int thr = D.V <= ASM_SOFT_MAX ? std::max(128, (D.V + 31) / 32 * 32) : NTHREADS;
  const int bytes = ((D.V + 3) / 2) * (int)sizeof(double) + (D.maxrl <= 32 ? (thr / 8) * D.maxrl * 9 * (int)sizeof(double) : 0);
  static size_t attr[MAX_DEVICES] = {}, attr3[MAX_DEVICES] = {};
  const bool small = D.V <= ASM_SOFT_MAX;
  if (small) ensure_smem(k_assemble_soft<3>, attr3, bytes);
  else ensure_smem(k_assemble_soft<2>, attr, bytes);
  if (D.NEs > 0) k_asm_edges<<<dim3((D.NEs + NTHREADS - 1) / NTHREADS, ne), NTHREADS, 0, s>>>(D, env0, force);
  if (small) k_assemble_soft<3><<<ne, thr, bytes, s>>>(D, env0, force);
  else k_assemble_soft<2><<<ne, thr, bytes, s>>>(D, env0, force);
  if (D.ND > 0) k_assemble_body<<<ne, NTHREADS, 0, s>>>(D, env0, force);
}
static size_t spmv_smem(const Dev& D) { return (size_t)(NTHREADS / 32) * D.ND * 12 * sizeof(double) + 8; }

// which PCG kernel serves this batch: the env-resident k_pcg_r / k_pcg_r512 when the condensed operator,
// the kernel's static shared memory and the vectors fit the device's opt-in shared memory per block,
// else the streamed-operator k_pcg.  Env overrides for experiments: TAC_PCG_RESIDENT=0 (always stream),
// TAC_PCG_R_LB512=1 (512-thread register budget), TAC_PCG_LPR ∈ {1,2,4}, TAC_PCG_THREADS ≤ 512.
struct PcgPlan { int path; int threads; size_t bytes; int lpr; };

template <int NC>
static cudaError_t cl_attr(size_t bytes) {
  cudaError_t e = cudaFuncSetAttribute(k_pcg_cl<NC>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
  if (e == cudaSuccess && NC > 8) e = cudaFuncSetAttribute(k_pcg_cl<NC>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  return e;
}
template <int NC>
static size_t cl_static_smem() {
  cudaFuncAttributes fa;
  if (cudaFuncGetAttributes(&fa, k_pcg_cl<NC>) != cudaSuccess) { cudaGetLastError(); return (size_t)1 << 30; }
  return fa.sharedSizeBytes;
}
// the cluster plan fits: static + dynamic shared memory within the opt-in limit, attributes accepted
// and at least one cluster can be resident (cached per device)
static bool cl_fits(const Dev& D) {
  static int ok[MAX_DEVICES][5] = {};             // 0 unknown, 1 yes, 2 no (per device, per cluster size)
  const int dev = cur_device();
  const int k = D.cl.nc == 1 ? 0 : D.cl.nc == 2 ? 1 : D.cl.nc == 4 ? 2 : D.cl.nc == 8 ? 3 : 4;
  static size_t sized[MAX_DEVICES][5] = {};
  if (ok[dev][k] == 2 && sized[dev][k] >= D.cl.smem) return false;
  if (ok[dev][k] == 1 && sized[dev][k] >= D.cl.smem) return true;
  int optin = 0;
  cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  size_t st = 0;
  cudaError_t e = cudaSuccess;
  switch (D.cl.nc) {
    case 1: st = cl_static_smem<1>(); e = cl_attr<1>(D.cl.smem); break;
    case 2: st = cl_static_smem<2>(); e = cl_attr<2>(D.cl.smem); break;
    case 4: st = cl_static_smem<4>(); e = cl_attr<4>(D.cl.smem); break;
    case 8: st = cl_static_smem<8>(); e = cl_attr<8>(D.cl.smem); break;
    case 16: st = cl_static_smem<16>(); e = cl_attr<16>(D.cl.smem); break;
    default: e = cudaErrorInvalidValue;
  }
  bool good = e == cudaSuccess && st + D.cl.smem <= (size_t)optin;
  if (!good) cudaGetLastError();
  ok[dev][k] = good ? 1 : 2;
  sized[dev][k] = D.cl.smem;
  return good;
}

template <int NC>
static void launch_cl(const Dev& D, int env0, int ne, int force, cudaStream_t s) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(ne * NC);
  cfg.blockDim = dim3(D.cl.threads);
  cfg.dynamicSmemBytes = D.cl.smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = NC;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = NC > 1 ? 1 : 0;
  cudaLaunchKernelEx(&cfg, k_pcg_cl<NC>, D, D.cl, env0, force);
}
static PcgPlan pcg_plan(const Dev& D) {
  static const int lpr_env = getenv("TAC_PCG_LPR") ? atoi(getenv("TAC_PCG_LPR")) : 1;
  static const int thr_env = getenv("TAC_PCG_THREADS") ? atoi(getenv("TAC_PCG_THREADS")) : 0;
  static const int resident = getenv("TAC_PCG_RESIDENT") ? atoi(getenv("TAC_PCG_RESIDENT")) : 1;
  static const int lb512 = getenv("TAC_PCG_R_LB512") ? atoi(getenv("TAC_PCG_R_LB512")) : 0;
  static const int cluster_env = getenv("TAC_PCG_CLUSTER") ? atoi(getenv("TAC_PCG_CLUSTER")) : -1;
  const int lpr = (lpr_env == 2 || lpr_env == 4) ? lpr_env : 1;
  const int thr = (thr_env >= 128 && thr_env <= PCG_R_THREADS && thr_env % 32 == 0) ? thr_env : pcg_r_threads(D.V);
  const size_t rb = pcg_r_bytes(D, thr);
  // preference: the single-CTA env-resident k_pcg_r (measured faster than k_pcg_cl with one CTA on C2:
  // 229 vs 285 ms / 10 steps), else the streamed k_pcg; TAC_PCG_CLUSTER=n forces the cluster-resident
  // k_pcg_cl with n CTAs per env
  const bool force_cl = cluster_env > 0;
  if (resident && !force_cl) {
    const bool use512 = thr > 384 || lb512;
    cudaFuncAttributes fa;
    int optin = 0;
    const cudaError_t e1 = use512 ? cudaFuncGetAttributes(&fa, k_pcg_r512) : cudaFuncGetAttributes(&fa, k_pcg_r);
    const cudaError_t e2 = cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, cur_device());
    if (e1 == cudaSuccess && e2 == cudaSuccess && rb + fa.sharedSizeBytes <= (size_t)optin)
      return PcgPlan{use512 ? PCG_RESIDENT512 : PCG_RESIDENT, thr, rb, lpr};
    cudaGetLastError();
  }
  // the cluster kernel only on request: on C3 (16-CTA clusters, ≤ 9 envs in flight) it measured 10.3 s
  // of PCG per 4 steps against 5.7 s for the streamed kernel (profiles/r2_c3_pcg_ab.json)
  if (resident && force_cl && D.cl.nc > 0 && cl_fits(D)) return PcgPlan{PCG_CLUSTER, D.cl.threads, D.cl.smem, 1};
  const size_t with_vec = spmv_smem(D) + (size_t)5 * D.n * sizeof(double);
  const size_t with_d = spmv_smem(D) + (size_t)D.n * sizeof(double);
  if (with_vec <= 200 * 1024) return PcgPlan{PCG_STREAM_VSM, NTHREADS, with_vec, lpr};
  if (with_d <= 110 * 1024) return PcgPlan{PCG_STREAM_D, NTHREADS, with_d, lpr};   // 2 CTAs per SM
  return PcgPlan{PCG_STREAM, NTHREADS, spmv_smem(D), lpr};
}

int pcg_path(const Dev& D) { return pcg_plan(D).path; }
const char* pcg_path_name(int path) {
  switch (path) {
    case PCG_RESIDENT: return "k_pcg_r";
    case PCG_RESIDENT512: return "k_pcg_r512";
    case PCG_STREAM_VSM: return "k_pcg (streamed operator, vectors in shared memory)";
    case PCG_STREAM: return "k_pcg (streamed operator)";
    case PCG_STREAM_D: return "k_pcg (streamed operator, search direction in shared memory)";
    case PCG_CLUSTER: return "k_pcg_cl";
    default: return "";
  }
}

void launch_cluster_pcg(const Dev& D, int env0, int ne, int force, cudaStream_t s) {
  switch (D.cl.nc) {
    case 1: launch_cl<1>(D, env0, ne, force, s); return;
    case 2: launch_cl<2>(D, env0, ne, force, s); return;
    case 4: launch_cl<4>(D, env0, ne, force, s); return;
    case 8: launch_cl<8>(D, env0, ne, force, s); return;
    case 16: launch_cl<16>(D, env0, ne, force, s); return;
  }
}
bool tail_pcg_available(const Dev& D) { return D.cl.nc > 1 && cl_fits(D); }

void launch_pcg(const Dev& D, int env0, int ne, int force, cudaStream_t s) {
  PcgPlan pl = pcg_plan(D);
  if (pl.path == PCG_CLUSTER) {
    switch (D.cl.nc) {
      case 1: launch_cl<1>(D, env0, ne, force, s); return;
      case 2: launch_cl<2>(D, env0, ne, force, s); return;
      case 4: launch_cl<4>(D, env0, ne, force, s); return;
      case 8: launch_cl<8>(D, env0, ne, force, s); return;
      case 16: launch_cl<16>(D, env0, ne, force, s); return;
    }
  }
  if (pl.path == PCG_RESIDENT || pl.path == PCG_RESIDENT512) {
    static size_t c384[MAX_DEVICES] = {}, c512[MAX_DEVICES] = {};
    const bool ok = pl.path == PCG_RESIDENT ? ensure_smem(k_pcg_r, c384, pl.bytes) : ensure_smem(k_pcg_r512, c512, pl.bytes);
    if (ok) {
      if (pl.path == PCG_RESIDENT) k_pcg_r<<<ne, pl.threads, pl.bytes, s>>>(D, env0, force, pl.lpr);
      else k_pcg_r512<<<ne, pl.threads, pl.bytes, s>>>(D, env0, force, pl.lpr);
      return;
    }
    const size_t with_vec = spmv_smem(D) + (size_t)5 * D.n * sizeof(double);   // attribute refused: stream
    pl = PcgPlan{with_vec <= 200 * 1024 ? PCG_STREAM_VSM : PCG_STREAM, NTHREADS,
                 with_vec <= 200 * 1024 ? with_vec : spmv_smem(D), pl.lpr};
  }
  static size_t cst[MAX_DEVICES] = {};
  static const int sfused = getenv("TAC_PCG_STREAM_FUSED") ? atoi(getenv("TAC_PCG_STREAM_FUSED")) : 1;
  static const int slpr = getenv("TAC_PCG_STREAM_LPR") ? atoi(getenv("TAC_PCG_STREAM_LPR")) : 1;
  const int vsm = pl.path == PCG_STREAM_VSM ? 1 : (pl.path == PCG_STREAM_D ? 2 : 0), lpr = slpr == 2 || slpr == 4 ? slpr : 1;
  ensure_smem(k_pcg<2>, cst, pl.bytes);
  k_pcg<2><<<ne, NTHREADS, pl.bytes, s>>>(D, env0, force, vsm, sfused, lpr);
}
void launch_spmv(const Dev& D, int env0, const double* x, double* y, cudaStream_t s) {
  k_spmv<<<1, NTHREADS, spmv_smem(D), s>>>(D, env0, x, y);
}
void launch_ccd(const Dev& D, int env0, int ne, int force, cudaStream_t s) {
  k_ccd<<<ne, NTHREADS, 0, s>>>(D, env0, force);
}
void launch_energy(const Dev& D, int env0, int ne, double alpha, cudaStream_t s) {
  k_energy<<<ne, NTHREADS, 0, s>>>(D, env0, alpha);
}
void launch_linesearch(const Dev& D, int env0, int ne, cudaStream_t s) {
  // 3 CTAs/SM (80 registers, some spills) measured faster than 2 (C3 line search 374 -> 344 ms / 10 steps);
  // TAC_LS_MINB=2 restores the 128-register budget
  static const int minb = getenv("TAC_LS_MINB") ? atoi(getenv("TAC_LS_MINB")) : 3;
  if (minb == 3) k_linesearch<3><<<ne, NTHREADS, 0, s>>>(D, env0);
  else k_linesearch<2><<<ne, NTHREADS, 0, s>>>(D, env0);
}
void launch_control(const Dev& D, int env0, int ne, cudaStream_t s) {
  k_control<<<ne, NTHREADS, 0, s>>>(D, env0);
}
void launch_begin(const Dev& D, int env0, int ne, cudaStream_t s) { k_begin<<<ne, NTHREADS, 0, s>>>(D, env0); }
void launch_end(const Dev& D, int env0, int ne, cudaStream_t s) { k_end<<<ne, NTHREADS, 0, s>>>(D, env0); }
void launch_scatter_y(const Dev& D, int env0, int ne, int which, cudaStream_t s) {
  k_scatter_y<<<ne, 128, 0, s>>>(D, env0, which);
}
void launch_gather_y(const Dev& D, int env0, int ne, int which, cudaStream_t s) {
  k_gather_y<<<ne, 128, 0, s>>>(D, env0, which);
}
void launch_validate(const Dev& D, int env0, int ne, cudaStream_t s) { k_validate<<<ne, NTHREADS, 0, s>>>(D, env0); }
void launch_readout(const Dev& D, int env0, int ne, cudaStream_t s) { k_readout<<<ne, 128, 0, s>>>(D, env0); }
void launch_depth(const Dev& D, int env0, int ne, int H, int W, double* depth, double* normal, cudaStream_t s) {
  const int ncell = ((W + DEPTH_CELL - 1) / DEPTH_CELL) * ((H + DEPTH_CELL - 1) / DEPTH_CELL);
  static size_t attr[MAX_DEVICES] = {};
  const size_t fixed = (size_t)24 * D.maxcv + (size_t)4 * (2 * ncell + 1) + 64;
  const int ent_cap = (int)std::max<size_t>(64, ((size_t)200 * 1024 - std::min<size_t>(fixed, (size_t)200 * 1024)) / 4);
  const size_t bytes = fixed + (size_t)4 * ent_cap;
  ensure_smem(k_depth, attr, bytes);
  k_depth<<<ne * D.npads, DEPTH_THREADS, bytes, s>>>(D, env0, H, W, ent_cap, depth, normal);
}
void launch_fk(const Dev& D, int env0, int ne, const double* q, cudaStream_t s) {
  const int n = ne * D.n_links;
  if (n > 0) k_fk<<<(n + 127) / 128, 128, 0, s>>>(D, env0, ne, q);
}
void launch_begin_sched(const Dev& D, int env0, int ne, const double* sched, cudaStream_t s) {
  k_begin_sched<<<ne, NTHREADS, 0, s>>>(D, env0, sched);
}
void launch_advance(const Dev& D, int env0, int ne, const double* sched, int nsteps, double* oc, double* om,
                    double* of, cudaStream_t s) {
  k_advance<<<ne, NTHREADS, 0, s>>>(D, env0, sched, nsteps, oc, om, of);
}

}  // namespace tac
