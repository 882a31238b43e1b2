// api.cu — host side of libtaccel_cuda.so: the C ABI of include/taccel.h.
// Template preparation (orientation, D_m⁻¹, lumped masses, canonical surfaces, rest areas, M^y by
// closed-form tet moments, BSR pattern + gather lists), workspace carving, and the host-driven
// Newton loop (one 4-byte device→host flag per Newton iteration is the only crossing).
#include <algorithm>
#include <chrono>
#include <array>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <cstdlib>
#include <map>
#include <numeric>
#include <string>
#include <tuple>
#include <vector>

#include "../../include/taccel.h"
#include "impl.cuh"
#include "launch.h"

using namespace tac;

static thread_local std::string g_err;
static tac_status fail(tac_status s, const std::string& msg) { g_err = msg; return s; }
#define CUDA_TRY(x)                                                                         \
  do {                                                                                      \
    cudaError_t _e = (x);                                                                   \
    if (_e != cudaSuccess) return fail(TAC_E_CUDA, std::string(#x) + ": " + cudaGetErrorString(_e)); \
  } while (0)

extern "C" const char* tac_last_error(void) { return g_err.c_str(); }

// every entry point runs on the batch's device and restores the caller's current device on return
struct DevGuard {
  int prev = -1;
  cudaError_t err = cudaSuccess;
  explicit DevGuard(int dev) {
    if (cudaGetDevice(&prev) != cudaSuccess) { prev = -1; cudaGetLastError(); }
    if (prev != dev) err = cudaSetDevice(dev);
  }
  ~DevGuard() {
    int cur = -1;
    if (prev >= 0 && cudaGetDevice(&cur) == cudaSuccess && cur != prev) cudaSetDevice(prev);
  }
};
#define ON_DEVICE(b)                                                                          \
  DevGuard _dg((b)->device);                                                                  \
  if (_dg.err != cudaSuccess) return fail(TAC_E_CUDA, std::string("cudaSetDevice: ") + cudaGetErrorString(_dg.err))

// ---------------------------------------------------------------------------------------------
// host template
// ---------------------------------------------------------------------------------------------
struct HostT {
  int V = 0, T = 0, NA = 0, ND = 0, NVall = 0, NSV = 0, NT = 0, NE = 0, NEs = 0, NC = 0, NK = 0, NB = 0, n = 0;
  int npads = 0, NCOAT = 0, NMARK = 0;
  double cell = 0;
  std::vector<int> tets;            // T*4
  std::vector<double> Dmi, vol, mu, lam, mass, Xrest;
  std::vector<int> sedge, vadj_ptr, vadj, vdiag_ptr, vdiag, eblk_ptr, eblk;
  std::vector<int> rptr, rcol, rblk_ptr, rblk;   // row-ordered symmetric BSR (off-diagonal)
  std::vector<int> rupx;                         // [NNZ] 2·(edge id) + (block stored transposed)
  std::vector<int> eup;                          // [NEs] row-ordered index of the edge's upper block
  std::vector<int> elo;                          // [NEs] row-ordered index of the edge's lower (transposed) block
  std::vector<int> tri_blk, edge_blk;            // [NT][6], [NE][2] BSR index of (v_i, v_j) within a soft primitive (-1)
  int NNZ = 0;
  std::vector<int> body_kind, dof_slot, dof_body;
  std::vector<double> My, MyInv, bmass, bs1, bvol, bkappa;
  std::vector<int> vert_body, vert_aff;
  std::vector<double> vert_xbar;
  std::vector<int> sverts, tris, tri_body, edges, edge_body, body_sv_ptr;
  std::vector<double> A_v, A_e, elen2;
  std::vector<unsigned char> allowed;
  std::vector<int> att_vert, att_body, att_of_vert, kin_body, kin_of_body, affv_list, kin_vlist;
  std::vector<double> att_local;
  std::vector<int> coat_vert, coat_pad, mark_tri, mark_pad, pad_mount;
  std::vector<double> mark_bary, pad_T;
  std::vector<int> ct_ptr, ct_tri, coat_ptr;     // depth maps: coated triangles per pad, coated-vertex ranges
  std::vector<double> cam;                       // [npads][5]
  // cluster PCG plan (k_pcg_cl): soft rows split into cl_nc contiguous ranges of cl_rpr rows
  int cl_nc = 0, cl_rpr = 0, cl_threads = 0, cl_nvt = 0, cl_nle_max = 0, cl_nlb_max = 0, cl_cplcap = 0;
  size_t cl_smem_bytes = 0;
  std::vector<int> cl_eptr, cl_edge, cl_bptr, cl_lrptr, cl_blk;   // cl_blk: 2 ints per block
  // sliced-ELL layout of the row-ordered soft blocks (streamed PCG)
  std::vector<int> ell_len, ell_cb, ell_col, ell_row;
  std::vector<long long> ell_vb, ell_pos;
  size_t ell_total = 0;
};

// Cluster PCG plan for nc CTAs per env (pcg_cluster.cuh): rows [r·rpr, (r+1)·rpr) on rank r; each rank
// stores the upper blocks of the soft edges touching its rows and, per row, (2·local edge + transposed,
// rank << 16 | local row of the column vertex).  False if the rank does not fit one CTA.
static bool plan_cluster(HostT& H, int nc, size_t budget) {
  const int V = H.V, ND = H.ND;
  if (V == 0) return false;
  const int rpr = (V + nc - 1) / nc;
  if (rpr > 65535) return false;
  const int nvt = (rpr + 31) / 32 * 32;
  const int threads = nvt + 32 * ((ND + 1) / 2);
  if (threads > CL_MAX_THREADS) return false;
  std::vector<int> eptr(1, 0), edge, bptr(1, 0), lrptr, blk;
  int nle_max = 0, nlb_max = 0;
  for (int r = 0; r < nc; ++r) {
    const int v0 = r * rpr, v1 = std::min(V, v0 + rpr);
    std::vector<int> es;
    for (int v = v0; v < v1; ++v)
      for (int j = H.rptr[v]; j < H.rptr[v + 1]; ++j) es.push_back(H.rupx[j] >> 1);
    std::sort(es.begin(), es.end());
    es.erase(std::unique(es.begin(), es.end()), es.end());
    std::map<int, int> loc;
    for (size_t i = 0; i < es.size(); ++i) loc[es[i]] = (int)i;
    edge.insert(edge.end(), es.begin(), es.end());
    eptr.push_back((int)edge.size());
    int nb = 0;
    for (int v = v0; v < v0 + rpr; ++v) {
      lrptr.push_back(nb);
      if (v >= v1) continue;
      for (int j = H.rptr[v]; j < H.rptr[v + 1]; ++j) {
        const int col = H.rcol[j];
        blk.push_back(2 * loc[H.rupx[j] >> 1] + (H.rupx[j] & 1));
        blk.push_back(((col / rpr) << 16) | (col % rpr));
        ++nb;
      }
    }
    lrptr.push_back(nb);
    bptr.push_back(bptr.back() + nb);
    nle_max = std::max(nle_max, (int)es.size());
    nlb_max = std::max(nlb_max, nb);
  }
  const int nw = threads / 32;
  const size_t base = cl_smem(rpr, nle_max, nlb_max, ND, nw, 0).end;
  if (base > budget) return false;
  const long want = (long)rpr * std::max(ND, 0);
  const long fit = (long)((budget - base) / 320);
  H.cl_cplcap = (int)std::max(0L, std::min(want, fit));
  H.cl_nc = nc; H.cl_rpr = rpr; H.cl_threads = threads; H.cl_nvt = nvt; H.cl_nle_max = nle_max; H.cl_nlb_max = nlb_max;
  H.cl_smem_bytes = cl_smem(rpr, nle_max, nlb_max, ND, nw, H.cl_cplcap).end;
  H.cl_eptr = eptr; H.cl_edge = edge; H.cl_bptr = bptr; H.cl_lrptr = lrptr; H.cl_blk = blk;
  return true;
}

// smallest cluster (1, 2, 4, 8, 16 CTAs per env) whose ranks fit the opt-in shared memory of sm_100
// (227 KB per CTA, minus the kernel's static shared memory and a margin); TAC_PCG_CLUSTER=n forces n
static void choose_cluster(HostT& H) {
  const size_t budget = 227 * 1024 - 4 * 1024;
  static const int force_nc = getenv("TAC_PCG_CLUSTER") ? atoi(getenv("TAC_PCG_CLUSTER")) : -1;
  H.cl_nc = 0;
  if (force_nc == 0) return;
  // with the tail split (TAC_PCG_TAIL_NEWTON > 0) the cluster kernel serves single slow envs, so it
  // should spread an env over several SMs: at least 4 CTAs
  static const int tail = getenv("TAC_PCG_TAIL_NEWTON") ? atoi(getenv("TAC_PCG_TAIL_NEWTON")) : 0;
  for (int nc : {1, 2, 4, 8, 16}) {
    if (force_nc > 0 && nc != force_nc) continue;
    if (force_nc <= 0 && tail > 0 && nc < 4) continue;
    if (plan_cluster(H, nc, budget)) {
      if (getenv("TAC_DEBUG_PLAN"))
        fprintf(stderr, "cluster plan: nc=%d rpr=%d threads=%d nle_max=%d nlb_max=%d cplcap=%d smem=%zu\n", H.cl_nc, H.cl_rpr,
                H.cl_threads, H.cl_nle_max, H.cl_nlb_max, H.cl_cplcap, H.cl_smem_bytes);
      return;
    }
  }
}

static std::array<double, 3> sub3(const double* a, const double* b) { return {a[0] - b[0], a[1] - b[1], a[2] - b[2]}; }
static std::array<double, 3> cross3(std::array<double, 3> a, std::array<double, 3> b) {
  return {a[1] * b[2] - a[2] * b[1], a[2] * b[0] - a[0] * b[2], a[0] * b[1] - a[1] * b[0]};
}
static double dot3(std::array<double, 3> a, std::array<double, 3> b) { return a[0] * b[0] + a[1] * b[1] + a[2] * b[2]; }

static std::array<int, 3> canon_tri(int a, int b, int c) {
  if (a <= b && a <= c) return {a, b, c};
  if (b <= a && b <= c) return {b, c, a};
  return {c, a, b};
}
static std::array<int, 3> sorted3(std::array<int, 3> t) { std::sort(t.begin(), t.end()); return t; }

static void sort_canonical(std::vector<std::array<int, 3>>& tris) {
  std::stable_sort(tris.begin(), tris.end(), [](const std::array<int, 3>& x, const std::array<int, 3>& y) {
    return sorted3(x) < sorted3(y);
  });
}
static std::vector<std::array<int, 2>> tri_edges(const std::vector<std::array<int, 3>>& tris) {
  std::vector<std::array<int, 2>> e;
  for (auto& t : tris)
    for (int i = 0; i < 3; ++i) {
      int a = t[i], b = t[(i + 1) % 3];
      e.push_back({std::min(a, b), std::max(a, b)});
    }
  std::sort(e.begin(), e.end());
  e.erase(std::unique(e.begin(), e.end()), e.end());
  return e;
}

// closed-form moments of the solid bounded by an outward triangle surface: for each signed tet
// (0, a, b, c): V = a·(b×c)/6, ∫x = V(a+b+c)/4, ∫xxᵀ = V/20 (Σ v vᵀ + s sᵀ), s = a+b+c
static void body_moments(const double* X, const std::vector<std::array<int, 3>>& tris, double rho, double* vol,
                         double* mass, double* s1, double* My) {
  double V = 0, S1[3] = {0, 0, 0}, S2[9] = {0};
  for (auto& t : tris) {
    const double *a = X + 3 * t[0], *b = X + 3 * t[1], *c = X + 3 * t[2];
    double v = (a[0] * (b[1] * c[2] - b[2] * c[1]) - a[1] * (b[0] * c[2] - b[2] * c[0]) + a[2] * (b[0] * c[1] - b[1] * c[0])) / 6.0;
    V += v;
    double s[3];
    for (int i = 0; i < 3; ++i) { s[i] = a[i] + b[i] + c[i]; S1[i] += v * s[i] / 4.0; }
    for (int i = 0; i < 3; ++i)
      for (int j = 0; j < 3; ++j) S2[3 * i + j] += v / 20.0 * (a[i] * a[j] + b[i] * b[j] + c[i] * c[j] + s[i] * s[j]);
  }
  *vol = V;
  *mass = rho * V;
  for (int i = 0; i < 3; ++i) s1[i] = rho * S1[i];
  // M^y = ∫ρ JᵀJ with y = (t, A row-major): tt = m I, t_i–A_ij = s1_j, A_ij–A_ik = S2_jk
  for (int i = 0; i < 144; ++i) My[i] = 0.0;
  for (int i = 0; i < 3; ++i) {
    My[12 * i + i] = rho * V;
    for (int j = 0; j < 3; ++j) {
      My[12 * i + 3 + 3 * i + j] = rho * S1[j];
      My[12 * (3 + 3 * i + j) + i] = rho * S1[j];
      for (int k = 0; k < 3; ++k) My[12 * (3 + 3 * i + j) + 3 + 3 * i + k] = rho * S2[3 * j + k];
    }
  }
}

static tac_status build_template(const tac_scene_desc* sc, const tac_config* cfg, HostT& H) {
  if (!sc || !cfg) return fail(TAC_E_INVALID, "null scene or config");
  const int ns = sc->n_soft, na = sc->n_affine;
  H.NA = na;
  H.npads = ns;
  H.NB = ns + na;
  if (H.NB > 32) return fail(TAC_E_INVALID, "more than 32 bodies (soft + affine) per env");
  // ---- soft ----
  std::vector<std::vector<std::array<int, 3>>> soft_tris(ns);
  int off = 0;
  for (int p = 0; p < ns; ++p) {
    const tac_soft_desc& S = sc->soft[p];
    if (S.n_verts <= 0 || S.n_tets <= 0 || !S.rest_pos || !S.tets) return fail(TAC_E_INVALID, "empty soft body");
    if (S.mount_body >= na) return fail(TAC_E_INVALID, "mount_body out of range");
    double mu = S.youngs / (2.0 * (1.0 + S.poisson));
    double lam = S.youngs * S.poisson / ((1.0 + S.poisson) * (1.0 - 2.0 * S.poisson));
    std::vector<double> m(S.n_verts, 0.0);
    std::map<std::array<int, 3>, std::pair<int, std::array<int, 3>>> faces;
    for (int t = 0; t < S.n_tets; ++t) {
      int v[4];
      for (int k = 0; k < 4; ++k) {
        v[k] = S.tets[4 * t + k];
        if (v[k] < 0 || v[k] >= S.n_verts) return fail(TAC_E_INVALID, "tet index out of range");
      }
      const double* X = S.rest_pos;
      auto d1 = sub3(X + 3 * v[1], X + 3 * v[0]), d2 = sub3(X + 3 * v[2], X + 3 * v[0]), d3 = sub3(X + 3 * v[3], X + 3 * v[0]);
      double det = dot3(d1, cross3(d2, d3));
      if (std::fabs(det / 6.0) < 1e-15)
        return fail(TAC_E_VALIDATION, "degenerate tet " + std::to_string(t) + " of soft body " + std::to_string(p));
      if (det < 0) std::swap(v[1], v[2]);
      d1 = sub3(X + 3 * v[1], X + 3 * v[0]); d2 = sub3(X + 3 * v[2], X + 3 * v[0]); d3 = sub3(X + 3 * v[3], X + 3 * v[0]);
      double Dm[9] = {d1[0], d2[0], d3[0], d1[1], d2[1], d3[1], d1[2], d2[2], d3[2]};
      double Di[9];
      inv33(Dm, Di);
      double vol = det33(Dm) / 6.0;
      for (int k = 0; k < 4; ++k) { H.tets.push_back(off + v[k]); m[v[k]] += S.density * vol / 4.0; }
      for (int i = 0; i < 9; ++i) H.Dmi.push_back(Di[i]);
      H.vol.push_back(vol);
      H.mu.push_back(mu);
      H.lam.push_back(lam);
      const int fl[4][3] = {{v[0], v[2], v[1]}, {v[0], v[1], v[3]}, {v[0], v[3], v[2]}, {v[1], v[2], v[3]}};
      for (auto& f : fl) {
        auto key = sorted3({f[0], f[1], f[2]});
        auto it = faces.find(key);
        if (it == faces.end()) faces[key] = {1, canon_tri(f[0] + off, f[1] + off, f[2] + off)};
        else it->second.first += 1;
      }
    }
    for (auto& kv : faces)
      if (kv.second.first == 1) soft_tris[p].push_back(kv.second.second);
    sort_canonical(soft_tris[p]);
    for (int i = 0; i < S.n_verts; ++i) {
      H.mass.push_back(m[i]);
      for (int c = 0; c < 3; ++c) H.Xrest.push_back(S.rest_pos[3 * i + c]);
    }
    off += S.n_verts;
  }
  H.V = off;
  H.T = (int)H.vol.size();
  if (H.V > 8000) return fail(TAC_E_CAPACITY, "more than 8000 soft vertices per env");
  if (ns + na > 32) return fail(TAC_E_CAPACITY, "more than 32 bodies per env");
  // ---- affine ----
  int nd = 0;
  for (int b = 0; b < na; ++b) {
    const tac_affine_desc& A = sc->affine[b];
    if (A.n_verts <= 0 || A.n_tris <= 0 || !A.rest_pos || !A.tris) return fail(TAC_E_INVALID, "empty affine body");
    H.body_kind.push_back(A.kind);
    H.dof_slot.push_back(A.kind == TAC_BODY_STATIC ? -1 : nd);
    if (A.kind != TAC_BODY_STATIC) { H.dof_body.push_back(b); ++nd; }
    H.bkappa.push_back(A.kappa_s);
  }
  H.ND = nd;
  H.n = 3 * H.V + 12 * nd;
  // ---- global contact primitives ----
  H.NVall = H.V;
  for (int b = 0; b < na; ++b) H.NVall += sc->affine[b].n_verts;
  H.vert_body.assign(H.NVall, 0);
  H.vert_aff.assign(H.NVall, -1);
  H.vert_xbar.assign(3 * (size_t)H.NVall, 0.0);
  {
    int o = 0;
    for (int p = 0; p < ns; ++p)
      for (int i = 0; i < sc->soft[p].n_verts; ++i, ++o) {
        H.vert_body[o] = p;
        for (int c = 0; c < 3; ++c) H.vert_xbar[3 * o + c] = sc->soft[p].rest_pos[3 * i + c];
      }
  }
  std::vector<std::array<int, 3>> all_tris;
  std::vector<std::array<int, 2>> all_edges;
  for (int p = 0; p < ns; ++p) {
    for (auto& t : soft_tris[p]) { all_tris.push_back(t); H.tri_body.push_back(p); }
    for (auto& e : tri_edges(soft_tris[p])) { all_edges.push_back(e); H.edge_body.push_back(p); }
  }
  H.My.assign(144 * (size_t)na, 0.0);
  H.bmass.assign(na, 0.0);
  H.bs1.assign(3 * na, 0.0);
  H.bvol.assign(na, 0.0);
  int o = H.V;
  for (int b = 0; b < na; ++b) {
    const tac_affine_desc& A = sc->affine[b];
    std::vector<std::array<int, 3>> tl, tg;
    for (int t = 0; t < A.n_tris; ++t) {
      int a0 = A.tris[3 * t], a1 = A.tris[3 * t + 1], a2 = A.tris[3 * t + 2];
      if (a0 < 0 || a1 < 0 || a2 < 0 || a0 >= A.n_verts || a1 >= A.n_verts || a2 >= A.n_verts)
        return fail(TAC_E_INVALID, "triangle index out of range");
      auto n = cross3(sub3(A.rest_pos + 3 * a1, A.rest_pos + 3 * a0), sub3(A.rest_pos + 3 * a2, A.rest_pos + 3 * a0));
      if (0.5 * std::sqrt(dot3(n, n)) < 1e-12)
        return fail(TAC_E_VALIDATION, "degenerate triangle " + std::to_string(t) + " of affine body " + std::to_string(b));
      tl.push_back({a0, a1, a2});
      tg.push_back(canon_tri(a0 + o, a1 + o, a2 + o));
    }
    body_moments(A.rest_pos, tl, A.density, &H.bvol[b], &H.bmass[b], &H.bs1[3 * b], &H.My[144 * (size_t)b]);
    if (!(H.bvol[b] > 0)) return fail(TAC_E_VALIDATION, "affine body " + std::to_string(b) + " has non-positive volume");
    for (int i = 0; i < A.n_verts; ++i) {
      H.vert_body[o + i] = ns + b;
      H.vert_aff[o + i] = b;
      for (int c = 0; c < 3; ++c) H.vert_xbar[3 * (o + i) + c] = A.rest_pos[3 * i + c];
    }
    sort_canonical(tg);
    for (auto& t : tg) { all_tris.push_back(t); H.tri_body.push_back(ns + b); }
    for (auto& e : tri_edges(tg)) { all_edges.push_back(e); H.edge_body.push_back(ns + b); }
    o += A.n_verts;
  }
  // (M^y)⁻¹ per body by Gauss-Jordan with partial pivoting (SPD 12×12)
  H.MyInv.assign(144 * (size_t)na, 0.0);
  for (int b = 0; b < na; ++b) {
    double A[12][24];
    for (int i = 0; i < 12; ++i)
      for (int j = 0; j < 24; ++j) A[i][j] = j < 12 ? H.My[144 * (size_t)b + 12 * i + j] : (j - 12 == i ? 1.0 : 0.0);
    for (int c = 0; c < 12; ++c) {
      int piv = c;
      for (int r = c + 1; r < 12; ++r) if (std::fabs(A[r][c]) > std::fabs(A[piv][c])) piv = r;
      for (int j = 0; j < 24; ++j) std::swap(A[c][j], A[piv][j]);
      const double d = A[c][c];
      for (int j = 0; j < 24; ++j) A[c][j] /= d;
      for (int r = 0; r < 12; ++r)
        if (r != c) { const double f = A[r][c]; for (int j = 0; j < 24; ++j) A[r][j] -= f * A[c][j]; }
    }
    for (int i = 0; i < 12; ++i)
      for (int j = 0; j < 12; ++j) H.MyInv[144 * (size_t)b + 12 * i + j] = A[i][12 + j];
  }
  H.NT = (int)all_tris.size();
  H.NE = (int)all_edges.size();
  for (auto& t : all_tris) for (int k = 0; k < 3; ++k) H.tris.push_back(t[k]);
  for (auto& e : all_edges) for (int k = 0; k < 2; ++k) H.edges.push_back(e[k]);
  {
    std::vector<char> is_s(H.NVall, 0);
    for (int v : H.tris) is_s[v] = 1;
    for (int v = 0; v < H.NVall; ++v) if (is_s[v]) H.sverts.push_back(v);
    H.NSV = (int)H.sverts.size();
    H.body_sv_ptr.assign(H.NB + 1, 0);
    for (int v : H.sverts) H.body_sv_ptr[H.vert_body[v] + 1]++;
    for (int b = 0; b < H.NB; ++b) H.body_sv_ptr[b + 1] += H.body_sv_ptr[b];
  }
  // rest areas A_v, A_e (1/3 of incident rest triangle areas) and rest edge lengths
  H.A_v.assign(H.NVall, 0.0);
  H.A_e.assign(H.NE, 0.0);
  {
    std::map<std::array<int, 2>, int> eid;
    for (int i = 0; i < H.NE; ++i) eid[all_edges[i]] = i;
    for (auto& t : all_tris) {
      const double* X = H.vert_xbar.data();
      auto n = cross3(sub3(X + 3 * t[1], X + 3 * t[0]), sub3(X + 3 * t[2], X + 3 * t[0]));
      double a = 0.5 * std::sqrt(dot3(n, n));
      if (a < 1e-12) return fail(TAC_E_VALIDATION, "degenerate surface triangle");
      for (int k = 0; k < 3; ++k) {
        H.A_v[t[k]] += a / 3.0;
        int u = t[k], w = t[(k + 1) % 3];
        H.A_e[eid[{std::min(u, w), std::max(u, w)}]] += a / 3.0;
      }
    }
    // hash cell = the median surface edge of the soft pads (the primitives every contact involves), or of
    // all bodies without pads — a finely tessellated rigid body (the C5 tile) must not shrink the cells
    // until every link and table face lands in the broad phase's large-primitive list
    std::vector<double> len, len_soft;
    for (size_t i = 0; i < all_edges.size(); ++i) {
      const auto& e = all_edges[i];
      auto d = sub3(&H.vert_xbar[3 * e[1]], &H.vert_xbar[3 * e[0]]);
      H.elen2.push_back(dot3(d, d));
      len.push_back(std::sqrt(dot3(d, d)));
      if (H.edge_body[i] < ns) len_soft.push_back(len.back());
    }
    std::vector<double>& lsel = len_soft.empty() ? len : len_soft;
    std::sort(lsel.begin(), lsel.end());
    double med = lsel.empty() ? 1.0 : lsel[lsel.size() / 2];
    H.cell = std::max(2.0 * cfg->dhat, med);
  }
  // body-pair mask (reading R8)
  H.allowed.assign((size_t)H.NB * H.NB, 0);
  for (int a = 0; a < H.NB; ++a)
    for (int b = 0; b < H.NB; ++b) {
      bool ok = a != b;
      for (int r = 0; r < 2 && ok; ++r) {
        int s = r ? b : a, t = r ? a : b;
        if (s < ns && sc->soft[s].mount_body >= 0 && ns + sc->soft[s].mount_body == t) ok = false;
      }
      int ka = a < ns ? 0 : sc->affine[a - ns].kind, kb = b < ns ? 0 : sc->affine[b - ns].kind;
      if (ka != 0 && kb != 0) ok = false;
      if (sc->collide && !sc->collide[(size_t)a * H.NB + b]) ok = false;
      H.allowed[(size_t)a * H.NB + b] = ok ? 1 : 0;
    }
  // soft BSR pattern: undirected tet edges, vertex adjacency, element→block gather lists
  {
    std::vector<std::array<int, 2>> se;
    for (int t = 0; t < H.T; ++t)
      for (int a = 0; a < 4; ++a)
        for (int b = a + 1; b < 4; ++b) {
          int u = H.tets[4 * t + a], w = H.tets[4 * t + b];
          se.push_back({std::min(u, w), std::max(u, w)});
        }
    std::sort(se.begin(), se.end());
    se.erase(std::unique(se.begin(), se.end()), se.end());
    H.NEs = (int)se.size();
    std::map<std::array<int, 2>, int> sid;
    for (int i = 0; i < H.NEs; ++i) { sid[se[i]] = i; H.sedge.push_back(se[i][0]); H.sedge.push_back(se[i][1]); }
    std::vector<std::vector<int>> vadj(H.V), vdiag(H.V), eblk(H.NEs);
    for (int i = 0; i < H.NEs; ++i) { vadj[se[i][0]].push_back(2 * i); vadj[se[i][1]].push_back(2 * i + 1); }
    for (int t = 0; t < H.T; ++t)
      for (int a = 0; a < 4; ++a) {
        vdiag[H.tets[4 * t + a]].push_back(4 * t + a);
        for (int b = 0; b < 4; ++b) {
          int u = H.tets[4 * t + a], w = H.tets[4 * t + b];
          if (u < w) eblk[sid[{u, w}]].push_back(16 * t + 4 * a + b);
        }
      }
    auto flat = [](std::vector<std::vector<int>>& L, std::vector<int>& ptr, std::vector<int>& ent) {
      ptr.assign(1, 0);
      for (auto& l : L) { ent.insert(ent.end(), l.begin(), l.end()); ptr.push_back((int)ent.size()); }
    };
    flat(vadj, H.vadj_ptr, H.vadj);
    flat(vdiag, H.vdiag_ptr, H.vdiag);
    flat(eblk, H.eblk_ptr, H.eblk);
    // row-ordered off-diagonal blocks: row v lists its neighbours u ascending; block (v,u) gathers
    // tet entries 16t + 4a + b with local a ↔ v and b ↔ u
    std::vector<std::vector<int>> nb(H.V);
    for (auto& e2 : se) { nb[e2[0]].push_back(e2[1]); nb[e2[1]].push_back(e2[0]); }
    std::map<std::array<int, 2>, int> rid;
    H.rptr.assign(1, 0);
    for (int v = 0; v < H.V; ++v) {
      std::sort(nb[v].begin(), nb[v].end());
      for (int u : nb[v]) {
        rid[{v, u}] = (int)H.rcol.size();
        H.rcol.push_back(u);
        H.rupx.push_back(2 * sid[{std::min(u, v), std::max(u, v)}] + (u < v ? 1 : 0));
        if (u > v) { H.eup.resize(H.NEs); H.eup[sid[{v, u}]] = (int)H.rcol.size() - 1; }
        else { H.elo.resize(H.NEs); H.elo[sid[{u, v}]] = (int)H.rcol.size() - 1; }
      }
      H.rptr.push_back((int)H.rcol.size());
    }
    H.NNZ = (int)H.rcol.size();
    // BSR block of each ordered vertex pair of a soft contact primitive (k_pairs_x's soft-neighbour
    // records): triangles (0,1),(0,2),(1,0),(1,2),(2,0),(2,1); edges (0,1),(1,0)
    auto blk = [&](int v, int u) {
      if (v >= H.V || u >= H.V) return -1;
      for (int q = H.rptr[v]; q < H.rptr[v + 1]; ++q)
        if (H.rcol[q] == u) return q;
      return -1;
    };
    H.tri_blk.assign((size_t)H.NT * 6, -1);
    for (int t = 0; t < H.NT; ++t) {
      const int* tv = &H.tris[3 * t];
      int o = 0;
      for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j)
          if (i != j) H.tri_blk[6 * (size_t)t + o++] = blk(tv[i], tv[j]);
    }
    H.edge_blk.assign((size_t)H.NE * 2, -1);
    for (int e2 = 0; e2 < H.NE; ++e2) {
      H.edge_blk[2 * (size_t)e2] = blk(H.edges[2 * e2], H.edges[2 * e2 + 1]);
      H.edge_blk[2 * (size_t)e2 + 1] = blk(H.edges[2 * e2 + 1], H.edges[2 * e2]);
    }
    std::vector<std::vector<int>> rb(H.NNZ);
    for (int t = 0; t < H.T; ++t)
      for (int a = 0; a < 4; ++a)
        for (int b = 0; b < 4; ++b)
          if (a != b) rb[rid[{H.tets[4 * t + a], H.tets[4 * t + b]}]].push_back(16 * t + 4 * a + b);
    flat(rb, H.rblk_ptr, H.rblk);
  }
  // constraints: ∂⁻G vertices and kinematic bodies
  H.att_of_vert.assign(H.V, -1);
  {
    int off2 = 0;
    for (int p = 0; p < ns; ++p) {
      const tac_soft_desc& S = sc->soft[p];
      if (S.mount_body >= 0)
        for (int i = 0; i < S.n_attached; ++i) {
          int v = S.attached[i];
          if (v < 0 || v >= S.n_verts) return fail(TAC_E_INVALID, "attached vertex out of range");
          const double* X = S.rest_pos + 3 * v;
          const double* t = S.mount_T;
          const double* R = S.mount_T + 3;
          H.att_of_vert[off2 + v] = (int)H.att_vert.size();
          H.att_vert.push_back(off2 + v);
          H.att_body.push_back(S.mount_body);
          for (int r = 0; r < 3; ++r) H.att_local.push_back(t[r] + R[3 * r] * X[0] + R[3 * r + 1] * X[1] + R[3 * r + 2] * X[2]);
        }
      for (int i = 0; i < S.n_coated; ++i) { H.coat_vert.push_back(off2 + S.coated[i]); H.coat_pad.push_back(p); }
      for (int i = 0; i < S.n_markers; ++i) {
        for (int k = 0; k < 3; ++k) { H.mark_tri.push_back(off2 + S.marker_tri[3 * i + k]); H.mark_bary.push_back(S.marker_bary[3 * i + k]); }
        H.mark_pad.push_back(p);
      }
      H.pad_mount.push_back(S.mount_body);
      for (int k = 0; k < 12; ++k) H.pad_T.push_back(S.mount_T[k]);
      off2 += S.n_verts;
    }
  }
  H.NC = (int)H.att_vert.size();
  H.NCOAT = (int)H.coat_vert.size();
  // coated triangles per pad (surface triangles with 3 coated vertices, canonical surface order) and
  // each pad's camera box (rest extent of its coated vertices in the sensor frame, z_ref = max rest z)
  {
    std::vector<int> cidx(H.V, -1);
    for (int i = 0; i < H.NCOAT; ++i) cidx[H.coat_vert[i]] = i;
    H.ct_ptr.assign(1, 0);
    H.coat_ptr.assign(1, 0);
    for (int p = 0; p < ns; ++p) {
      for (auto& t : soft_tris[p]) {
        const int a = cidx[t[0]], b = cidx[t[1]], c = cidx[t[2]];
        if (a >= 0 && b >= 0 && c >= 0) { H.ct_tri.push_back(a); H.ct_tri.push_back(b); H.ct_tri.push_back(c); }
      }
      H.ct_ptr.push_back((int)H.ct_tri.size() / 3);
      int n_c = 0;
      double x0 = 1e300, x1 = -1e300, y0 = 1e300, y1 = -1e300, zr = -1e300;
      for (int i = 0; i < H.NCOAT; ++i)
        if (H.coat_pad[i] == p) {
          ++n_c;
          const double* X = &H.Xrest[3 * (size_t)H.coat_vert[i]];
          x0 = std::min(x0, X[0]); x1 = std::max(x1, X[0]); y0 = std::min(y0, X[1]); y1 = std::max(y1, X[1]); zr = std::max(zr, X[2]);
        }
      H.coat_ptr.push_back(H.coat_ptr.back() + n_c);
      for (double v : {x0, x1, y0, y1, zr}) H.cam.push_back(v);
    }
  }
  H.NMARK = (int)H.mark_pad.size();
  H.kin_of_body.assign(na, -1);
  for (int b = 0; b < na; ++b)
    if (sc->affine[b].kind == TAC_BODY_KINEMATIC) { H.kin_of_body[b] = (int)H.kin_body.size(); H.kin_body.push_back(b); }
  H.NK = (int)H.kin_body.size();
  for (int gv = H.V; gv < H.NVall; ++gv) {
    int b = H.vert_aff[gv];
    if (H.dof_slot[b] >= 0) H.affv_list.push_back(gv);
    if (H.kin_of_body[b] >= 0) H.kin_vlist.push_back(gv);
  }
  if (H.NT + H.NE >= (1 << 29)) return fail(TAC_E_CAPACITY, "too many primitives");
  choose_cluster(H);
  // sliced ELL (SELL-32-σ) for the streamed PCG: rows sorted by length (descending, stable), groups of 32
  // consecutive sorted rows padded to the group's longest row; ell_row maps a slot to its vertex; both
  // blocks of a soft edge are stored.  Symmetric upper-only variants with transposed reads of the lower
  // neighbours were measured slower twice: natural row order (C3 PCG 7.2 -> 7.6 s per 10 steps) and a reverse
  // Cuthill-McKee slot order with window-sorted groups (6.1 -> 12.4 s: the extra loop's registers spill in the
  // SpMV, and even the two-sided path compiled beside it slowed to 9.9 s)
  {
    const int G = (H.V + 31) / 32;
    std::vector<int> order(H.V);
    std::iota(order.begin(), order.end(), 0);
    std::stable_sort(order.begin(), order.end(), [&](int a, int b) {
      return H.rptr[a + 1] - H.rptr[a] > H.rptr[b + 1] - H.rptr[b];
    });
    H.ell_row.assign((size_t)32 * G, -1);
    for (int i = 0; i < H.V; ++i) H.ell_row[i] = order[i];
    H.ell_pos.assign(H.NNZ, 0);
    long long vb = 0;
    int cb = 0;
    for (int g = 0; g < G; ++g) {
      int len = 0;
      for (int l = 0; l < 32; ++l) {
        const int v = H.ell_row[32 * g + l];
        if (v >= 0) len = std::max(len, H.rptr[v + 1] - H.rptr[v]);
      }
      H.ell_len.push_back(len);
      H.ell_vb.push_back(vb);
      H.ell_cb.push_back(cb);
      for (int j = 0; j < len; ++j)
        for (int l = 0; l < 32; ++l) {
          const int v = H.ell_row[32 * g + l];
          const bool real = v >= 0 && H.rptr[v] + j < H.rptr[v + 1];
          H.ell_col.push_back(real ? H.rcol[H.rptr[v] + j] : (v >= 0 ? v : 0));
          if (real) H.ell_pos[H.rptr[v] + j] = vb + (long long)9 * 32 * j + l;
        }
      vb += (long long)9 * 32 * len;
      cb += 32 * len;
    }
    H.ell_total = (size_t)vb;
  }
  return TAC_OK;
}

// ---------------------------------------------------------------------------------------------
// workspace layout
// ---------------------------------------------------------------------------------------------
struct Carver {
  char* base;
  size_t off = 0;
  template <class T>
  T* take(size_t count) {
    off = (off + 255) & ~(size_t)255;
    T* p = base ? reinterpret_cast<T*>(base + off) : nullptr;
    off += count * sizeof(T) + 16;
    return p;
  }
};

struct tac_batch {
  Dev D;
  HostT H;
  int device = 0;
  char* ws = nullptr;
  size_t ws_bytes = 0;
  int* h_flag = nullptr;  // pinned [3]
  void* chain_mem = nullptr;                 // forward-kinematics chain (tac_set_chain)
  void* trace_mem = nullptr;                 // Newton-iteration trace (tac_debug_trace)
  std::vector<EnvCtl> hctl;
  // tracing
  bool prof = false;
  double prof_ms[TAC_NPHASES] = {0};
  long long prof_n[TAC_NPHASES] = {0};
  std::vector<cudaEvent_t> ev_pool;
  std::vector<std::pair<int, int>> pending;  // (phase, event index of start; stop = +1)
  size_t ev_used = 0;
  std::vector<int> it_active;                // per Newton iteration of the last step: envs still active
  std::vector<double> it_ms;                 // and host wall time of the iteration
};

enum { PH_POSITIONS = 0, PH_BROAD_STATIC, PH_NARROW, PH_TETS, PH_PAIRS, PH_ASSEMBLE, PH_PCG, PH_BROAD_SWEPT, PH_CCD,
       PH_LINESEARCH, PH_CONTROL, PH_BEGIN, PH_END, PH_READOUT, PH_SETSTATE, PH_OTHER };
static const char* kPhaseNames[TAC_NPHASES] = {"positions", "broad_static", "narrow", "nh_tets", "barrier_pairs",
                                              "assemble", "pcg", "broad_swept", "accd", "line_search", "control",
                                              "step_begin", "step_end", "readout", "set_state", "other"};

struct ProfScope {
  tac_batch* b; int ph; cudaStream_t st; int idx = -1;
  ProfScope(tac_batch* b_, int ph_, cudaStream_t st_) : b(b_), ph(ph_), st(st_) {
    if (!b->prof) return;
    if (b->ev_used + 2 > b->ev_pool.size()) {
      for (int i = 0; i < 64; ++i) { cudaEvent_t e; cudaEventCreate(&e); b->ev_pool.push_back(e); }
    }
    idx = (int)b->ev_used;
    b->ev_used += 2;
    cudaEventRecord(b->ev_pool[idx], st);
  }
  ~ProfScope() {
    if (idx < 0) return;
    cudaEventRecord(b->ev_pool[idx + 1], st);
    b->pending.push_back({ph, idx});
  }
};

// resolve recorded events (the stream must be synchronised)
static void prof_flush(tac_batch* b) {
  for (auto& pe : b->pending) {
    float ms = 0.f;
    if (cudaEventElapsedTime(&ms, b->ev_pool[pe.second], b->ev_pool[pe.second + 1]) == cudaSuccess) {
      b->prof_ms[pe.first] += ms;
      b->prof_n[pe.first] += 1;
    }
  }
  b->pending.clear();
  b->ev_used = 0;
}
#define PROF(ph) ProfScope _ps_##__LINE__(b, ph, st)

static size_t layout(Carver& C, Dev& D, const HostT& H, int E) {
  auto ti = [&](const std::vector<int>& v) { return C.take<int>(std::max<size_t>(v.size(), 1)); };
  auto td = [&](const std::vector<double>& v) { return C.take<double>(std::max<size_t>(v.size(), 1)); };
  D.tets = ti(H.tets); D.Dmi = td(H.Dmi); D.vol = td(H.vol); D.mu = td(H.mu); D.lam = td(H.lam); D.mass = td(H.mass);
  D.sedge = ti(H.sedge); D.vadj_ptr = ti(H.vadj_ptr); D.vadj = ti(H.vadj); D.vdiag_ptr = ti(H.vdiag_ptr);
  D.vdiag = ti(H.vdiag); D.eblk_ptr = ti(H.eblk_ptr); D.eblk = ti(H.eblk);
  D.rptr = ti(H.rptr); D.rcol = ti(H.rcol); D.rupx = ti(H.rupx); D.eup = ti(H.eup); D.elo = ti(H.elo); D.tri_blk = ti(H.tri_blk); D.edge_blk = ti(H.edge_blk); D.rblk_ptr = ti(H.rblk_ptr); D.rblk = ti(H.rblk);
  D.body_kind = ti(H.body_kind); D.dof_slot = ti(H.dof_slot); D.dof_body = ti(H.dof_body); D.My = td(H.My); D.MyInv = td(H.MyInv);
  D.bmass = td(H.bmass); D.bs1 = td(H.bs1); D.bvol = td(H.bvol); D.bkappa = td(H.bkappa);
  D.vert_body = ti(H.vert_body); D.vert_aff = ti(H.vert_aff); D.vert_xbar = td(H.vert_xbar);
  D.sverts = ti(H.sverts); D.body_sv_ptr = ti(H.body_sv_ptr); D.tris = ti(H.tris); D.tri_body = ti(H.tri_body); D.edges = ti(H.edges);
  D.edge_body = ti(H.edge_body); D.A_v = td(H.A_v); D.A_e = td(H.A_e); D.elen2 = td(H.elen2);
  D.allowed = C.take<unsigned char>(std::max<size_t>(H.allowed.size(), 1));
  D.att_vert = ti(H.att_vert); D.att_body = ti(H.att_body); D.att_local = td(H.att_local);
  D.att_of_vert = ti(H.att_of_vert); D.kin_body = ti(H.kin_body); D.kin_of_body = ti(H.kin_of_body);
  D.affv_list = ti(H.affv_list); D.kin_vlist = ti(H.kin_vlist);
  D.coat_vert = ti(H.coat_vert); D.coat_pad = ti(H.coat_pad); D.mark_tri = ti(H.mark_tri);
  D.mark_bary = td(H.mark_bary); D.mark_pad = ti(H.mark_pad); D.pad_mount = ti(H.pad_mount);
  D.pad_T = td(H.pad_T); D.Xrest = td(H.Xrest);
  D.ct_ptr = ti(H.ct_ptr); D.ct_tri = ti(H.ct_tri); D.coat_ptr = ti(H.coat_ptr); D.cam = td(H.cam);
  {
    auto tl = [&](const std::vector<long long>& v) { return C.take<long long>(std::max<size_t>(v.size(), 1)); };
    D.ell_row = ti(H.ell_row); D.ell_len = ti(H.ell_len); D.ell_vb = tl(H.ell_vb); D.ell_cb = ti(H.ell_cb); D.ell_col = ti(H.ell_col);
    D.ell_pos = tl(H.ell_pos);
  }
  D.cl.eptr = ti(H.cl_eptr); D.cl.edge = ti(H.cl_edge); D.cl.bptr = ti(H.cl_bptr); D.cl.lrptr = ti(H.cl_lrptr);
  D.cl.blk = reinterpret_cast<const int2*>(ti(H.cl_blk));
  const size_t e = (size_t)E, n = H.n;
  D.ctl = C.take<EnvCtl>(e);
  D.q = C.take<double>(e * n); D.qn = C.take<double>(e * n); D.vel = C.take<double>(e * n);
  D.qt = C.take<double>(e * n); D.g = C.take<double>(e * n); D.p = C.take<double>(e * n);
  D.r = C.take<double>(e * n); D.z = C.take<double>(e * n); D.dd = C.take<double>(e * n); D.Ad = C.take<double>(e * n);
  D.ystat = C.take<double>(e * H.NA * 12); D.ystage = C.take<double>(e * H.NA * 12);
  D.s_att = C.take<double>(e * H.NC * 3 + 1); D.lam_att = C.take<double>(e * H.NC * 3 + 1);
  D.s_kin = C.take<double>(e * H.NK * 12 + 1); D.lam_kin = C.take<double>(e * H.NK * 12 + 1);
  D.ykin = C.take<double>(e * H.NK * 12 + 1);
  D.P = C.take<double>(e * H.NVall * 3); D.Pd = C.take<double>(e * H.NVall * 3);
  D.Hd = C.take<double>(e * H.V * 9 + 1);
  D.Ho = C.take<double>(D.asm_ell ? 1 : e * H.NNZ * 9 + 1);   // row-ordered soft blocks (not kept when asm_ell)
  D.Hb = C.take<double>(e * H.ND * 144 + 1); D.Pinv_s = C.take<double>(e * H.V * 9 + 1);
  D.Pinv_b = C.take<double>(e * H.ND * 144 + 1);
  D.Dg_s = C.take<double>(e * H.V * 9 + 1); D.Dg_b = C.take<double>(e * H.ND * 144 + 1);
  const size_t ea = (size_t)D.asm_envs;   // assembly scratch (tets → pairs → assemble) for one chunk of envs
  D.tetbuf = C.take<double>(ea * TETBUF * H.T + 1);
  D.cand_a = C.take<int>(e * D.cand_cap); D.cand_b = C.take<int>(e * D.cand_cap);
  D.ent = C.take<int>(e * D.ent_cap * 2); D.big = C.take<int>(e * BIG_CAP);
  D.tbox = C.take<double>(e * (H.NT + H.NE) * 6);
  D.vref = C.take<double>(e * H.NSV * 6 + 1);
  D.act_info = C.take<int>(e * D.act_cap * 4); D.act_vid = C.take<int>(e * D.act_cap * 4);
  D.act_H = C.take<double>(e * D.res_cap * PH);   // residual pairs' 12×12 only (by residual index)
  D.act_out = C.take<double>(1);
  D.spos = C.take<int>(e * 4 * D.act_cap); D.sout = C.take<double>(e * 4 * D.act_cap * 3);
  D.act_slot = C.take<int>(e * 4 * D.act_cap); D.act_xb = C.take<double>(e * 12 * D.act_cap);
  D.cptr = C.take<int>(e * (H.V + 1)); D.clist = C.take<int>(e * 4 * D.act_cap);
  D.bptr = C.take<int>(e * (H.ND + 1)); D.blist = C.take<int>(e * 4 * D.act_cap);
  D.act_res = C.take<int>(e * D.act_cap); D.res_list = C.take<int>(e * D.act_cap);
  D.rcnt = C.take<int>(e * H.V + 1); D.cpl_ptr = C.take<int>(e * (H.V + 1));
  D.cpl_v = C.take<int>(e * D.cpl_cap + 1); D.cpl_d = C.take<int>(e * D.cpl_cap + 1);
  D.cpl_val = C.take<double>(e * 36 * D.cpl_cap + 1); D.cpl_out = C.take<double>(e * 3 * D.cpl_cap + 1);
  D.srec = C.take<double>(ea * 4 * D.act_cap * SREC); D.snb = C.take<int>(ea * 4 * D.act_cap * 2);
  D.sbody = C.take<int>(ea * 4 * D.act_cap); D.brec = C.take<double>((size_t)D.brec_envs * D.act_cap * 2 * BREC);
  D.bpart = C.take<double>(ea * (size_t)((D.act_cap + 31) / 32) * std::max(H.ND, 1) * BPART);
  D.qcnt = C.take<int>(e * (size_t)(H.NSV + H.NE) + 1);
  D.qtmp = C.take<int>(e * (size_t)(H.NSV + H.NE) * 2 * 32 + 1);
  D.lsl = C.take<int>(e * (size_t)D.cand_cap);
  D.eterm = C.take<double>(e * 8);
  D.out_coat = C.take<double>(e * H.NCOAT * 3 + 1); D.out_mpos = C.take<double>(e * H.NMARK * 3 + 1);
  D.out_mflow = C.take<double>(e * H.NMARK * 3 + 1);
  {
    const size_t fc = D.mu_f > 0.0 ? (size_t)D.act_cap : 1;
    D.fr_info = C.take<int>(e * fc * 4); D.fr_vid = C.take<int>(e * fc * 4); D.fr_slot = C.take<int>(e * fc * 4);
    D.fr_res = C.take<int>(e * fc); D.fr_xb = C.take<double>(e * fc * 12); D.fr_dat = C.take<double>(e * fc * 16);
  }
  D.Hell = C.take<double>(D.ell_groups ? e * D.ell_total : 1);
  D.any_active = C.take<int>(3);
  D.act_list = C.take<int>(6 * e);
  return C.off + 256;
}

static void fill_dims(Dev& D, const HostT& H, const tac_config* cfg, int E, const tac_scene_desc* sc) {
  D.maxrl = 0;
  for (size_t v = 0; v + 1 < H.rptr.size(); ++v) D.maxrl = std::max(D.maxrl, H.rptr[v + 1] - H.rptr[v]);
  D.E = E; D.V = H.V; D.T = H.T; D.NA = H.NA; D.ND = H.ND; D.NVall = H.NVall; D.NSV = H.NSV; D.NT = H.NT;
  D.NE = H.NE; D.NEs = H.NEs; D.NNZ = H.NNZ; D.NC = H.NC; D.NK = H.NK; D.NB = H.NB; D.n = H.n; D.npads = H.npads;
  D.NCOAT = H.NCOAT; D.NMARK = H.NMARK; D.NAV = (int)H.affv_list.size(); D.NKV = (int)H.kin_vlist.size();
  D.cand_cap = std::max(cfg->cand_capacity_per_env, 64);
  D.act_cap = std::max(cfg->active_capacity_per_env, 16);
  D.res_cap = std::max(64, D.act_cap / 4);      // residual (matrix-free) pairs: two soft bodies or two DoF bodies
  D.ent_cap = 16 * (H.NT + H.NE) + 4096;
  // every coupling (v, d) owns at least one soft slot of an active pair, and each (v, d) occurs once
  D.cpl_cap = (int)std::max<long long>(1, std::min<long long>((long long)H.V * H.ND, 4LL * D.act_cap));
  D.max_step = cfg->max_step_rel;
  D.dt = cfg->dt; D.dhat = cfg->dhat; D.kappa = cfg->kappa; D.tolN = cfg->newton_tol_rel; D.tolAL = cfg->al_tol_rel;
  D.eta = cfg->pcg_eta; D.armijo = cfg->armijo_c; D.accd_s = cfg->accd_s; D.rho0 = cfg->al_rho0; D.cell = H.cell;
  D.max_newton = cfg->max_newton; D.max_al = cfg->max_al_rounds; D.max_pcg = cfg->max_pcg;
  D.max_accd = cfg->max_accd_iters; D.mollify = cfg->ee_mollifier; D.hmode = cfg->hessian_mode;
  D.hold_cap = std::max(cfg->hold_cap, 1); D.lm_mu0 = cfg->lm_mu0; D.bp_margin = cfg->bp_margin; D.K = (double)std::max(cfg->ls_expand, 1);
  D.mu_f = cfg->mu_friction; D.eps_v = cfg->eps_v; D.eta_max = cfg->pcg_eta_max;
  // assembly scratch in chunks of asm_envs envs (TAC_ASM_CHUNK, default 1024): the per-tet and per-pair
  // records live only from k_tets / k_pairs* to k_assemble_*, so the Newton loop runs those three phases
  // chunk by chunk over the envs of the iteration and the scratch is sized for one chunk
  {
    static const int chunk = getenv("TAC_ASM_CHUNK") ? std::max(1, atoi(getenv("TAC_ASM_CHUNK"))) : 1024;
    D.asm_envs = std::max(1, std::min(E, chunk));
  }
  D.brec_envs = cfg->hessian_mode == 2 ? 1 : D.asm_envs;
  for (int i = 0; i < 3; ++i) D.grav[i] = sc->gravity[i];
  D.elist = nullptr; D.elist_out = nullptr;
  D.NCT = (int)H.ct_tri.size() / 3; D.maxct = 0; D.maxcv = 0;
  for (int p = 0; p + 1 < (int)H.ct_ptr.size(); ++p) {
    D.maxct = std::max(D.maxct, H.ct_ptr[p + 1] - H.ct_ptr[p]);
    D.maxcv = std::max(D.maxcv, H.coat_ptr[p + 1] - H.coat_ptr[p]);
  }
  D.n_links = 0; D.n_joints = 0;
  D.trace = nullptr; D.trace_env = -1; D.trace_cap = 0; D.trace_n = nullptr;
  {
    static const int tn = getenv("TAC_PCG_TAIL_NEWTON") ? atoi(getenv("TAC_PCG_TAIL_NEWTON")) : 0;
    D.tail_newton = tn;
  }
  D.ell_total = H.ell_total;
  // the streamed PCG (envs that do not fit one SM, or TAC_PCG_RESIDENT=0) reads the soft blocks in the
  // sliced-ELL copy
  {
    const char* res = getenv("TAC_PCG_RESIDENT");
    const bool streamed = (res && atoi(res) == 0) || pcg_r_bytes(D, pcg_r_threads(D.V)) > (size_t)(227 - 4) * 1024;
    D.ell_groups = streamed ? (int)H.ell_len.size() : 0;
    // the assembly writes the soft blocks straight into the sliced-ELL layout (no row-ordered copy, no
    // per-launch conversion in k_pcg) unless a cluster PCG (which reads the row-ordered blocks) may run
    const char* cl = getenv("TAC_PCG_CLUSTER");
    D.asm_ell = D.ell_groups > 0 && !(cl && atoi(cl) > 0) && D.tail_newton == 0 ? 1 : 0;
  }
  D.cl.nc = H.cl_nc; D.cl.rpr = H.cl_rpr; D.cl.threads = H.cl_threads; D.cl.nvt = H.cl_nvt;
  D.cl.nle_max = H.cl_nle_max; D.cl.nlb_max = H.cl_nlb_max; D.cl.cplcap = H.cl_cplcap; D.cl.smem = H.cl_smem_bytes;
}

static tac_status check_cfg(const tac_config* c) {
  if (!(c->max_step_rel > 0) || !(c->dt > 0) || !(c->dhat > 0) || !(c->kappa >= 0) || c->max_newton <= 0 || c->max_al_rounds <= 0 ||
      c->max_pcg <= 0 || !(c->pcg_eta > 0) || !(c->accd_s > 0 && c->accd_s < 1) || c->hessian_mode < 0 ||
      c->hessian_mode > 2 || !(c->lm_mu0 > 0) || !(c->bp_margin >= 0) || c->ls_expand < 1 || (c->ls_expand & (c->ls_expand - 1)) != 0 ||
      !(c->mu_friction >= 0) || !(c->eps_v > 0) ||
      !(c->pcg_eta_max == 0.0 || (c->pcg_eta_max >= c->pcg_eta && c->pcg_eta_max < 1.0)))
    return fail(TAC_E_INVALID, "invalid tac_config");
  if (c->mu_friction > 0 && c->hessian_mode != 2)
    return fail(TAC_E_INVALID, "friction (mu_friction > 0) requires hessian_mode 2");
  return TAC_OK;
}

extern "C" tac_status tac_workspace_size(const tac_scene_desc* scene, int32_t n_envs, const tac_config* cfg, size_t* bytes) {
  if (!scene || !cfg || !bytes || n_envs <= 0) return fail(TAC_E_INVALID, "null argument or n_envs <= 0");
  tac_status s = check_cfg(cfg);
  if (s) return s;
  HostT H;
  s = build_template(scene, cfg, H);
  if (s) return s;
  Dev D{};
  fill_dims(D, H, cfg, n_envs, scene);
  Carver C{nullptr};
  *bytes = layout(C, D, H, n_envs);
  return TAC_OK;
}

template <class T>
static cudaError_t up(const T* dst, const std::vector<T>& v, cudaStream_t s) {
  if (v.empty()) return cudaSuccess;
  return cudaMemcpyAsync((void*)dst, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice, s);
}

extern "C" tac_status tac_batch_create(const tac_scene_desc* scene, int32_t n_envs, const tac_config* cfg, int32_t device,
                                       void* workspace, size_t ws_bytes, void* stream, tac_batch** out) {
  if (!scene || !cfg || !out || !workspace || n_envs <= 0) return fail(TAC_E_INVALID, "null argument or n_envs <= 0");
  if (((uintptr_t)workspace) & 255) return fail(TAC_E_WORKSPACE, "workspace must be 256-byte aligned");
  tac_status s = check_cfg(cfg);
  if (s) return s;
  DevGuard _dg(device);
  if (_dg.err != cudaSuccess) return fail(TAC_E_CUDA, std::string("cudaSetDevice: ") + cudaGetErrorString(_dg.err));
  tac_batch* b = new tac_batch();
  b->device = device;
  s = build_template(scene, cfg, b->H);
  if (s) { delete b; return s; }
  fill_dims(b->D, b->H, cfg, n_envs, scene);
  Carver C{(char*)workspace};
  size_t need = layout(C, b->D, b->H, n_envs);
  if (need > ws_bytes) {
    delete b;
    return fail(TAC_E_WORKSPACE, "workspace too small: need " + std::to_string(need) + " bytes");
  }
  b->ws = (char*)workspace;
  b->ws_bytes = ws_bytes;
  cudaStream_t st = (cudaStream_t)stream;
  const HostT& H = b->H;
  Dev& D = b->D;
  cudaError_t e = init_tables();
  // host-buffer calls (tac_step_schedule with host pointers) stage through stream-ordered allocations;
  // keep freed pool memory mapped so repeated calls do not re-map it
  if (e == cudaSuccess) {
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
      uint64_t thr = UINT64_MAX;
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    }
  }
  if (e == cudaSuccess) e = cudaMemsetAsync(workspace, 0, need, st);
#define UP(f) if (e == cudaSuccess) e = up(D.f, H.f, st)
  UP(tets); UP(Dmi); UP(vol); UP(mu); UP(lam); UP(mass); UP(sedge); UP(vadj_ptr); UP(vadj); UP(vdiag_ptr); UP(vdiag);
  UP(eblk_ptr); UP(eblk); UP(rptr); UP(rcol); UP(rupx); UP(eup); UP(elo); UP(tri_blk); UP(edge_blk); UP(rblk_ptr); UP(rblk); UP(body_kind); UP(dof_slot); UP(dof_body); UP(My); UP(MyInv); UP(bmass); UP(bs1); UP(bvol); UP(bkappa);
  UP(vert_body); UP(vert_aff); UP(vert_xbar); UP(sverts); UP(body_sv_ptr); UP(tris); UP(tri_body); UP(edges); UP(edge_body);
  UP(A_v); UP(A_e); UP(elen2); UP(allowed); UP(att_vert); UP(att_body); UP(att_local); UP(att_of_vert);
  UP(kin_body); UP(kin_of_body); UP(affv_list); UP(kin_vlist); UP(coat_vert); UP(coat_pad); UP(mark_tri);
  UP(mark_bary); UP(mark_pad); UP(pad_mount); UP(pad_T); UP(Xrest); UP(ct_ptr); UP(ct_tri); UP(coat_ptr); UP(cam);
#undef UP
  if (e == cudaSuccess) e = up(D.ell_row, H.ell_row, st);
  if (e == cudaSuccess) e = up(D.ell_len, H.ell_len, st);
  if (e == cudaSuccess) e = up(D.ell_vb, H.ell_vb, st);
  if (e == cudaSuccess) e = up(D.ell_cb, H.ell_cb, st);
  if (e == cudaSuccess) e = up(D.ell_col, H.ell_col, st);
  if (e == cudaSuccess) e = up(D.ell_pos, H.ell_pos, st);
  if (e == cudaSuccess) e = up(D.cl.eptr, H.cl_eptr, st);
  if (e == cudaSuccess) e = up(D.cl.edge, H.cl_edge, st);
  if (e == cudaSuccess) e = up(D.cl.bptr, H.cl_bptr, st);
  if (e == cudaSuccess) e = up(D.cl.lrptr, H.cl_lrptr, st);
  if (e == cudaSuccess) e = up(reinterpret_cast<const int*>(D.cl.blk), H.cl_blk, st);
  b->hctl.assign(n_envs, EnvCtl{});
  for (auto& c : b->hctl) { c.phase = PHASE_IDLE; c.disabled = 1; c.status = ENV_DISABLED; c.L = 1.0; c.rho = cfg->al_rho0; c.Keff = 1.0; }
  if (e == cudaSuccess) e = cudaMemcpyAsync(D.ctl, b->hctl.data(), sizeof(EnvCtl) * n_envs, cudaMemcpyHostToDevice, st);
  if (e == cudaSuccess) e = cudaMallocHost(&b->h_flag, 3 * sizeof(int));
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  if (e != cudaSuccess) { delete b; return fail(TAC_E_CUDA, std::string("create: ") + cudaGetErrorString(e)); }
  *out = b;
  return TAC_OK;
}

extern "C" tac_status tac_batch_destroy(tac_batch* b) {
  if (!b) return TAC_OK;
  DevGuard _dg(b->device);
  if (b->h_flag) cudaFreeHost(b->h_flag);
  if (b->chain_mem) cudaFree(b->chain_mem);
  if (b->trace_mem) cudaFree(b->trace_mem);
  for (auto e : b->ev_pool) cudaEventDestroy(e);
  delete b;
  return TAC_OK;
}

extern "C" tac_status tac_batch_dims(const tac_batch* b, int32_t dims[10]) {
  if (!b || !dims) return fail(TAC_E_INVALID, "null argument");
  const HostT& H = b->H;
  int d[10] = {H.V, H.T, H.NA, H.NK, H.NCOAT, H.NMARK, H.n, H.NVall, H.NT, H.NE};
  for (int i = 0; i < 10; ++i) dims[i] = d[i];
  return TAC_OK;
}

static tac_status check_range(tac_batch* b, int env0, int n) {
  if (!b) return fail(TAC_E_INVALID, "null batch");
  if (env0 < 0 || n <= 0 || env0 + n > b->D.E) return fail(TAC_E_INVALID, "env range out of bounds");
  return TAC_OK;
}

static tac_status pull_ctl(tac_batch* b, cudaStream_t st) {
  CUDA_TRY(cudaMemcpyAsync(b->hctl.data(), b->D.ctl, sizeof(EnvCtl) * b->D.E, cudaMemcpyDeviceToHost, st));
  CUDA_TRY(cudaStreamSynchronize(st));
  return TAC_OK;
}

static tac_status write_status(tac_batch* b, int env0, int n, uint8_t* out, cudaStream_t st) {
  if (!out) return TAC_OK;
  std::vector<uint8_t> s(n);
  for (int i = 0; i < n; ++i) s[i] = (uint8_t)b->hctl[env0 + i].status;
  CUDA_TRY(cudaMemcpyAsync(out, s.data(), n, cudaMemcpyDefault, st));
  CUDA_TRY(cudaStreamSynchronize(st));
  return TAC_OK;
}

extern "C" tac_status tac_set_state(tac_batch* b, int32_t env0, int32_t n, const double* x, const double* xdot,
                                    const double* y, const double* ydot, uint8_t* env_status, void* stream) {
  tac_status s = check_range(b, env0, n);
  if (s) return s;
  ON_DEVICE(b);
  if ((!x && b->D.V) || !y) return fail(TAC_E_INVALID, "x and y are required");
  cudaStream_t st = (cudaStream_t)stream;
  Dev& D = b->D;
  const size_t pitch = (size_t)D.n * sizeof(double), w = (size_t)3 * D.V * sizeof(double);
  if (D.V) {
    CUDA_TRY(cudaMemcpy2DAsync(D.q + (size_t)env0 * D.n, pitch, x, w, w, n, cudaMemcpyDefault, st));
    if (xdot) CUDA_TRY(cudaMemcpy2DAsync(D.vel + (size_t)env0 * D.n, pitch, xdot, w, w, n, cudaMemcpyDefault, st));
    else CUDA_TRY(cudaMemset2DAsync(D.vel + (size_t)env0 * D.n, pitch, 0, w, n, st));
  }
  const size_t ybytes = (size_t)n * D.NA * 12 * sizeof(double);
  CUDA_TRY(cudaMemcpyAsync(D.ystage + (size_t)env0 * D.NA * 12, y, ybytes, cudaMemcpyDefault, st));
  launch_scatter_y(D, env0, n, 0, st);
  if (ydot) {
    CUDA_TRY(cudaMemcpyAsync(D.ystage + (size_t)env0 * D.NA * 12, ydot, ybytes, cudaMemcpyDefault, st));
    launch_scatter_y(D, env0, n, 1, st);
  } else {
    launch_scatter_y(D, env0, n, 2, st);
  }
  launch_positions(D, env0, n, 0, 1, st);
  launch_broad(D, env0, n, 0, 1, st);
  launch_validate(D, env0, n, st);
  CUDA_TRY(cudaGetLastError());
  s = pull_ctl(b, st);
  if (s) return s;
  return write_status(b, env0, n, env_status, st);
}

static bool is_device_ptr(const void* p);

extern "C" tac_status tac_set_chain(tac_batch* b, const tac_chain_desc* ch) {
  if (!b || !ch || ch->n_links <= 0 || ch->n_links > 64 || ch->n_joints < 0 || !ch->parent || !ch->origin || !ch->axis ||
      !ch->joint || !ch->body || !ch->kin_body)
    return fail(TAC_E_INVALID, "bad chain description");
  ON_DEVICE(b);
  Dev& D = b->D;
  const HostT& H = b->H;
  const int nl = ch->n_links;
  std::vector<int> kin(nl);
  for (int i = 0; i < nl; ++i) {
    if (ch->parent[i] >= i || ch->parent[i] < -1) return fail(TAC_E_INVALID, "chain parents must precede their links");
    if (ch->joint[i] >= ch->n_joints || ch->joint[i] < -1) return fail(TAC_E_INVALID, "joint index out of range");
    const int kb = ch->kin_body[i];
    if (kb < 0 || kb >= H.NA || H.kin_of_body[kb] < 0) return fail(TAC_E_INVALID, "chain link drives a non-kinematic body");
    kin[i] = H.kin_of_body[kb];
    const double* a = ch->axis + 3 * i;
    if (ch->joint[i] >= 0 && std::fabs(a[0] * a[0] + a[1] * a[1] + a[2] * a[2] - 1.0) > 1e-12)
      return fail(TAC_E_INVALID, "joint axis must be a unit vector");
  }
  const size_t bytes = sizeof(int) * 3 * nl + sizeof(double) * (27 * (size_t)nl + 12 * (size_t)D.E) + 256;
  if (b->chain_mem) { cudaFree(b->chain_mem); b->chain_mem = nullptr; }
  CUDA_TRY(cudaMalloc(&b->chain_mem, bytes));
  char* m = (char*)b->chain_mem;
  double* origin = (double*)m; double* axis = origin + 12 * nl; double* body = axis + 3 * nl; double* base = body + 12 * nl;
  int* parent = (int*)(base + 12 * (size_t)D.E); int* joint = parent + nl; int* kinb = joint + nl;
  CUDA_TRY(cudaMemcpy(origin, ch->origin, sizeof(double) * 12 * nl, cudaMemcpyHostToDevice));
  CUDA_TRY(cudaMemcpy(axis, ch->axis, sizeof(double) * 3 * nl, cudaMemcpyHostToDevice));
  CUDA_TRY(cudaMemcpy(body, ch->body, sizeof(double) * 12 * nl, cudaMemcpyHostToDevice));
  CUDA_TRY(cudaMemcpy(parent, ch->parent, sizeof(int) * nl, cudaMemcpyHostToDevice));
  CUDA_TRY(cudaMemcpy(joint, ch->joint, sizeof(int) * nl, cudaMemcpyHostToDevice));
  CUDA_TRY(cudaMemcpy(kinb, kin.data(), sizeof(int) * nl, cudaMemcpyHostToDevice));
  std::vector<double> ident((size_t)12 * D.E, 0.0);
  for (int e = 0; e < D.E; ++e) { ident[12 * e + 3] = 1.0; ident[12 * e + 7] = 1.0; ident[12 * e + 11] = 1.0; }
  CUDA_TRY(cudaMemcpy(base, ident.data(), sizeof(double) * 12 * D.E, cudaMemcpyHostToDevice));
  D.n_links = nl; D.n_joints = ch->n_joints;
  D.ch_parent = parent; D.ch_origin = origin; D.ch_axis = axis; D.ch_joint = joint; D.ch_body = body; D.ch_kin = kinb;
  D.ch_base = base;
  return TAC_OK;
}

extern "C" tac_status tac_set_joint_targets(tac_batch* b, int32_t env0, int32_t n, const double* base, const double* q,
                                           void* stream) {
  tac_status s = check_range(b, env0, n);
  if (s) return s;
  if (!b->chain_mem) return fail(TAC_E_INVALID, "no chain: call tac_set_chain first");
  if (!q && b->D.n_joints > 0) return fail(TAC_E_INVALID, "q is required");
  ON_DEVICE(b);
  Dev& D = b->D;
  cudaStream_t st = (cudaStream_t)stream;
  if (base) CUDA_TRY(cudaMemcpyAsync(D.ch_base + (size_t)env0 * 12, base, sizeof(double) * 12 * n, cudaMemcpyDefault, st));
  const double* dq = q;
  void* tmp = nullptr;
  if (q && !is_device_ptr(q)) {
    CUDA_TRY(cudaMallocAsync(&tmp, sizeof(double) * (size_t)n * std::max(D.n_joints, 1), st));
    CUDA_TRY(cudaMemcpyAsync(tmp, q, sizeof(double) * (size_t)n * D.n_joints, cudaMemcpyHostToDevice, st));
    dq = (const double*)tmp;
  }
  launch_fk(D, env0, n, dq, st);
  CUDA_TRY(cudaGetLastError());
  if (tmp) CUDA_TRY(cudaFreeAsync(tmp, st));
  return TAC_OK;
}

extern "C" tac_status tac_get_targets(tac_batch* b, int32_t env0, int32_t n, double* y_kin, void* stream) {
  tac_status s = check_range(b, env0, n);
  if (s) return s;
  if (!y_kin) return fail(TAC_E_INVALID, "y_kin is null");
  ON_DEVICE(b);
  cudaStream_t st = (cudaStream_t)stream;
  if (b->D.NK) CUDA_TRY(cudaMemcpyAsync(y_kin, b->D.ykin + (size_t)env0 * b->D.NK * 12, sizeof(double) * 12 * b->D.NK * n,
                                        cudaMemcpyDefault, st));
  CUDA_TRY(cudaStreamSynchronize(st));
  return TAC_OK;
}

extern "C" tac_status tac_set_targets(tac_batch* b, int32_t env0, int32_t n, const double* y_kin, void* stream) {
  tac_status s = check_range(b, env0, n);
  if (s) return s;
  ON_DEVICE(b);
  if (b->D.NK == 0) return TAC_OK;
  if (!y_kin) return fail(TAC_E_INVALID, "y_kin is null");
  CUDA_TRY(cudaMemcpyAsync(b->D.ykin + (size_t)env0 * b->D.NK * 12, y_kin, (size_t)n * b->D.NK * 12 * sizeof(double),
                           cudaMemcpyDefault, (cudaStream_t)stream));
  return TAC_OK;
}

static double now_ms() {
  return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

struct Sched {
  const double* sched;
  int nsteps;
  double *oc, *om, *of;
};

// Newton iterations until every env of [env0, env0+ne) converged or failed.  After the first
// iteration the kernels run over the compacted list of envs k_control left active (grid = their
// count, read back with the one 4-byte flag per iteration), so the tail of a lockstep step — a few
// slow envs — does not pay for thousands of early-exiting CTAs per launch.  TAC_COMPACT=0 disables it.
static tac_status newton_loop(tac_batch* b, int env0, int ne, cudaStream_t st, const Sched* sc = nullptr) {
  Dev& D = b->D;
  static const int compact = getenv("TAC_COMPACT") ? atoi(getenv("TAC_COMPACT")) : 1;
  b->it_active.clear();
  b->it_ms.clear();
  double t0 = now_ms();
  { PROF(PH_POSITIONS); launch_positions(D, env0, ne, 0, 0, st); }
  { PROF(PH_BROAD_STATIC); launch_broad(D, env0, ne, 0, 0, st); }
  const long max_it = (long)(D.max_newton + 2) * (sc ? sc->nsteps : 1);
  Dev L = D;                              // per-iteration launch copy (active-env list)
  int n_run = ne, e0 = env0, n_tail = 0, n_bulk = ne;
  const bool split = compact && D.tail_newton > 0 && tail_pcg_available(D);
  if (!split) L.tail_newton = 0;
  for (long it = 0; it < max_it; ++it) {
    const size_t nb = (size_t)((it + 1) & 1) * 3 * D.E;
    L.elist_out = compact ? D.act_list + nb : nullptr;
    { PROF(PH_POSITIONS); launch_positions(L, e0, n_run, 0, 0, st); }
    { PROF(PH_NARROW); launch_narrow(L, e0, n_run, 0, st); }
    for (int c0 = 0; c0 < n_run; c0 += D.asm_envs) {   // assembly scratch chunks (see fill_dims)
      Dev Lc = L;
      if (Lc.elist) Lc.elist += c0;
      const int m = std::min(D.asm_envs, n_run - c0);
      { PROF(PH_TETS); launch_tets(Lc, e0 + c0, m, 0, st); }
      { PROF(PH_PAIRS); launch_pairs(Lc, e0 + c0, m, 0, st); }
      { PROF(PH_ASSEMBLE); launch_assemble(Lc, e0 + c0, m, 0, st); }
    }
    if (split && it > 0) {                   // per env: tail envs on the cluster kernel, the rest default
      const int* cur = L.elist;
      Dev Lt = L, Lb = L;
      Lt.elist = cur + D.E;
      Lb.elist = cur + 2 * (size_t)D.E;
      if (n_bulk) { PROF(PH_PCG); launch_pcg(Lb, 0, n_bulk, 0, st); }
      if (n_tail) { PROF(PH_PCG); launch_cluster_pcg(Lt, 0, n_tail, 0, st); }
    } else {
      PROF(PH_PCG);
      launch_pcg(L, e0, n_run, 0, st);
    }
    { PROF(PH_POSITIONS); launch_positions(L, e0, n_run, 1, 0, st); }
    { PROF(PH_BROAD_SWEPT); launch_broad(L, e0, n_run, 1, 0, st); }
    { PROF(PH_CCD); launch_ccd(L, e0, n_run, 0, st); }
    { PROF(PH_LINESEARCH); launch_linesearch(L, e0, n_run, st); }
    CUDA_TRY(cudaMemsetAsync(D.any_active, 0, 3 * sizeof(int), st));
    { PROF(PH_CONTROL); launch_control(L, e0, n_run, st); }
    if (sc) { PROF(PH_END); launch_advance(L, e0, n_run, sc->sched, sc->nsteps, sc->oc, sc->om, sc->of, st); }
    CUDA_TRY(cudaMemcpyAsync(b->h_flag, D.any_active, 3 * sizeof(int), cudaMemcpyDeviceToHost, st));
    CUDA_TRY(cudaStreamSynchronize(st));
    CUDA_TRY(cudaGetLastError());
    if (b->prof) prof_flush(b);
    double t1 = now_ms();
    b->it_active.push_back(*b->h_flag);
    b->it_ms.push_back(t1 - t0);
    t0 = t1;
    if (!*b->h_flag) break;
    if (compact) {
      L.elist = D.act_list + nb;
      n_run = b->h_flag[0];
      n_tail = b->h_flag[1];
      n_bulk = b->h_flag[2];
      e0 = 0;
    }
  }
  return TAC_OK;
}

extern "C" tac_status tac_step(tac_batch* b, int32_t n_steps, uint8_t* env_status, void* stream) {
  if (!b || n_steps < 0) return fail(TAC_E_INVALID, "bad arguments");
  ON_DEVICE(b);
  cudaStream_t st = (cudaStream_t)stream;
  Dev& D = b->D;
  bool any_failed = false;
  for (int s = 0; s < n_steps; ++s) {
    { PROF(PH_BEGIN); launch_begin(D, 0, D.E, st); }
    tac_status r = newton_loop(b, 0, D.E, st);
    if (r) return r;
    { PROF(PH_END); launch_end(D, 0, D.E, st); }
    CUDA_TRY(cudaGetLastError());
  }
  tac_status r = pull_ctl(b, st);
  if (b->prof) prof_flush(b);
  if (r) return r;
  for (auto& c : b->hctl)
    if (c.phase == PHASE_FAILED) any_failed = true;
  r = write_status(b, 0, D.E, env_status, st);
  if (r) return r;
  return any_failed ? fail(TAC_E_ENV_FAILED, "one or more envs failed (see env_status)") : TAC_OK;
}

static bool is_device_ptr(const void* p) {  // (declared above)
  if (!p) return false;
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) { cudaGetLastError(); return false; }
  return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

extern "C" tac_status tac_step_schedule(tac_batch* b, int32_t n_steps, const double* y_kin_sched, double* coated_disp,
                                        double* marker_pos, double* marker_flow, uint8_t* env_status, void* stream) {
  if (!b || n_steps <= 0) return fail(TAC_E_INVALID, "bad arguments");
  ON_DEVICE(b);
  if (b->D.NK > 0 && !y_kin_sched) return fail(TAC_E_INVALID, "y_kin_sched is required when the scene has kinematic bodies");
  cudaStream_t st = (cudaStream_t)stream;
  Dev& D = b->D;
  const size_t sbytes = (size_t)n_steps * D.E * D.NK * 12 * sizeof(double);
  const size_t cbytes = (size_t)n_steps * D.E * D.NCOAT * 3 * sizeof(double);
  const size_t mbytes = (size_t)n_steps * D.E * D.NMARK * 3 * sizeof(double);
  // stage host buffers through stream-ordered device allocations
  double* dsched = D.ykin;
  void* tmp_s = nullptr;
  if (D.NK > 0) {
    if (is_device_ptr(y_kin_sched)) dsched = const_cast<double*>(y_kin_sched);
    else {
      CUDA_TRY(cudaMallocAsync(&tmp_s, sbytes, st));
      CUDA_TRY(cudaMemcpyAsync(tmp_s, y_kin_sched, sbytes, cudaMemcpyDefault, st));
      dsched = (double*)tmp_s;
    }
  }
  const bool want_out = coated_disp && marker_pos && marker_flow;
  double *oc = nullptr, *om = nullptr, *of = nullptr;
  void* tmp_o = nullptr;
  const bool out_dev = want_out && is_device_ptr(coated_disp);
  if (want_out) {
    if (out_dev) { oc = coated_disp; om = marker_pos; of = marker_flow; }
    else {
      CUDA_TRY(cudaMallocAsync(&tmp_o, cbytes + 2 * mbytes + 64, st));
      oc = (double*)tmp_o;
      om = (double*)((char*)tmp_o + cbytes);
      of = (double*)((char*)tmp_o + cbytes + mbytes);
    }
  }
  { PROF(PH_BEGIN); launch_begin_sched(D, 0, D.E, dsched, st); }
  Sched sc{dsched, n_steps, oc, om, of};
  tac_status r = newton_loop(b, 0, D.E, st, &sc);
  if (r) return r;
  CUDA_TRY(cudaGetLastError());
  if (want_out && !out_dev) {
    CUDA_TRY(cudaMemcpyAsync(coated_disp, oc, cbytes, cudaMemcpyDefault, st));
    CUDA_TRY(cudaMemcpyAsync(marker_pos, om, mbytes, cudaMemcpyDefault, st));
    CUDA_TRY(cudaMemcpyAsync(marker_flow, of, mbytes, cudaMemcpyDefault, st));
  }
  if (tmp_s) CUDA_TRY(cudaFreeAsync(tmp_s, st));
  if (tmp_o) CUDA_TRY(cudaFreeAsync(tmp_o, st));
  r = pull_ctl(b, st);
  if (r) return r;
  if (b->prof) prof_flush(b);
  bool any_failed = false;
  for (auto& c : b->hctl)
    if (c.phase == PHASE_FAILED) any_failed = true;
  r = write_status(b, 0, D.E, env_status, st);
  if (r) return r;
  return any_failed ? fail(TAC_E_ENV_FAILED, "one or more envs failed (see env_status)") : TAC_OK;
}

extern "C" tac_status tac_get_state(tac_batch* b, int32_t env0, int32_t n, double* x, double* xdot, double* y,
                                    double* ydot, void* stream) {
  tac_status s = check_range(b, env0, n);
  if (s) return s;
  ON_DEVICE(b);
  cudaStream_t st = (cudaStream_t)stream;
  Dev& D = b->D;
  const size_t pitch = (size_t)D.n * sizeof(double), w = (size_t)3 * D.V * sizeof(double);
  if (x && D.V) CUDA_TRY(cudaMemcpy2DAsync(x, w, D.q + (size_t)env0 * D.n, pitch, w, n, cudaMemcpyDefault, st));
  if (xdot && D.V) CUDA_TRY(cudaMemcpy2DAsync(xdot, w, D.vel + (size_t)env0 * D.n, pitch, w, n, cudaMemcpyDefault, st));
  const size_t ybytes = (size_t)n * D.NA * 12 * sizeof(double);
  if (y) {
    launch_gather_y(D, env0, n, 0, st);
    CUDA_TRY(cudaMemcpyAsync(y, D.ystage + (size_t)env0 * D.NA * 12, ybytes, cudaMemcpyDefault, st));
  }
  if (ydot) {
    launch_gather_y(D, env0, n, 1, st);
    CUDA_TRY(cudaMemcpyAsync(ydot, D.ystage + (size_t)env0 * D.NA * 12, ybytes, cudaMemcpyDefault, st));
  }
  CUDA_TRY(cudaStreamSynchronize(st));
  return TAC_OK;
}

extern "C" tac_status tac_get_gel_deformation(tac_batch* b, int32_t env0, int32_t n, double* coated_disp,
                                              double* marker_pos, double* marker_flow, void* stream) {
  tac_status s = check_range(b, env0, n);
  if (s) return s;
  ON_DEVICE(b);
  cudaStream_t st = (cudaStream_t)stream;
  Dev& D = b->D;
  { PROF(PH_READOUT); launch_readout(D, env0, n, st); }
  if (coated_disp && D.NCOAT)
    CUDA_TRY(cudaMemcpyAsync(coated_disp, D.out_coat + (size_t)env0 * D.NCOAT * 3, (size_t)n * D.NCOAT * 3 * 8, cudaMemcpyDefault, st));
  if (marker_pos && D.NMARK)
    CUDA_TRY(cudaMemcpyAsync(marker_pos, D.out_mpos + (size_t)env0 * D.NMARK * 3, (size_t)n * D.NMARK * 3 * 8, cudaMemcpyDefault, st));
  if (marker_flow && D.NMARK)
    CUDA_TRY(cudaMemcpyAsync(marker_flow, D.out_mflow + (size_t)env0 * D.NMARK * 3, (size_t)n * D.NMARK * 3 * 8, cudaMemcpyDefault, st));
  CUDA_TRY(cudaStreamSynchronize(st));
  if (b->prof) prof_flush(b);
  return TAC_OK;
}

extern "C" tac_status tac_get_depth_maps(tac_batch* b, int32_t env0, int32_t n, int32_t H, int32_t W, double* depth,
                                         double* normal, void* stream) {
  tac_status s = check_range(b, env0, n);
  if (s) return s;
  if (H < 2 || W < 2 || (long long)H * W > (1LL << 24)) return fail(TAC_E_INVALID, "depth map size must be 2..16M pixels");
  if (!depth && !normal) return TAC_OK;
  ON_DEVICE(b);
  Dev& D = b->D;
  if (D.npads == 0 || D.NCT == 0) return fail(TAC_E_INVALID, "no coated triangles");
  cudaStream_t st = (cudaStream_t)stream;
  const size_t npx = (size_t)n * D.npads * H * W;
  double *dd = depth, *dn = normal;
  void* tmp = nullptr;
  const bool hd = depth && !is_device_ptr(depth), hn = normal && !is_device_ptr(normal);
  if (hd || hn) {
    CUDA_TRY(cudaMallocAsync(&tmp, npx * 8 * ((hd ? 1 : 0) + (hn ? 3 : 0)) + 64, st));
    double* t = (double*)tmp;
    if (hd) { dd = t; t += npx; }
    if (hn) dn = t;
  }
  { PROF(PH_READOUT); launch_depth(D, env0, n, H, W, dd, dn, st); }
  CUDA_TRY(cudaGetLastError());
  if (hd) CUDA_TRY(cudaMemcpyAsync(depth, dd, npx * 8, cudaMemcpyDeviceToHost, st));
  if (hn) CUDA_TRY(cudaMemcpyAsync(normal, dn, npx * 24, cudaMemcpyDeviceToHost, st));
  if (tmp) CUDA_TRY(cudaFreeAsync(tmp, st));
  CUDA_TRY(cudaStreamSynchronize(st));
  if (b->prof) prof_flush(b);
  return TAC_OK;
}

extern "C" tac_status tac_get_stats(tac_batch* b, tac_env_stats* out, void* stream) {
  if (!b || !out) return fail(TAC_E_INVALID, "null argument");
  ON_DEVICE(b);
  tac_status s = pull_ctl(b, (cudaStream_t)stream);
  if (s) return s;
  for (int e = 0; e < b->D.E; ++e) {
    const EnvCtl& c = b->hctl[e];
    out[e].status = c.status; out[e].newton_iters = c.newton; out[e].pcg_iters = c.pcg; out[e].ls_backtracks = c.ls_bt;
    out[e].n_active = c.n_act - c.n_fr; out[e].al_rounds = c.al_rounds; out[e].n_candidates = c.ncand;
    out[e].alpha_min = c.alpha_min; out[e].energy = c.energy; out[e].constraint_residual = c.residual;
    out[e].pcg_iters_total = c.pcg_total; out[e].pcg_alg_bytes_total = c.pcg_bytes;
    out[e].diag[0] = c.alpha_ccd; out[e].diag[1] = c.gp; out[e].diag[2] = c.ls_E0; out[e].diag[3] = c.ls_E1;
    out[e].min_dist = c.min_d2 < b->D.dhat * b->D.dhat ? std::sqrt(c.min_d2) : HUGE_VAL;
    out[e].n_residual = c.n_res; out[e].n_couplings = c.n_cpl;
    out[e].lm_mu = c.mu_used;
    out[e].n_friction = c.n_fr; out[e].capacity_flags = c.cap_seen;
  }
  return TAC_OK;
}

extern "C" tac_status tac_profile_enable(tac_batch* b, int32_t enable) {
  if (!b) return fail(TAC_E_INVALID, "null batch");
  b->prof = enable != 0;
  return TAC_OK;
}

extern "C" tac_status tac_profile_read(tac_batch* b, double* ms, int64_t* launches, int32_t reset) {
  if (!b) return fail(TAC_E_INVALID, "null batch");
  for (int i = 0; i < TAC_NPHASES; ++i) {
    if (ms) ms[i] = b->prof_ms[i];
    if (launches) launches[i] = b->prof_n[i];
    if (reset) { b->prof_ms[i] = 0; b->prof_n[i] = 0; }
  }
  return TAC_OK;
}

extern "C" tac_status tac_profile_iterations(tac_batch* b, int32_t* active, double* ms, int32_t cap, int32_t* n) {
  if (!b) return fail(TAC_E_INVALID, "null batch");
  int m = (int)b->it_active.size();
  if (n) *n = m;
  for (int i = 0; i < std::min(m, cap); ++i) {
    if (active) active[i] = b->it_active[i];
    if (ms) ms[i] = b->it_ms[i];
  }
  return TAC_OK;
}

extern "C" const char* tac_profile_phase_name(int32_t phase) {
  return (phase >= 0 && phase < TAC_NPHASES) ? kPhaseNames[phase] : "";
}

// ---------------------------------------------------------------------------------------------
// parity hooks: evaluate one env at a given (x, y) without changing its state
// ---------------------------------------------------------------------------------------------
struct DebugScope {
  tac_batch* b; int e; cudaStream_t st;
  std::vector<double> q, vel, ystat;
  EnvCtl ctl;
  bool ok = false;
};

static tac_status dbg_enter(DebugScope& S, const double* x, const double* y, const double* lam_att,
                            const double* lam_kin, double rho, int exact = 0) {
  tac_batch* b = S.b;
  Dev& D = b->D;
  const int e = S.e;
  S.q.resize(D.n); S.vel.resize(D.n); S.ystat.resize((size_t)D.NA * 12);
  CUDA_TRY(cudaMemcpyAsync(S.q.data(), D.q + (size_t)e * D.n, D.n * 8, cudaMemcpyDeviceToHost, S.st));
  CUDA_TRY(cudaMemcpyAsync(S.vel.data(), D.vel + (size_t)e * D.n, D.n * 8, cudaMemcpyDeviceToHost, S.st));
  CUDA_TRY(cudaMemcpyAsync(S.ystat.data(), D.ystat + (size_t)e * D.NA * 12, D.NA * 96, cudaMemcpyDeviceToHost, S.st));
  CUDA_TRY(cudaMemcpyAsync(&S.ctl, D.ctl + e, sizeof(EnvCtl), cudaMemcpyDeviceToHost, S.st));
  CUDA_TRY(cudaStreamSynchronize(S.st));
  S.ok = true;
  // x̃ = q + Δt v and targets from the env's current state (k_begin), then overwrite the iterate
  EnvCtl c = S.ctl;
  c.disabled = 0;
  CUDA_TRY(cudaMemcpyAsync(D.ctl + e, &c, sizeof(EnvCtl), cudaMemcpyHostToDevice, S.st));
  launch_begin(D, e, 1, S.st);
  if (D.mu_f > 0.0) {                 // lagged friction frozen at the env's state xⁿ (as at a step start)
    launch_positions(D, e, 1, 0, 1, S.st);
    launch_broad(D, e, 1, 0, 1, S.st);
    launch_narrow(D, e, 1, 1, S.st);
  }
  if (D.V) CUDA_TRY(cudaMemcpyAsync(D.q + (size_t)e * D.n, x, (size_t)3 * D.V * 8, cudaMemcpyHostToDevice, S.st));
  CUDA_TRY(cudaMemcpyAsync(D.ystage + (size_t)e * D.NA * 12, y, (size_t)D.NA * 96, cudaMemcpyHostToDevice, S.st));
  launch_scatter_y(D, e, 1, 0, S.st);
  if (lam_att && D.NC) CUDA_TRY(cudaMemcpyAsync(D.lam_att + (size_t)e * D.NC * 3, lam_att, (size_t)D.NC * 24, cudaMemcpyHostToDevice, S.st));
  if (lam_kin && D.NK) CUDA_TRY(cudaMemcpyAsync(D.lam_kin + (size_t)e * D.NK * 12, lam_kin, (size_t)D.NK * 96, cudaMemcpyHostToDevice, S.st));
  if (rho > 0) CUDA_TRY(cudaMemcpyAsync(&D.ctl[e].rho, &rho, sizeof(double), cudaMemcpyHostToDevice, S.st));
  static int flag[2] = {0, 1};
  CUDA_TRY(cudaMemcpyAsync(&D.ctl[e].exact, &flag[exact ? 1 : 0], sizeof(int), cudaMemcpyHostToDevice, S.st));
  static const double zero = 0.0;
  CUDA_TRY(cudaMemcpyAsync(&D.ctl[e].mu, &zero, sizeof(double), cudaMemcpyHostToDevice, S.st));
  CUDA_TRY(cudaStreamSynchronize(S.st));
  return TAC_OK;
}

static tac_status dbg_leave(DebugScope& S) {
  if (!S.ok) return TAC_OK;
  Dev& D = S.b->D;
  const int e = S.e;
  CUDA_TRY(cudaMemcpyAsync(D.q + (size_t)e * D.n, S.q.data(), D.n * 8, cudaMemcpyHostToDevice, S.st));
  CUDA_TRY(cudaMemcpyAsync(D.vel + (size_t)e * D.n, S.vel.data(), D.n * 8, cudaMemcpyHostToDevice, S.st));
  CUDA_TRY(cudaMemcpyAsync(D.ystat + (size_t)e * D.NA * 12, S.ystat.data(), D.NA * 96, cudaMemcpyHostToDevice, S.st));
  S.ctl.bp_ref = 0;                         // the debug build replaced the candidate list
  S.ctl.bp_valid = 0;
  CUDA_TRY(cudaMemcpyAsync(D.ctl + e, &S.ctl, sizeof(EnvCtl), cudaMemcpyHostToDevice, S.st));
  CUDA_TRY(cudaStreamSynchronize(S.st));
  return TAC_OK;
}

static tac_status dbg_assemble(tac_batch* b, int e, cudaStream_t st) {
  Dev& D = b->D;
  launch_positions(D, e, 1, 0, 1, st);
  launch_broad(D, e, 1, 0, 1, st);
  launch_narrow(D, e, 1, 1, st);
  launch_tets(D, e, 1, 1, st);
  launch_pairs(D, e, 1, 1, st);
  launch_assemble(D, e, 1, 1, st);
  CUDA_TRY(cudaGetLastError());
  return TAC_OK;
}

#define DBG_CHECK(b, env)                                                        \
  if (!(b) || (env) < 0 || (env) >= (b)->D.E) return fail(TAC_E_INVALID, "bad env"); \
  if (!x || !y) return fail(TAC_E_INVALID, "x and y are required");                   \
  ON_DEVICE(b)

extern "C" tac_status tac_debug_eval(tac_batch* b, int32_t env, const double* x, const double* y, const double* lam_att,
                                     const double* lam_kin, double rho, int32_t exact_hessian, const double* v_in,
                                     double* e_terms, double* grad, double* hv, void* stream) {
  DBG_CHECK(b, env);
  if (b->D.mu_f > 0.0 && !exact_hessian) return fail(TAC_E_INVALID, "friction batches evaluate the exact Hessian only");
  DebugScope S{b, env, (cudaStream_t)stream};
  tac_status s = dbg_enter(S, x, y, lam_att, lam_kin, rho, exact_hessian);
  Dev& D = b->D;
  if (!s) s = dbg_assemble(b, env, S.st);
  if (!s && e_terms) {
    launch_energy(D, env, 1, 0.0, S.st);
    double t[8];
    cudaMemcpyAsync(t, D.eterm + (size_t)env * 8, 64, cudaMemcpyDeviceToHost, S.st);
    cudaStreamSynchronize(S.st);
    for (int i = 0; i < 7; ++i) e_terms[i] = t[i];
  }
  if (!s && grad) {
    cudaMemcpyAsync(grad, D.g + (size_t)env * D.n, D.n * 8, cudaMemcpyDeviceToHost, S.st);
    cudaStreamSynchronize(S.st);
  }
  if (!s && hv && v_in) {
    cudaMemcpyAsync(D.dd + (size_t)env * D.n, v_in, D.n * 8, cudaMemcpyHostToDevice, S.st);
    launch_spmv(D, env, D.dd + (size_t)env * D.n, D.Ad + (size_t)env * D.n, S.st);
    cudaMemcpyAsync(hv, D.Ad + (size_t)env * D.n, D.n * 8, cudaMemcpyDeviceToHost, S.st);
    if (cudaStreamSynchronize(S.st) != cudaSuccess) s = fail(TAC_E_CUDA, "debug spmv failed");
  }
  if (!s && cudaGetLastError() != cudaSuccess) s = fail(TAC_E_CUDA, "debug eval kernel failed");
  tac_status s2 = dbg_leave(S);
  return s ? s : s2;
}

static tac_status copy_pairs(tac_batch* b, int env, bool active, int32_t* pairs, int32_t cap, int32_t* count, cudaStream_t st) {
  Dev& D = b->D;
  EnvCtl c;
  CUDA_TRY(cudaMemcpyAsync(&c, D.ctl + env, sizeof(EnvCtl), cudaMemcpyDeviceToHost, st));
  CUDA_TRY(cudaStreamSynchronize(st));
  if (c.overflow) return fail(TAC_E_CAPACITY, "pair capacity exceeded");
  int n = active ? c.n_act - c.n_fr : c.ncand;         // barrier pairs (friction entries follow them)
  if (count) *count = n;
  if (!pairs) return TAC_OK;
  int m = std::min(n, cap);
  if (active) {
    std::vector<int> info((size_t)4 * std::max(m, 1));
    CUDA_TRY(cudaMemcpy(info.data(), D.act_info + (size_t)env * D.act_cap * 4, (size_t)m * 16, cudaMemcpyDeviceToHost));
    for (int i = 0; i < m; ++i) { pairs[3 * i] = info[4 * i]; pairs[3 * i + 1] = info[4 * i + 2]; pairs[3 * i + 2] = info[4 * i + 3]; }
  } else {
    std::vector<int> a(std::max(m, 1)), bb(std::max(m, 1));
    CUDA_TRY(cudaMemcpy(a.data(), D.cand_a + (size_t)env * D.cand_cap, (size_t)m * 4, cudaMemcpyDeviceToHost));
    CUDA_TRY(cudaMemcpy(bb.data(), D.cand_b + (size_t)env * D.cand_cap, (size_t)m * 4, cudaMemcpyDeviceToHost));
    for (int i = 0; i < m; ++i) { pairs[3 * i] = (a[i] >> 30) & 1; pairs[3 * i + 1] = a[i] & ((1 << 30) - 1); pairs[3 * i + 2] = bb[i]; }
  }
  return TAC_OK;
}

extern "C" tac_status tac_debug_active_pairs(tac_batch* b, int32_t env, const double* x, const double* y, int32_t* pairs,
                                             int32_t cap, int32_t* count, void* stream) {
  DBG_CHECK(b, env);
  DebugScope S{b, env, (cudaStream_t)stream};
  tac_status s = dbg_enter(S, x, y, nullptr, nullptr, 0.0);
  Dev& D = b->D;
  if (!s) {
    launch_positions(D, env, 1, 0, 1, S.st);
    launch_broad(D, env, 1, 0, 1, S.st);
    launch_narrow(D, env, 1, 1, S.st);
    s = copy_pairs(b, env, true, pairs, cap, count, S.st);
  }
  tac_status s2 = dbg_leave(S);
  return s ? s : s2;
}

static tac_status dbg_set_p(tac_batch* b, int env, const double* p, cudaStream_t st) {
  Dev& D = b->D;
  if (p) CUDA_TRY(cudaMemcpyAsync(D.p + (size_t)env * D.n, p, D.n * 8, cudaMemcpyHostToDevice, st));
  else CUDA_TRY(cudaMemsetAsync(D.p + (size_t)env * D.n, 0, D.n * 8, st));
  return TAC_OK;
}

extern "C" tac_status tac_debug_candidates(tac_batch* b, int32_t env, const double* x, const double* y, const double* p,
                                           int32_t* pairs, int32_t cap, int32_t* count, void* stream) {
  DBG_CHECK(b, env);
  DebugScope S{b, env, (cudaStream_t)stream};
  tac_status s = dbg_enter(S, x, y, nullptr, nullptr, 0.0);
  Dev& D = b->D;
  if (!s) s = dbg_set_p(b, env, p, S.st);
  if (!s) {
    launch_positions(D, env, 1, 1, 1, S.st);
    launch_broad(D, env, 1, p ? 1 : 0, 1, S.st);
    s = copy_pairs(b, env, false, pairs, cap, count, S.st);
  }
  tac_status s2 = dbg_leave(S);
  return s ? s : s2;
}

extern "C" tac_status tac_debug_accd(tac_batch* b, int32_t env, const double* x, const double* y, const double* p,
                                     double* alpha, void* stream) {
  DBG_CHECK(b, env);
  if (!p || !alpha) return fail(TAC_E_INVALID, "p and alpha are required");
  DebugScope S{b, env, (cudaStream_t)stream};
  tac_status s = dbg_enter(S, x, y, nullptr, nullptr, 0.0);
  Dev& D = b->D;
  if (!s) s = dbg_set_p(b, env, p, S.st);
  if (!s) {
    launch_positions(D, env, 1, 1, 1, S.st);
    launch_broad(D, env, 1, 1, 1, S.st);
    launch_ccd(D, env, 1, 1, S.st);
    EnvCtl c;
    cudaMemcpyAsync(&c, D.ctl + env, sizeof(EnvCtl), cudaMemcpyDeviceToHost, S.st);
    if (cudaStreamSynchronize(S.st) != cudaSuccess) s = fail(TAC_E_CUDA, "debug accd failed");
    else *alpha = c.Keff * c.alpha_ccd;
  }
  tac_status s2 = dbg_leave(S);
  return s ? s : s2;
}

extern "C" tac_status tac_debug_pcg(tac_batch* b, int32_t env, const double* x, const double* y, int32_t exact_hessian,
                                    double mu, double* p, int32_t* iters, double* mu_used, void* stream) {
  DBG_CHECK(b, env);
  if (mu < 0) return fail(TAC_E_INVALID, "mu must be >= 0");
  if (b->D.mu_f > 0.0 && !exact_hessian) return fail(TAC_E_INVALID, "friction batches solve with the exact Hessian only");
  DebugScope S{b, env, (cudaStream_t)stream};
  tac_status s = dbg_enter(S, x, y, nullptr, nullptr, 0.0, exact_hessian);
  Dev& D = b->D;
  if (!s) CUDA_TRY(cudaMemcpyAsync(&D.ctl[env].mu, &mu, sizeof(double), cudaMemcpyHostToDevice, S.st));
  if (!s) s = dbg_assemble(b, env, S.st);
  if (!s) {
    launch_pcg(D, env, 1, 1, S.st);
    EnvCtl c;
    cudaMemcpyAsync(&c, D.ctl + env, sizeof(EnvCtl), cudaMemcpyDeviceToHost, S.st);
    if (p) cudaMemcpyAsync(p, D.p + (size_t)env * D.n, D.n * 8, cudaMemcpyDeviceToHost, S.st);
    if (cudaStreamSynchronize(S.st) != cudaSuccess) s = fail(TAC_E_CUDA, "debug pcg failed");
    else {
      if (iters) *iters = c.pcg;
      if (mu_used) *mu_used = c.mu_used;
    }
  }
  tac_status s2 = dbg_leave(S);
  return s ? s : s2;
}

extern "C" tac_status tac_debug_inject_fault(tac_batch* b, int32_t env, int32_t status, void* stream) {
  if (!b || env < 0 || env >= b->D.E) return fail(TAC_E_INVALID, "bad env");
  if (status < TAC_ENV_NEWTON_STALL || status > TAC_ENV_NONFINITE) return fail(TAC_E_INVALID, "status must be 1..4");
  ON_DEVICE(b);
  cudaStream_t st = (cudaStream_t)stream;
  int v = status;
  CUDA_TRY(cudaMemcpyAsync(&b->D.ctl[env].fault, &v, sizeof(int), cudaMemcpyHostToDevice, st));
  CUDA_TRY(cudaStreamSynchronize(st));
  return TAC_OK;
}

extern "C" tac_status tac_debug_trace(tac_batch* b, int32_t env, int32_t cap, double* rows, int32_t* n) {
  if (!b || env >= b->D.E || cap < 0) return fail(TAC_E_INVALID, "bad arguments");
  ON_DEVICE(b);
  Dev& D = b->D;
  if (env >= 0 && cap > 0 && !rows) {                    // start tracing env: (re)allocate and reset
    if (b->trace_mem) { cudaFree(b->trace_mem); b->trace_mem = nullptr; }
    CUDA_TRY(cudaMalloc(&b->trace_mem, sizeof(double) * 10 * (size_t)cap + 16));
    D.trace = (double*)b->trace_mem;
    D.trace_n = (int*)(D.trace + 10 * (size_t)cap);
    D.trace_cap = cap;
    D.trace_env = env;
    CUDA_TRY(cudaMemset(D.trace_n, 0, sizeof(int)));
    return TAC_OK;
  }
  if (env < 0) { D.trace_env = -1; return TAC_OK; }       // stop tracing
  if (!D.trace) return fail(TAC_E_INVALID, "no trace");
  int m = 0;
  CUDA_TRY(cudaDeviceSynchronize());
  CUDA_TRY(cudaMemcpy(&m, D.trace_n, sizeof(int), cudaMemcpyDeviceToHost));
  if (n) *n = m;
  if (rows) CUDA_TRY(cudaMemcpy(rows, D.trace, sizeof(double) * 10 * std::min(m, cap), cudaMemcpyDeviceToHost));
  return TAC_OK;
}

extern "C" const char* tac_pcg_kernel_name(const tac_batch* b) {
  if (!b) return "";
  DevGuard _dg(b->device);
  return pcg_path_name(pcg_path(b->D));
}
