// impl.cuh — device-side batch layout shared by the kernels and the host API.
//
// Layout in HBM (one workspace, caller-owned):
//   template (read-only, shared by all envs, L2-resident): tets, D_m⁻¹, V_e, Lamé, lumped masses,
//     soft BSR pattern + element→block gather lists, affine M^y / moments, contact primitives,
//     rest areas, body-pair mask, constraint lists, readout tables.
//   per env (env-major; every per-env array is [E][...] contiguous per env):
//     DoF vectors q, qⁿ, v, q̃, g, p, r, z, d, Hd (n = 3V + 12·ND doubles each), vertex positions,
//     BSR values (3×3 per soft vertex and per soft edge), dense 12×12 per body, block-Jacobi
//     inverses, per-tet gradient+Hessian (SoA [90][T]), candidate and active pair lists with their
//     12×12 projected Hessians, broad-phase hash entries.
#pragma once
#include "common.cuh"

namespace tac {

constexpr int NTHREADS = 256;
constexpr int NBUCKET = 4096;      // spatial-hash buckets per env (shared memory)
constexpr int MAXCELLS = 32;       // targets spanning more cells go to the per-env "big" list
constexpr int BIG_CAP = 8192;
constexpr int TETBUF = 90;         // 12 gradient + 78 packed Hessian
constexpr int PH = 78;
constexpr int SREC = 66;          // per soft slot record: g 3 | H_ss 9 | coupling 36 | soft neighbours 18
constexpr int BREC = 90;          // per (pair, body) record: packed JᵀHJ 78 | Jᵀg 12
constexpr int BPART = 12 + 2 * PH; // per (32-pair chunk, body) partial: Jᵀg 12 | condensed JᵀHJ 78 | residual JᵀHJ 78

enum { PHASE_ACTIVE = 0, PHASE_DONE = 1, PHASE_FAILED = 2, PHASE_IDLE = 3 };
enum { ENV_OK = 0, ENV_NEWTON_STALL = 1, ENV_AL_INFEASIBLE = 2, ENV_CAPACITY = 3, ENV_NONFINITE = 4,
       ENV_BAD_STATE = 5, ENV_DISABLED = 6 };

struct EnvCtl {
  int phase, status, inner_conv, newton, pcg, ls_bt, al_rounds, n_act, ncand, overflow;
  int disabled, pad_;
  int exact, hold, nfail, xfail;   // exact-Hessian-first control (reading R14b)
  int bp_ref, bp_valid;            // reusable candidate list state (reading R11b)
  int step, pad2_;                 // step index in a scheduled multi-step call
  int n_res, n_cpl;                // residual pairs (matrix-free in the SpMV) and soft–body couplings
  long long pcg_total;
  double pcg_bytes;
  double Keff;
  double mu;              // LM shift for the next solve (hessian_mode 2)
  double ls_E0, ls_E1;
  double alpha_ccd, alpha_min, rho, r_prev, L, energy, residual, gp, pnorm, alpha;
  double min_d2;          // min squared primitive distance over the candidates classified by the last narrow phase
  double mu_used;         // LM shift of the last solve (hessian_mode 2)
  int fault, pad3_;       // test-only fault injection (tac_debug_inject_fault): env status forced at k_control
  int n_fr, fr_frozen;    // lagged friction pairs of this step (appended after the barrier pairs), frozen at xⁿ
  int cap_seen, cap_need; // capacity overflows seen since batch creation (bits: 1 candidates, 2 big-target list,
                          // 4 hash entries, 8 active pairs) and the largest candidate count requested
  double ew_rz0, ew_eta;  // relaxed PCG tolerance (R24): r₀ᵀz₀ and η of the last accepted solve of this step
  int ew_has, pad4_;      // 1 once this step has an accepted solve
};

// ---- env-resident cluster PCG (pcg_cluster.cuh): plan built on the host from the soft BSR pattern ----
constexpr int CL_MAX_THREADS = 384;
constexpr int CL_MAX_NC = 16;
struct ClSmem {            // carve of the dynamic shared memory (offsets in bytes, host and device agree)
  size_t U, u, hd, ub, pbody, wpart, hb, blk, rptr, cpp, cpld, cval, red, end;
};
__host__ __device__ inline size_t cl_align(size_t x) { return (x + 15) & ~(size_t)15; }
__host__ __device__ inline ClSmem cl_smem(int rpr, int nle, int nlb, int nd, int nw, int cplcap) {
  ClSmem s;
  size_t o = 0;
  s.U = o; o = cl_align(o + 72 * (size_t)nle);
  s.u = o; o = cl_align(o + 24 * (size_t)rpr);
  s.hd = o; o = cl_align(o + 72 * (size_t)rpr);
  s.ub = o; o = cl_align(o + 96 * (size_t)nd);
  s.pbody = o; o = cl_align(o + 96 * (size_t)nd);
  s.wpart = o; o = cl_align(o + 96 * (size_t)nd * nw);
  s.hb = o; o = cl_align(o + 2 * 1152 * (size_t)nd);      // bodies: (H_b + μM^y) and its block-Jacobi inverse
  s.blk = o; o = cl_align(o + 8 * (size_t)nlb);
  s.rptr = o; o = cl_align(o + 4 * (size_t)(rpr + 1));
  s.cpp = o; o = cl_align(o + 4 * (size_t)(rpr + 1));
  s.cpld = o; o = cl_align(o + 4 * (size_t)cplcap);
  s.cval = o; o = cl_align(o + 288 * (size_t)cplcap);
  s.red = o; o = cl_align(o + 8 * (8 + 2 * 32));
  s.end = o;
  return s;
}

// host-built plan (template data, shared by all envs of the batch)
struct ClPlan {
  int nc, rpr, threads, nvt, nle_max, nlb_max, cplcap;
  size_t smem;
  const int* eptr;      // [nc+1] local-edge list offsets
  const int* edge;      // local edges → global soft edge id
  const int* bptr;      // [nc+1] local-block list offsets
  const int* lrptr;     // [nc][rpr+1] block-row pointers relative to the rank's list
  const int2* blk;      // {2·local edge + transposed, rank << 16 | local row of the column vertex}
};


struct Dev {
  // ---- dims ----
  int NNZ;                // off-diagonal soft blocks in row order (2·NEs)
  int maxrl;              // longest soft BSR row (blocks)
  int E, V, T, NA, ND, NVall, NSV, NT, NE, NEs, NC, NK, NB, n, npads, NCOAT, NMARK;
  int cand_cap, act_cap, ent_cap, cpl_cap, res_cap;
  // ---- config ----
  double max_step;     // relative step cap (reading R17c)
  double dt, dhat, kappa, tolN, tolAL, eta, armijo, accd_s, rho0, cell;
  int max_newton, max_al, max_pcg, max_accd, mollify, hmode, hold_cap;
  double K;                 // line-search expansion bound (reading R17b)
  double lm_mu0;
  double bp_margin;         // δ of the reusable candidate list (0 = rebuild every iteration)
  double mu_f, eps_v;       // lagged friction: μ (0 = off) and ε_v
  double eta_max;           // relaxed PCG tolerance (R24): 0 = fixed η
  double grav[3];
  // ---- template ----
  const int* tets;        // [T][4]
  const double* Dmi;      // [T][9]
  const double* vol;      // [T]
  const double* mu;       // [T]
  const double* lam;      // [T]
  const double* mass;     // [V]
  const int* sedge;       // [NEs][2] soft edges (i<j) = off-diagonal BSR blocks
  const int* vadj_ptr;    // [V+1]
  const int* vadj;        // entries 2*edge + (v is the edge's second vertex)
  const int* vdiag_ptr;   // [V+1]
  const int* vdiag;       // entries 4*tet + local
  const int* eblk_ptr;    // [NEs+1]
  const int* eblk;        // entries 16*tet + 4*a + b (local a ↔ edge.i, b ↔ edge.j)
  const int* rptr;        // [V+1] row-ordered symmetric BSR
  const int* rcol;        // [NNZ] column (neighbour vertex)
  const int* tri_blk;     // [NT][6] BSR index of (v_i, v_j) of a soft triangle, ordered pairs (0,1),(0,2),(1,0),(1,2),(2,0),(2,1)
  const int* edge_blk;    // [NE][2] BSR index of (v0, v1), (v1, v0) of a soft edge
  const int* eup;         // [NEs] row-ordered index of each soft edge's upper block (i < j, row i)
  const int* elo;         // [NEs] row-ordered index of each soft edge's lower block (row j, the transpose)
  const int* rupx;        // [NNZ] 2·(soft edge id) + 1 if the block is the transpose of the edge's upper block
  const int* rblk_ptr;    // [NNZ+1]
  const int* rblk;        // entries 16*tet + 4*a + b (a ↔ row, b ↔ column)
  const int* body_kind;   // [NA]
  const int* dof_slot;    // [NA] (-1 static)
  const int* dof_body;    // [ND]
  const double* My;       // [NA][144]
  const double* MyInv;    // [NA][144] (M^y)⁻¹ (convergence test under an LM shift, reading R14d)
  const double* bmass;    // [NA]
  const double* bs1;      // [NA][3]
  const double* bvol;     // [NA]
  const double* bkappa;   // [NA]
  const int* vert_body;   // [NVall] global body id (pads first)
  const int* vert_aff;    // [NVall] affine body or -1
  const double* vert_xbar;// [NVall][3]
  const int* sverts;      // [NSV]
  const int* body_sv_ptr; // [NB+1] range of each body's surface vertices in sverts
  const int* tris;        // [NT][3]
  const int* tri_body;    // [NT]
  const int* edges;       // [NE][2]
  const int* edge_body;   // [NE]
  const double* A_v;      // [NVall]
  const double* A_e;      // [NE]
  const double* elen2;    // [NE]
  const unsigned char* allowed;  // [NB][NB]
  const int* att_vert;    // [NC]
  const int* att_body;    // [NC]
  const double* att_local;// [NC][3]
  const int* att_of_vert; // [V] (-1 if free)
  const int* kin_body;    // [NK]
  const int* kin_of_body; // [NA] (-1)
  const int* affv_list;   // vertices of dof bodies (for embedded norms): [NAV]
  int NAV;
  const int* kin_vlist;   // vertices of kinematic bodies [NKV]
  int NKV;
  // readout
  const int* coat_vert;   // [NCOAT] soft vertex id
  const int* coat_pad;    // [NCOAT]
  const int* mark_tri;    // [NMARK][3] soft vertex ids
  const double* mark_bary;// [NMARK][3]
  const int* mark_pad;    // [NMARK]
  const int* pad_mount;   // [npads]
  const double* pad_T;    // [npads][12]
  const double* Xrest;    // [V][3] pad-frame rest positions
  // depth maps (tac_get_depth_maps): coated triangles per pad (indices into the coat list), camera box
  const int* ct_ptr;      // [npads+1]
  const int* ct_tri;      // [NCT][3] indices into coat_vert
  const int* coat_ptr;    // [npads+1] range of each pad's coated vertices in coat_vert
  const double* cam;      // [npads][5] x0, x1, y0, y1, z_ref (sensor frame, rest)
  int NCT, maxct, maxcv;
  // ---- per env ----
  EnvCtl* ctl;            // [E]
  double *q, *qn, *vel, *qt, *g, *p, *r, *z, *dd, *Ad;   // [E][n]
  double* ystat;          // [E][NA][12]
  double* ystage;         // [E][NA][12] staging for host I/O
  double *s_att, *lam_att;// [E][NC][3]
  double *s_kin, *lam_kin, *ykin;  // [E][NK][12]
  double *P, *Pd;         // [E][NVall][3] positions at q, displacement of p
  double *Hd, *Ho;        // [E][V][9], [E][NNZ][9] (row-ordered off-diagonal blocks)
  double *Hb;             // [E][ND][144]
  double *Pinv_s, *Pinv_b;// [E][V][9], [E][ND][144]
  double *Dg_s, *Dg_b;    // raw block-Jacobi diagonal blocks (before the LM shift and inversion)
  double* tetbuf;         // [asm_envs][90][T]
  int *cand_a, *cand_b;   // [E][cand_cap] (cand_a bit 30 = EE)
  int* ent;               // [E][ent_cap][2]
  int* big;               // [E][BIG_CAP]
  int* qcnt;              // [E][NSV+NE] broad-phase query counts → segment offsets
  int* qtmp;              // [E][NSV+NE][2][32] per-query candidate slots of the broad phase
  int* lsl;               // [E][cand_cap] line-search candidate list (energy_terms lmode 1/2)
  double* tbox;           // [E][NT+NE][6] raw target boxes (broad-phase cache)
  double* vref;           // [E][NSV][6] reference boxes of surface vertices at the last build
  int* act_info;          // [E][act_cap][4] (kind, type, a, b)
  int* act_vid;           // [E][act_cap][4]
  double* act_H;          // [E][res_cap][78] packed 12×12 of the residual (matrix-free) pairs, by residual index
  double* act_out;        // [E][act_cap][12] (unused)
  int* act_slot;          // [E][4*act_cap] slot code: soft vertex ≥ 0, DoF body d → −1−d, static → INT_MIN
  double* act_xb;         // [E][4*act_cap][3] rest position x̄ of affine slots
  int* spos;              // [E][4*act_cap] slot → position in the soft output list (-1: not soft)
  double* sout;           // [E][4*act_cap][3] per-slot soft outputs of the pair SpMV pass
  // contact condensation: each active pair whose slots are soft vertices adjacent in the
  // BSR pattern and at most one DoF body is folded at assembly into the soft BSR blocks (soft–soft),
  // the body's 12×12 (J_sᵀH_stJ_t), and one 3×12 coupling block C_vd = Σ H_st J_t per (soft vertex v,
  // body d); the remaining "residual" pairs stay matrix-free (12×12 through J) in the SpMV
  int* act_res;           // [E][act_cap] 0 = condensed pair, else residual index + 1 (its act_H slot)
  int* res_list;          // [E][act_cap] residual pair indices (ascending)
  int* rcnt;              // [E][V] residual slots of v = first rcnt[v] entries of its clist range
  int* cpl_ptr;           // [E][V+1] coupling blocks of soft vertex v (ascending body)
  int* cpl_v;             // [E][cpl_cap]
  int* cpl_d;             // [E][cpl_cap]
  double* cpl_val;        // [E][36][cpl_cap] SoA, C_vd row-major 3×12
  double* cpl_out;        // [E][cpl_cap][3] SpMV scratch: C_vd x_d
  double* srec;           // [E][4*act_cap][SREC] per soft slot, vertex-sorted position (k_pairs)
  int* snb;               // [E][4*act_cap][2] BSR block of each soft neighbour record (-1 none)
  int* sbody;             // [E][4*act_cap] DoF body of the coupling record (-1 none / residual)
  double* brec;           // [brec_envs][act_cap][2][BREC] per (pair, DoF body) records (k_pairs, projected envs)
  int asm_ell;            // 1: the assembly writes the soft off-diagonal blocks into Hell (sliced ELL) only
  int asm_envs;           // env slots of the assembly scratch (tetbuf, srec/snb/sbody, bpart, brec): one chunk
  int brec_envs;          // E for hessian modes 0/1; 1 for mode 2, where only the one-env debug evaluations
                          // of the projected Hessian use these records
  double* bpart;          // [E][ceil(act_cap/32)][ND][BPART] per 32-pair chunk body partial sums
  int* cptr;              // [E][V+1] soft contribution lists
  int* clist;             // [E][4*act_cap]
  int* bptr;              // [E][ND+1] body contribution lists
  int* blist;             // [E][4*act_cap]
  double* eterm;          // [E][8]
  double* out_coat;       // [E][NCOAT][3]
  double* out_mpos;       // [E][NMARK][3]
  double* out_mflow;      // [E][NMARK][3]
  // lagged friction (reading R20): the active pairs at xⁿ, frozen once per step, appended after the
  // barrier pairs of every Newton iteration's active list (kind + 2)
  int* fr_info;           // [E][act_cap][4] (kind, type, a, b) at xⁿ
  int* fr_vid;            // [E][act_cap][4]
  int* fr_slot;           // [E][act_cap][4]
  int* fr_res;            // [E][act_cap]
  double* fr_xb;          // [E][act_cap][12]
  double* fr_dat;         // [E][act_cap][16] Δt²μλⁿ | n̂ 3 | Γ weights of slots 1..3 | yⁿ_j = x_j − x_0 (j = 1..3) 9
  // forward kinematics chain (tac_set_chain; separate device allocation owned by the batch)
  int n_links, n_joints;
  const int* ch_parent; const double* ch_origin; const double* ch_axis; const int* ch_joint; const double* ch_body;
  const int* ch_kin;      // kinematic index (0..NK-1) of each link's body
  double* ch_base;        // [E][12] base pose per env
  // Newton-iteration trace of one env (tac_debug_trace; test/diagnostic only): rows of
  // [newton, pcg iterations, μ used, ‖p‖_emb,∞, ‖M⁻¹g‖_emb,∞, gᵀp, α, E(q), E(q+αp), line-search backtracks]
  double* trace;          // [trace_cap][10]
  int trace_env, trace_cap;
  int* trace_n;
  int* any_active;        // [3] envs still active after k_control: total, tail (≥ tail_newton), bulk
  int tail_newton;        // > 0: envs with at least this many Newton iterations in the step solve with the
                          // cluster-resident PCG (k_pcg_cl), the others with the default kernel
  int* act_list;          // [2][3][E] compacted active-env lists (all, tail, bulk), double-buffered by iteration parity
  const int* elist;       // per launch: env list of this launch (nullptr = env0 + blockIdx)
  int* elist_out;         // per launch: list k_control / k_advance append the next iteration's active envs to
  ClPlan cl;              // cluster PCG plan (cl.nc = 0: not available for this template)
  // warp-interleaved (sliced ELL) copy of the row-ordered soft blocks for the streamed PCG: rows in groups
  // of 32 (one warp), group g padded to its longest row; value (slot j, component c, lane l) of group g at
  // ell_vb[g] + (9j + c)·32 + l, its column at ell_cb[g] + 32j + l — every warp load is 256 contiguous bytes
  int ell_groups;         // ⌈V/32⌉ (0: no ELL copy)
  size_t ell_total;       // doubles per env
  const int* ell_row;     // [32·groups] vertex of each slot (rows sorted by length, −1 padding)
  const int* ell_len;     // [groups] slots of the group
  const long long* ell_vb;// [groups] value base (doubles)
  const int* ell_cb;      // [groups] column base
  const int* ell_col;     // [Σ 32·len] column vertex (padding: the row itself, value 0)
  const long long* ell_pos;// [NNZ] value base of row-ordered block q (component c at + 32c)
  double* Hell;           // [E][ell_total]
};

// shared-memory bytes of the env-resident k_pcg_r (kernels.cu) for a batch: the host sizes the
// streamed path's ELL copy by it, the launcher decides which PCG kernel runs
constexpr int PCG_R_THREADS = 512;   // upper bound; the launch picks pcg_r_threads(V)
// threads of k_pcg_r: 4 lanes per soft row, as few row passes as fit in 512 threads with the rows
// split evenly over the passes (C2: V = 288 → 3 passes × 96 rows = 384 threads)
__host__ __device__ inline int pcg_r_threads(int V) {
  for (int passes = 1;; ++passes) {
    const int rows = (V + passes - 1) / passes;
    const int t = ((4 * rows + 31) / 32) * 32;
    if (t <= PCG_R_THREADS) return t < 128 ? 128 : t;
  }
}
__host__ __device__ inline size_t pcg_r_ncpl(const Dev& D) {          // coupling bound: ≤ 1 per (v, d)
  const size_t a = (size_t)D.V * D.ND, b = (size_t)D.cpl_cap;
  return a < b ? a : b;
}
__host__ __device__ inline size_t pcg_r_bytes(const Dev& D, int threads) {
  const size_t nd = (size_t)(threads / 32) * D.ND * 12 + 1 + 5 * (size_t)D.n + 9 * (size_t)D.NEs +
                    18 * (size_t)D.V + 288 * (size_t)D.ND + 3 * pcg_r_ncpl(D);
  const size_t ni = 3 * ((size_t)D.V + 1) + (size_t)D.V + 2 * (size_t)D.NNZ;
  return nd * sizeof(double) + ni * sizeof(int);
}

}  // namespace tac
