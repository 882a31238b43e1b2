/*
 * taccel.h — C ABI of the B200-native batched IPC + ABD Newton step (Taccel, arXiv 2504.12908).
 *
 * Implemented by libtaccel_cuda.so (paper_2504_12908_b200/csrc/, sm_100a, fp64, no CPU fallback).
 * The calls follow the paper's problem statement:
 *   load robots/objects/sensors ........ tac_batch_create
 *   initialise states, zero velocities .. tac_set_state
 *   apply kinematic targets s^y, s^x ..... tac_set_targets
 *   time-step by argmin E_IPC^AL ........ tac_step                (P:L127-131 Eq. unified_ipc_variational,
 *                                                                   P:L137 Eq. unified_ipc_AL)
 *   read positions / gel deformation .... tac_get_state, tac_get_gel_deformation
 *
 * Conventions (all calls):
 *   - SI units (m, kg, s); all floating point is IEEE binary64; indices int32; arrays row-major.
 *   - An affine state y is 12 doubles: t[3] then A[3][3] row-major; a body vertex with body-frame
 *     rest position xbar sits at t + A·xbar (embedding φ).
 *   - Buffers passed to set/get calls may be HOST or DEVICE memory (the library copies with
 *     cudaMemcpyDefault on `stream`); tac_debug_* take HOST buffers.
 *   - `stream` is a cudaStream_t (NULL = legacy default stream).
 *   - Functions return tac_status; on failure tac_last_error() returns a thread-local message that
 *     stays valid until the next call on that thread.  No C++ exception crosses the ABI.
 *   - Per-env failures never abort other envs: tac_step returns TAC_E_ENV_FAILED and sets
 *     that env's tac_env_status; the env is rolled back to its state at the start of the step and
 *     stays DISABLED until the next tac_set_state for it.
 *
 * Ownership: descriptor arrays are borrowed only during tac_batch_create (copied to the device).
 * The workspace is caller-owned device memory (e.g. a torch uint8 tensor) of at least
 * tac_workspace_size() bytes that must outlive the batch handle; the handle itself is heap memory
 * owned by the caller and released with tac_batch_destroy.  State/target buffers are borrowed per
 * call.
 *
 * Homogeneous batch: all envs of a batch share one template (topology, rest shapes, materials);
 * envs differ only through state (x, ẋ, y, ẏ — static bodies' poses are per-env through y) and
 * kinematic targets.
 *
 * Canonical contact primitives (used by tac_debug_active_pairs; the CPU oracle uses the same rule):
 *   global vertex ids: soft vertices (pads in order), then each affine body's vertices;
 *   triangles: per body in body order (pads first) — a pad's surface is the set of tet faces used
 *   by exactly one tet, oriented outward; each triangle is stored rotated so its smallest vertex
 *   id comes first, and a body's triangles are sorted by their sorted vertex triple;
 *   edges: per body, the unique (min,max) vertex pairs of its triangles, sorted.
 *   A PT pair is (kind=0, a=vertex id, b=triangle id); an EE pair is (kind=1, a=edge, b=edge, a<b).
 */
#ifndef TACCEL_H
#define TACCEL_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  TAC_OK = 0,
  TAC_E_INVALID = 1,     /* bad argument (null pointer, out-of-range env range, bad config) */
  TAC_E_VALIDATION = 2,  /* degenerate tet (|V| < 1e-15 m^3) or triangle (area < 1e-12 m^2) */
  TAC_E_ENV_FAILED = 3,  /* tac_step: at least one env failed; see per-env status              */
  TAC_E_CAPACITY = 4,    /* a fixed-capacity table is too small for the template              */
  TAC_E_WORKSPACE = 5,   /* workspace too small or misaligned (needs 256-byte alignment)     */
  TAC_E_CUDA = 6         /* CUDA runtime error (message has the CUDA error string)           */
} tac_status;

typedef enum {
  TAC_ENV_OK = 0,
  TAC_ENV_NEWTON_STALL = 1,   /* line search α < 1e-10 or Newton iteration cap reached          */
  TAC_ENV_AL_INFEASIBLE = 2,  /* AL residual above tolerance after max_al_rounds                */
  TAC_ENV_CAPACITY = 3,       /* candidate/active pair capacity exceeded                        */
  TAC_ENV_NONFINITE = 4,      /* NaN/Inf in the Newton system                                   */
  TAC_ENV_BAD_STATE = 5,      /* tac_set_state: inverted tet (det F <= 0) or a contact distance <= 0 */
  TAC_ENV_DISABLED = 6        /* failed earlier; waits for tac_set_state                         */
} tac_env_status;

typedef enum { TAC_BODY_DYNAMIC = 0, TAC_BODY_KINEMATIC = 1, TAC_BODY_STATIC = 2 } tac_body_kind;

/* A tetrahedral gel pad G_i.  rest_pos is in the pad (sensor) frame.  mount_T maps
 * pad frame → mount-body frame (^{l_j}_{G_i}T): x_link = t + R·x_pad.  Attached vertices (∂⁻G) are
 * driven by the AL to the mount body's target; coated vertices (∂⁺G) are read out. */
typedef struct {
  int32_t n_verts, n_tets;
  const double* rest_pos;        /* [n_verts][3]                                  */
  const int32_t* tets;           /* [n_tets][4], any orientation (fixed internally) */
  double youngs, poisson, density;
  int32_t mount_body;            /* affine body index, or -1 (free soft body: mount_T = world pose) */
  double mount_T[12];            /* t[3], R[3][3] row-major                       */
  int32_t n_attached; const int32_t* attached;     /* ∂⁻G vertex ids            */
  int32_t n_coated;   const int32_t* coated;       /* ∂⁺G vertex ids            */
  int32_t n_markers;  const int32_t* marker_tri;   /* [n_markers][3] vertex ids */
  const double* marker_bary;                       /* [n_markers][3], Σα = 1    */
} tac_soft_desc;

/* An ABD body: closed, outward-oriented triangle surface in its body frame. */
typedef struct {
  int32_t n_verts, n_tris;
  const double* rest_pos;        /* [n_verts][3] */
  const int32_t* tris;           /* [n_tris][3]  */
  int32_t kind;                  /* tac_body_kind */
  double density, kappa_s;       /* kg/m^3; orthogonality stiffness κ_s (Pa) */
} tac_affine_desc;

typedef struct {
  int32_t n_soft, n_affine;       /* n_soft + n_affine ≤ 32 (TAC_E_INVALID otherwise: body masks are 32-bit) */
  const tac_soft_desc* soft;
  const tac_affine_desc* affine;
  const uint8_t* collide;        /* [(n_soft+n_affine)^2] extra body-pair mask (1 = may collide), or NULL */
  double gravity[3];
} tac_scene_desc;

/* Solver constants (proposals; the paper fixes none — DESIGN.md §3). */
typedef struct {
  double dt, dhat, kappa;        /* Δt (s), barrier range d̂ (m), contact stiffness κ   */
  double max_step_rel;           /* Newton steps longer than max_step_rel·L_env (embedded ∞-norm)
                                    are scaled down to that length before CCD/line search (R17c)   */
  double newton_tol_rel;         /* converged iff ‖p‖_emb,∞ ≤ newton_tol_rel · L_env            */
  double al_tol_rel;             /* AL residual tolerance relative to L_env                     */
  double pcg_eta;                /* PCG stops at rᵀz ≤ η² r₀ᵀz₀                                 */
  double armijo_c, accd_s, al_rho0;
  int32_t max_newton, max_al_rounds, max_pcg, max_accd_iters, ee_mollifier;
  int32_t hessian_mode;          /* 0: PSD-projected element Hessians; 1: exact Hessian first, projected
                                    fallback with back-off when PCG meets dᵀHd ≤ 0 or gᵀp ≥ 0 (DESIGN R14b);
                                    2: exact Hessian with a mass-scaled Levenberg-Marquardt shift μM,
                                    μ ← max(lm_mu0, 10μ) on failure, μ/10 after success (DESIGN R14c) */
  int32_t ls_expand;             /* line-search expansion bound K (power of 2; 1 = plain backtracking):
                                    swept sets and ACCD cover [x, x + K·p]; after a full step α doubles
                                    while the energy keeps decreasing (DESIGN R17b)                    */
  int32_t hold_cap;              /* max projected iterations between exact-Hessian attempts           */
  double lm_mu0;                 /* first LM shift of hessian_mode 2                                  */
  double bp_margin;              /* δ (m): candidate lists are built with targets inflated by d̂+2δ and
                                    reused while every surface vertex stays within δ of its box at the
                                    last build; 0 = rebuild every Newton iteration (DESIGN R11b)       */
  int32_t cand_capacity_per_env, active_capacity_per_env;
  double mu_friction;            /* Coulomb coefficient μ of the lagged friction potential D_k; 0 = frictionless.
                                    μ > 0 requires hessian_mode 2 (the friction Hessian is PSD and is not projected) */
  double eps_v;                  /* ε_v (m/s) of the friction transition f1 */
  double pcg_eta_max;            /* relaxed PCG tolerance ("carefully relaxing convergence tolerances";
                                    DESIGN R24): 0 = the fixed η above; > 0 = per Newton iteration the
                                    Eisenstat–Walker forcing η_k = 0.9·(r₀ᵀz₀)_k/(r₀ᵀz₀)_{k−1}, safeguarded by
                                    0.9·η_{k−1}² when that exceeds 0.1, clamped to [pcg_eta, pcg_eta_max]; the first
                                    solve of a time step uses pcg_eta_max.  Must be 0 or in [pcg_eta, 1).      */
} tac_config;

typedef struct {
  int32_t status;                /* tac_env_status of the last step */
  int32_t newton_iters, pcg_iters, ls_backtracks, n_active, al_rounds, n_candidates;  /* last step */
  double alpha_min, energy, constraint_residual;                                     /* last step */
  int64_t pcg_iters_total;       /* cumulative since tac_batch_create                         */
  double pcg_alg_bytes_total;    /* cumulative algorithmic PCG bytes (DESIGN.md §5 B_pcg model) */
  double diag[4];                /* last Newton iteration: ACCD bound, gᵀp, E(q), E at the last trial α */
  double min_dist;               /* end of the last step: min primitive distance over the candidate pairs
                                    closer than d̂ (+inf if none) — the intersection-free certificate d > 0 */
  int32_t n_residual;            /* last Newton iteration: active pairs kept matrix-free in the SpMV (two
                                    soft bodies or two DoF bodies in one pair) */
  int32_t n_couplings;           /* last Newton iteration: condensed 3×12 soft–body coupling blocks */
  double lm_mu;                  /* LM shift μ of the last solve (hessian_mode 2; 0 = pure Newton) */
  int32_t n_friction;            /* lagged friction pairs of the last step (the active set at its start xⁿ) */
  int32_t capacity_flags;        /* capacity overflows since tac_batch_create (TAC_ENV_CAPACITY): 1 candidates,
                                    2 large-primitive list of the broad phase, 4 hash entries, 8 active pairs,
                                    16 residual (matrix-free) pairs, capacity max(64, active_capacity_per_env/4) */
} tac_env_stats;

struct tac_batch;
typedef struct tac_batch tac_batch;

/* Bytes of device workspace a batch of n_envs needs. */
tac_status tac_workspace_size(const tac_scene_desc* scene, int32_t n_envs, const tac_config* cfg, size_t* bytes);

/* Validate and pre-process the template (orientation, D_m⁻¹, lumped masses, surfaces, rest areas,
 * M^y, sparsity pattern and gather maps), carve `workspace` and upload.  Synchronises `stream`. */
tac_status tac_batch_create(const tac_scene_desc* scene, int32_t n_envs, const tac_config* cfg, int32_t device,
                            void* workspace, size_t ws_bytes, void* stream, tac_batch** out);
tac_status tac_batch_destroy(tac_batch* b);

/* Template sizes: [0]=soft verts V, [1]=tets, [2]=affine bodies NA, [3]=kinematic NK,
 * [4]=coated verts total, [5]=markers total, [6]=DoFs per env n, [7]=all contact vertices,
 * [8]=surface triangles, [9]=surface edges. */
tac_status tac_batch_dims(const tac_batch* b, int32_t dims[10]);

/* Set the state of envs [env0, env0+n): x [n][V][3], xdot [n][V][3] (NULL → 0), y [n][NA][12],
 * ydot [n][NA][12] (NULL → 0).  Resets per-env status and derives L_env (bounding-box diagonal of
 * all vertices).  Validates every env (det F > 0 for all tets, all contact distances > 0); envs
 * failing get TAC_ENV_BAD_STATE in env_status[n] (host or device, may be NULL). Host-blocking. */
tac_status tac_set_state(tac_batch* b, int32_t env0, int32_t n, const double* x, const double* xdot,
                         const double* y, const double* ydot, uint8_t* env_status, void* stream);

/* Kinematic targets s^y for the next step, y_kin [n][NK][12] in kinematic-body order; the
 * attached-vertex targets s^x follow from the mount links. */
tac_status tac_set_targets(tac_batch* b, int32_t env0, int32_t n, const double* y_kin, void* stream);

/* ---- on-device forward kinematics and action compilation ------
 * A robot is a tree of links, each driving one kinematic affine body.  Link i (parents before
 * children) has: parent (−1 = the env's base pose), origin[12] — the fixed transform (t, R row-major)
 * from the parent's joint frame to its own joint frame at zero joint angle, axis[3] — the unit joint axis
 * in its joint frame, joint — the index of its joint coordinate (revolute) or −1 (fixed), body[12] —
 * the kinematic body's frame relative to the link's joint frame, kin_body — the affine body index it
 * drives.  Joint frame of link i: J_i = J_parent · origin_i · Rot(axis_i, q_joint); target of its body:
 * J_i · body_i (homogeneous products).  The chain is copied (host arrays borrowed for the call). */
typedef struct {
  int32_t n_links, n_joints;
  const int32_t* parent;       /* [n_links] */
  const double* origin;        /* [n_links][12] */
  const double* axis;          /* [n_links][3] */
  const int32_t* joint;        /* [n_links] joint index or −1 */
  const double* body;          /* [n_links][12] */
  const int32_t* kin_body;     /* [n_links] kinematic affine body index */
} tac_chain_desc;
tac_status tac_set_chain(tac_batch* b, const tac_chain_desc* chain);
/* Action compilation on the device: joint targets q [n][n_joints] and base poses [n][12] (NULL = keep the
 * previous base, identity at first) of envs [env0, env0+n) → the kinematic targets s^y of every chain
 * link's body (the attached-vertex targets s^x follow from them at the next step).  Kinematic
 * bodies outside the chain keep their targets.  Host or device buffers; enqueued on `stream`. */
tac_status tac_set_joint_targets(tac_batch* b, int32_t env0, int32_t n, const double* base, const double* q, void* stream);
/* Current kinematic targets y_kin [n][NK][12] (as set by tac_set_targets / tac_set_joint_targets). */
tac_status tac_get_targets(tac_batch* b, int32_t env0, int32_t n, double* y_kin, void* stream);

/* Advance every enabled env by n_steps time steps.  Host-blocking.  env_status [E] (may be NULL). */
tac_status tac_step(tac_batch* b, int32_t n_steps, uint8_t* env_status, void* stream);

/* Scheduled multi-step mode: advance every enabled env through n_steps time steps, env k of step s
 * using kinematic targets y_kin_sched [n_steps][E][NK][12].  Envs advance independently: an env that
 * converged its step starts the next one at once (no lockstep wait for the slowest env); each env's
 * trajectory is bitwise identical to calling tac_set_targets + tac_step per step.  After each step of
 * each env its gel deformation is written to coated_disp [n_steps][E][Σcoated][3], marker_pos and
 * marker_flow [n_steps][E][Σmarkers][3] (all three NULL = no readout).  Buffers may be host or device
 * memory (host buffers are staged through stream-ordered device allocations).  Host-blocking. */
tac_status tac_step_schedule(tac_batch* b, int32_t n_steps, const double* y_kin_sched, double* coated_disp,
                             double* marker_pos, double* marker_flow, uint8_t* env_status, void* stream);

tac_status tac_get_state(tac_batch* b, int32_t env0, int32_t n, double* x, double* xdot, double* y,
                         double* ydot, void* stream);

/* Gel deformation in the pad (sensor) frame from the mount link's CURRENT pose:
 * coated_disp [n][Σcoated][3], marker_pos [n][Σmarkers][3] (world), marker_flow [n][Σmarkers][3]
 * (sensor frame).  Any pointer may be NULL. */
tac_status tac_get_gel_deformation(tac_batch* b, int32_t env0, int32_t n, double* coated_disp,
                                   double* marker_pos, double* marker_flow, void* stream);

tac_status tac_get_stats(tac_batch* b, tac_env_stats* out /* [E] host */, void* stream);

/* Depth and normal maps of the deformed coated surface ∂⁺G̃ of every pad ("extract the depth
 * and normal maps d(u,v), n(u,v) ... from the deformed coated surface"; reading R22): an orthographic
 * camera in each pad's sensor frame looks along −z at the coated face.  Pixel (i, j) of an H×W map
 * (H, W ≥ 2) samples the sensor-frame point (x₀ + j·(x₁−x₀)/(W−1), y₀ + i·(y₁−y₀)/(H−1)), a
 * corner-aligned grid over the rest extent [x₀,x₁]×[y₀,y₁] of the pad's coated vertices.  A coated
 * triangle (surface triangle with three coated vertices) covers a pixel when the pixel's barycentric
 * coordinates in the triangle's deformed xy projection are all ≥ −1e-9.  depth = z_ref − z, the largest
 * over covering triangles of the linearly interpolated deformed height z below the rest height z_ref of
 * the coated face (positive = indentation); normal = the normalised sum of the covering triangles'
 * (deformed, sensor-frame) area vectors, oriented +z.  Uncovered pixels: depth NaN, normal 0.
 * depth [n][npads][H][W], normal [n][npads][H][W][3] (either may be NULL), host or device memory. */
tac_status tac_get_depth_maps(tac_batch* b, int32_t env0, int32_t n, int32_t H, int32_t W, double* depth, double* normal,
                              void* stream);

const char* tac_last_error(void);

/* ---- tracing: CUDA-event phase timers on the launch stream ----------------------------------
 * When enabled, every kernel launch of tac_step is bracketed by cudaEventRecord on `stream` and
 * its device time is accumulated per phase.  tac_profile_read copies the per-phase totals (ms)
 * and launch counts for the TAC_NPHASES phases (names from tac_profile_phase_name) and optionally
 * resets them. */
#define TAC_NPHASES 16
tac_status tac_profile_enable(tac_batch* b, int32_t enable);
tac_status tac_profile_read(tac_batch* b, double* ms, int64_t* launches, int32_t reset);
const char* tac_profile_phase_name(int32_t phase);
/* Newton iterations of the last time step: envs still active after each iteration and the host
 * wall time of each iteration (ms); n = number of iterations (arrays filled up to cap). */
tac_status tac_profile_iterations(tac_batch* b, int32_t* active, double* ms, int32_t cap, int32_t* n);

/* ---- parity hooks (exported, test-only; host buffers) ---------------------------------------
 * tac_debug_eval: at (x [V][3], y [NA][12]) of env `env`, with x̃/ỹ from the env's last set_state
 * and kinematic targets from the last set_targets, and AL multipliers lam_att [NC][3],
 * lam_kin [NK][12] (NULL → 0) and penalty rho (≤ 0 → al_rho0): the six energy terms
 * e_terms[7] = {inertia, elastic, ortho, gravity, barrier, AL, friction}, the gradient grad [n] over
 * q = [x; y of non-static bodies] and hv = H·v_in [n] with H the PSD-projected Hessian (any
 * output may be NULL); exact_hessian = 1 uses the unprojected element Hessians instead.  The
 * active set is recomputed at (x, y) through the spatial hash.  With friction (μ > 0) the lagged
 * friction pairs and their data are frozen at the env's current state xⁿ (as at the start of a step),
 * and exact_hessian must be 1. */
tac_status tac_debug_eval(tac_batch* b, int32_t env, const double* x, const double* y, const double* lam_att,
                          const double* lam_kin, double rho, int32_t exact_hessian, const double* v_in,
                          double* e_terms, double* grad, double* hv, void* stream);
/* Active pairs at (x, y): rows (kind, a, b) in canonical order. */
tac_status tac_debug_active_pairs(tac_batch* b, int32_t env, const double* x, const double* y, int32_t* pairs,
                                  int32_t cap, int32_t* count, void* stream);
/* Candidate pairs (swept boxes over [q, q + K·p] with K = ls_expand, p [n] or NULL for static) in
 * canonical order. */
tac_status tac_debug_candidates(tac_batch* b, int32_t env, const double* x, const double* y, const double* p,
                                int32_t* pairs, int32_t cap, int32_t* count, void* stream);
/* α_max = K · min(1, min ACCD over the swept candidates along K·p), in units of p [n]. */
tac_status tac_debug_accd(tac_batch* b, int32_t env, const double* x, const double* y, const double* p,
                          double* alpha, void* stream);
/* Block-Jacobi PCG solve at (x, y) (AL as in tac_debug_eval) with the kernel tac_step uses:
 * exact_hessian = 0: H p = −g with the PSD-projected H (mu ignored);
 * exact_hessian = 1: (H + μM) p = −g with the EXACT H and M the mass matrix (reading R14c), starting
 * from μ = mu; if the solve meets negative curvature or gᵀp ≥ 0 the kernel raises μ ← max(μ₀, 10μ)
 * and re-solves in the same launch, exactly as in tac_step.  Outputs: p [n], PCG iterations of all
 * attempts, and the μ of the accepted solve (mu_used, may be NULL). */
tac_status tac_debug_pcg(tac_batch* b, int32_t env, const double* x, const double* y, int32_t exact_hessian,
                         double mu, double* p, int32_t* iters, double* mu_used, void* stream);
/* Fault injection (test-only): env `env` fails with `status` (TAC_ENV_NEWTON_STALL..TAC_ENV_NONFINITE)
 * at the end of the first Newton iteration of its next step — rolled back to the state at the start of
 * that step and DISABLED, exactly like a detected failure; other envs are unaffected. */
tac_status tac_debug_inject_fault(tac_batch* b, int32_t env, int32_t status, void* stream);

/* Newton-iteration trace of one env (diagnostic): rows = NULL, cap > 0 starts tracing env `env` into a
 * fresh device buffer of cap rows; env < 0 stops; rows != NULL copies min(n, cap) rows and the count n.
 * Row: [Newton iteration, PCG iterations, μ used, ‖p‖_emb,∞, ‖M⁻¹g‖_emb,∞ (under a shift), gᵀp,
 *       α (negative = line search failed), E(q), E(q+αp), backtracks]. */
tac_status tac_debug_trace(tac_batch* b, int32_t env, int32_t cap, double* rows, int32_t* n);

/* Name of the PCG kernel tac_step launches for this batch (env-resident "k_pcg_r"/"k_pcg_r512" when the
 * condensed operator fits one SM's shared memory, else the streamed-operator "k_pcg"). */
const char* tac_pcg_kernel_name(const tac_batch* b);

#ifdef __cplusplus
}
#endif
#endif /* TACCEL_H */
