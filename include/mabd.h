/*
 * mabd.h — C ABI of libmabd.so, the B200 (sm_100a, fp64) hot path of one M-ABD implicit step.
 *
 * Method: "M-ABD: Scalable, Efficient, and Robust Multi-Affine-Body Dynamics" (arxiv 2603.08079),
 * cited as P:<line> of /root/reference/PAPER.md (LaTeX source). One call of mabd_step(h, 1)
 * performs one Newton iteration of the implicit step (Table 1, "# Iter. 1"):
 *   (1) per body: polar R of A, f_A = (1/h)M_A q̇ + M_A[0;g] − [V vec(R Π(RᵀA)); 0]
 *       (P:195-199);
 *   (2) per body: δq̃ = diag₄(R) H̄⁻¹ diag₄(Rᵀ) f_A with the constant H̄ = M_A/h² + K̄_A
 *       (Alg. 1 with the exact R);
 *   (3) the dual (joint-space) solve (∇C̃ H̃⁻¹ ∇C̃ᵀ) λ = C(q̃) (footnote P:459), by topology:
 *       block-tridiagonal for chains, leaf-to-root elimination for trees (exact
 *       form, reading A12), sparse for loops/irregular nets;
 *   (4) q ← q̃ − H̃⁻¹∇C̃ᵀλ, q̇ ← (qⁿ⁺¹ − qⁿ)/h.
 *
 * Conventions
 *   - Everything is IEEE fp64, SI units.
 *   - q = [vec(A); t] ∈ R¹², vec column-major: q[3c + r] = A[r][c], q[9 + i] = t[i].
 *   - Arrays of bodies are row-major [n][12] ("AoS" from the caller's view); the library keeps its own
 *     SoA, topology-ordered copy on the device and undoes the ordering on output.
 *   - mbar is the packed symmetric 4×4 generalized mass M̄ with M_A = M̄ ⊗ I₃,
 *     upper triangle row-major (00,01,02,03,11,12,13,22,23,33); any SPD M̄ (any material frame: bodies
 *     are mapped to their central principal frame internally and back on output, reading R8).
 *   - Joints are point-coincidence constraints C = x_a(ȳ_a) − x_b(ȳ_b), x(ȳ) = Aȳ + t: a ball joint has
 *     1 point, the linear ("affine") hinge has 2 points on the axis. body_b = −1
 *     makes an anchor to the world point stored in ybar_b. The nonlinear joints of P:391-444 are
 *     joints.kind = 1 (five-row hinge), 2 (universal), 3 (prismatic); the sparse solver runs them.
 *
 * Ownership
 *   - Every input pointer is borrowed for the duration of the call only; the library copies what it needs.
 *   - Device memory: if options.workspace is non-NULL it must hold options.workspace_bytes ≥ the value
 *     returned by mabd_workspace_size and outlive the handle; the library sub-allocates from it and never
 *     allocates on the step path. If it is NULL the library allocates (cudaMalloc) inside mabd_create.
 *   - A handle is bound to the current CUDA device and to options.cuda_stream (NULL = legacy default
 *     stream) at creation; it is not thread-safe.
 *
 * Errors
 *   - Every call returns mabd_status; nothing is thrown across the ABI. mabd_last_error(handle) returns
 *     a message for the last failure on that handle (or on the calling thread if handle is NULL).
 *   - Invalid arguments return MABD_EINVAL and leave the handle unchanged.
 *   - mabd_step checks a device error word once at the end of the call (one 4-byte D2H copy and a
 *     stream synchronisation): det A ≤ 1e-9 or a non-finite value → MABD_ENONFINITE, a non-positive
 *     dual pivot → MABD_ESINGULAR. The message names the first failing step of the call.
 */
#ifndef MABD_H
#define MABD_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct mabd_ctx *mabd_handle;

typedef enum {
  MABD_OK = 0,
  MABD_EINVAL = 1,       /* bad argument (sizes, indices, h ≤ 0, non-SPD M̄, joint on one body …) */
  MABD_ESTATE = 2,       /* call out of order (e.g. step before prefactor)                        */
  MABD_ENOMEM = 3,       /* workspace too small / allocation failed                               */
  MABD_ECUDA = 4,        /* CUDA runtime error                                                    */
  MABD_ENCCL = 5,        /* NCCL error (multi-GPU)                                                */
  MABD_ESINGULAR = 6,    /* dual matrix not SPD (redundant joints)                                */
  MABD_ENONFINITE = 7,   /* non-finite state or det A ≤ 1e-9                                      */
  MABD_EUNSUPPORTED = 8  /* input outside this version's scope (topology / joint kind for a solver …) */
} mabd_status;

/* Bodies, in the caller's order. */
typedef struct {
  int64_t n;                 /* number of bodies, ≥ 1                                              */
  const double *q0;          /* [n][12] initial q                                          */
  const double *qd0;         /* [n][12] initial q̇                                                  */
  const double *mbar;        /* [n][10] packed M̄ (see above)                                       */
  const double *volume;      /* [n] V (m³): weight of the elastic force                  */
  const double *youngs;      /* [n] E (Pa)                                                         */
  const double *poisson;     /* [n] ν, in (−1, 0.5)                                                 */
  const int32_t *material;   /* [n] or NULL: ignored hint (the library detects shared materials)   */
  double gravity[3];         /* m/s²                                                               */
} mabd_bodies;

/* Joints made of 3-row point-coincidence constraints. */
typedef struct {
  int64_t n_joints;          /* K ≥ 0                                                              */
  const int32_t *body_a;     /* [K] in [0, n)                                                      */
  const int32_t *body_b;     /* [K] in [−1, n), −1 = world (anchor), ≠ body_a                      */
  const int32_t *npts;       /* [K] in {1 (ball / anchor), 2 (linear hinge, five-row hinge, universal),
                                3 (prismatic)}                                                       */
  const double *ybar_a;      /* [Σnpts][3] material points on body_a (body frame)                  */
  const double *ybar_b;      /* [Σnpts][3] material points on body_b, or world points for anchors  */
  const int32_t *kind;       /* [K] or NULL (all 0). 0: point joint (ball / linear 6-row hinge / anchor);
                                1: five-row hinge (Eq. hinge; R13): npts = 2, the points on
                                the axis (the axis in body_a's frame is ȳ_a[1] − ȳ_a[0]); the first point is a
                                ball, the second keeps only its two rows normal to the axis in the hinge frame
                                R_H = ΔR_H Rᵀ(A_a), re-evaluated every Newton iteration. Sparse solver only.
                                2: universal joint (Eq. universal; R17): npts = 2; point 0
                                is the centre (a ball); ȳ_a[1] − ȳ_a[0] is the axis a₁ in body_a's frame and
                                ȳ_b[1] − ȳ_b[0] the axis a₂ in body_b's (world for an anchor), a₁ ⟂ a₂ at creation;
                                one more row (A_a â₁)·(A_b e₂) = 0 keeps them orthogonal. Sparse solver only.
                                3: prismatic joint (Eq. prismatic; R17): npts = 3, all three points
                                coincident at creation; points 0, 1 on the sliding axis (ȳ_a[1] − ȳ_a[0] in
                                body_a's frame), point 2 off the axis. Five rows: the offset of point 0 normal to
                                the axis, the axes parallel, no twist. Sparse solver only. Rows of kinds 2, 3 are
                                linearised at every Newton iteration with R ≈ A and their exact gradient.       */
  const double *limits;      /* [K][8] or NULL: joint limits of five-row hinges (R14): lo, hi
                                (rad; ±inf = none), u_a (3, ⟂ the axis, body a's frame), u_b (3, body b's frame,
                                or world for an anchor) with u_a, u_b equal in the world at creation, so the hinge
                                angle θ = atan2(a_w·(u_aw × u_bw), u_aw·u_bw) is 0 there. A limit violated at a
                                Newton iteration's linearisation point holds θ at the bound for that iteration
                                (one extra row; its residual is the dual-space penalty). Ignored for kind 0.      */
} mabd_joints;

typedef struct {
  int32_t newton_iters;      /* Newton iterations per step, 1..16 (0 = 1; Table 1 uses 1). Iteration i is
                                linearised at the previous iterate (footnote P:459); K > 1 uses 96 more
                                bytes per body of workspace and K + 2 times the launches              */
  int32_t residual_rhs;      /* 1 (0 = default = 1): include −C(qⁿ) in the dual rhs (footnote P:459,
                                DESIGN.md reading A4); any other value → MABD_EINVAL                  */
  int32_t solver;            /* 0 auto | 1 chain | 2 tree | 3 sparse | 4 line Gauss-Seidel (the paper's
                                Case IV; R10: an iterative dual solve, never chosen by
                                auto; converged to gs_tol, warm-started from the previous step's λ)
                                | 5 loop breakers (the paper's Case III; R12: the joints
                                that close loops (≤ 8 points, ≤ 1 per body) are removed, the remaining forest
                                runs on the chain / tree solver 2 + 3·points times per iteration and the
                                breakers' multipliers solve the small Schur system; exact; no wrenches)   */
  int32_t rank, world;       /* multi-GPU; world = 1 → single GPU                                  */
  const void *nccl_unique_id;/* 128-byte ncclUniqueId, or NULL when world = 1                      */
  void *workspace;           /* device memory from the caller (torch), or NULL                     */
  size_t workspace_bytes;
  void *cuda_stream;         /* cudaStream_t, or NULL                                              */
  int32_t no_graphs;         /* 0: each step is replayed as one CUDA graph captured on cuda_stream (needs a
                                non-NULL stream; rebuilt after mabd_prefactor / mabd_set_wrench); 1: plain
                                stream launches                                                        */
  int32_t rotation;          /* MABD_ROTATION_POLAR (0): exact R = polar(A). 
                                MABD_ROTATION_LENGTH_PRESERVING (1): the polar-free variant of P:283-310
                                (Alg. 1; reading R9): the free solve maps each 3-block by the
                                length-preserving Aᵀ / A of Eq. len_preserving, the elastic force is the StVK
                                force of E = ½(AᵀA − I), and constraint forces use diag₄(A)H̄⁻¹diag₄(Aᵀ)
                                ("A ≈ R"). Equal to (0) at rigid states; an approximation otherwise. */
  int32_t host_exchange;     /* world > 1 without NCCL: this process advances rank `rank`'s share and the
                                caller moves the per-step exchange (mabd_step_exchange_begin / end); see
                                there. One Newton iteration only.                                       */
  int32_t gs_sweeps;         /* solver 4: maximum sweeps per step (0 = 200)                           */
  double gs_tol;             /* solver 4: stop when max|C(q̃) − Sλ| ≤ gs_tol · max|C(q̃)| (0 = 1e-12)   */
} mabd_options;

enum { MABD_ROTATION_POLAR = 0, MABD_ROTATION_LENGTH_PRESERVING = 1 };

/* Topology/solver actually selected (mabd_query). */
enum { MABD_SOLVER_CHAIN = 1, MABD_SOLVER_TREE = 2, MABD_SOLVER_SPARSE = 3, MABD_SOLVER_LINE_GS = 4,
       MABD_SOLVER_LOOP_BREAKER = 5 };

/* Device bytes mabd_create will sub-allocate for these inputs (host analysis only; no GPU work). */
mabd_status mabd_workspace_size(const mabd_bodies *bodies, const mabd_joints *joints,
                                const mabd_options *opts, size_t *bytes);

/* The problem statement of P:459-475 (Eq. kkt): M affine bodies (mass M_A = M̄ ⊗ I₃; elastic
 * weight V with E, ν) and K joints. Validates (MABD_EINVAL on bad sizes, indices, non-SPD M̄,
 * a joint on one body, npts ∉ {1, 2} (3 for kind 3), bad kind / limits / options), maps every body to its canonical frame
 * (R8), classifies the joint topology (forest of ball-joint paths → chain, forest → tree, cycles → sparse;
 * SURVEY A14) or takes options.solver, orders bodies and joints for that solver, and copies everything into the
 * device workspace. Borrows the arrays for the duration of the call. World > 1 with an NCCL id: collective. */
mabd_status mabd_create(const mabd_bodies *bodies, const mabd_joints *joints,
                        const mabd_options *opts, mabd_handle *out);

/* Build the constant per-material H̄⁻¹ data and the solver plan for step size h > 0.
 * mabd_step with another h re-prefactors transparently. */
mabd_status mabd_prefactor(mabd_handle h_, double h);

/* Advance nsteps ≥ 0 implicit steps of size h on the handle's stream: per step, options.newton_iters Newton
 * iterations of the linearised KKT (footnote P:459), each the four stages of the hot path — per-body
 * co-rotated r.h.s., back-substitution through H̄ (Alg. 1), the dual
 * solve S λ = C(q̃), S = ∇C̃ H̃⁻¹ ∇C̃ᵀ, the primal update —
 * then q̇ⁿ⁺¹ = (qⁿ⁺¹ − qⁿ)/h. Asynchronous apart from the final error-word check described above (ESINGULAR,
 * ENONFINITE name the first failing step; ECUDA / ENCCL for launch or exchange failures). */
mabd_status mabd_step(mabd_handle h_, double h, int64_t nsteps);

/* Enqueue nsteps steps on the handle's stream and return without synchronising (a serving loop, or a timed
 * region that must not contain host waits). The device error word accumulates over async calls; mabd_check (or the
 * next mabd_step) synchronises, reports the first failing step since the last check and resets it. */
mabd_status mabd_step_async(mabd_handle h_, double h, int64_t nsteps);

/* Synchronise the handle's stream and report errors of the steps enqueued since the last check (see mabd_step). */
mabd_status mabd_check(mabd_handle h_);

/* Caller-driven exchange for split scenes (options.world > 1, options.host_exchange = 1): the step
 * of a chain or tree split across ranks has one all-gather (per-rank top systems, resp. the subtree roots'
 * condensed blocks). mabd_step_exchange_begin(h) runs this rank's share up to it and synchronises;
 * mabd_exchange_info gives the buffer's shape (doubles per rank, ranks, this rank's slot); mabd_exchange_copy
 * copies this rank's slot out to host_all[slot·per_rank …] (to_device = 0) or the whole host_all in
 * (to_device = 1, after the caller's all-gather); mabd_step_exchange_end finishes the step and checks errors. Any
 * transport works (a test uses gloo between processes). mabd_get_state then returns this rank's bodies current
 * and the others stale (the NCCL path broadcasts them). */
mabd_status mabd_step_exchange_begin(mabd_handle h_, double h);
mabd_status mabd_exchange_info(mabd_handle h_, int64_t *doubles_per_rank, int32_t *ranks, int32_t *my_slot);
mabd_status mabd_exchange_copy(mabd_handle h_, double *host_all, int32_t to_device);
mabd_status mabd_step_exchange_end(mabd_handle h_);

/* Copy the current state (q, q̇; P:184 layout) out, in the caller's body order and material frames ([n][12] each;
 * either pointer may be NULL): the internal SoA, topology order and canonical frames (R8) are undone.
 * out_on_device != 0 means the pointers are device memory. Synchronises the handle's stream. With world > 1 and
 * NCCL, every rank's share is broadcast first, so all ranks return the full state. */
mabd_status mabd_get_state(mabd_handle h_, double *q_out, double *qd_out, int out_on_device);

/* Overwrite the state (checkpoint restore; stage tests). Same layout as mabd_get_state. */
mabd_status mabd_set_state(mabd_handle h_, const double *q, const double *qd, int in_on_device);

/* Constant external wrenches: W is [n][6] = (τ, f) per body in the caller's
 * order, world frame, applied in every step (and Newton iteration) as f_A,ext = G(A)ᵀW at the linearisation
 * point: ½ τ × q_c on the column c of A, f on t. Host or device pointer (in_on_device); the values are copied.
 * W = NULL removes the wrenches. Uses the handle's stream; a host W synchronises it. */
mabd_status mabd_set_wrench(mabd_handle h_, const double *W, int in_on_device);

/* Introspection: selected solver, number of device kernel launches per step, bodies, dual rows. */
mabd_status mabd_query(mabd_handle h_, int32_t *solver, int32_t *launches_per_step, int64_t *n_bodies,
                       int64_t *n_dual_rows);

/* Multi-GPU (chain scenes). Every rank passes the full scene with options.world = W, options.rank = r and a
 * 128-byte ncclUniqueId that rank 0 obtained from mabd_nccl_unique_id and shared (e.g. through
 * torch.distributed); mabd_create is then collective. Rank r advances a contiguous share of the chain
 * windows; long chains crossing ranks exchange one 27-double "top" system per rank per step
 * (ncclAllGather, in-stream). mabd_get_state broadcasts every rank's share first, so all ranks return the
 * full state. With world > 1 and nccl_unique_id == NULL the W parts are emulated in one process (one GPU,
 * same arithmetic, the all-gather is a no-op): used to test the partitioned algorithm on one device. */
mabd_status mabd_nccl_unique_id(void *out, size_t bytes);

/* Host-only analysis for tests: out[0..9] = {parts, windows, long windows, this rank's window range lo/hi,
 * long-window range lo/hi, left_open, right_open, sequential-top unknowns} of the chain split; with
 * n_out >= 20 also out[10..19] = {solver, tree parts, bottom groups, groups per part, gather slots per part,
 * this rank's group range lo/hi and body range lo/hi, joints into bottom groups} of the tree split
 * (SURVEY §8(e)). No device work. */
mabd_status mabd_partition_info(const mabd_bodies *bodies, const mabd_joints *joints,
                                const mabd_options *opts, int64_t *out, int64_t n_out);

/* Host-only analysis of the sparse solver's plan for a scene (no device work; forces the sparse solver):
 * out[0..7] = {assembly-tree fronts, levels, largest front (rows), front storage (doubles), flops of one
 * numeric factorization (fp64, the algorithmic Cholesky count 2·Σ(nn³/6 + nn²mm/2 + nn·mm²/2) over the fronts,
 * nn eliminated and mm boundary rows), task-list ints, launches per step, dual rows}. */
mabd_status mabd_sparse_plan_stats(const mabd_bodies *bodies, const mabd_joints *joints, double *out);

/* Host-only plan of the line Gauss-Seidel solver (solver 4; R10) for a scene: counts = {points, chains,
 * colours}; when the arrays are non-NULL they receive the joint points in chain order ([points], point index = the
 * running index over the joints' points), the chain offsets ([chains + 1]) and the colour offsets into the chains
 * ([colours + 1]). Call once with NULL arrays for the sizes. No device work. */
mabd_status mabd_line_gs_plan(const mabd_bodies *bodies, const mabd_joints *joints, int32_t *chain_pts,
                              int32_t *chain_off, int32_t *color_off, int64_t *counts);

/* Statistics of the last step: the sparse solver's iterative-refinement passes run in the last Newton iteration
 * (0 or 1: a pass runs only when the factorization's residual max|r − Sλ| exceeds 1e-10 · max|r|; R2);
 * the line Gauss-Seidel solver's sweeps run in the last step; 0 for the chain and tree solvers.
 * Synchronises the handle's stream. */
mabd_status mabd_solver_stats(mabd_handle h_, int64_t *last_iterations);

/* Release device memory owned by the library; NULL is a no-op. */
mabd_status mabd_destroy(mabd_handle h_);

/* Last error message for the handle (or for the calling thread when h_ is NULL). Never NULL. */
const char *mabd_last_error(mabd_handle h_);

#ifdef __cplusplus
}
#endif
#endif /* MABD_H */
