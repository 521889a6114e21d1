// Host-side plan: topology analysis, ordering and the device memory layout (internal).
#pragma once
#include <cuda_runtime.h>

#include <functional>
#include <string>
#include <vector>

#include "../../include/mabd.h"
#include "mabd_internal.h"
#include "mabd_kernels.h"

namespace mabd {

struct BtdLevel {
  int64_t n_u;     // unknowns at this level
  int64_t windows; // CTAs
  bool fused;      // top level (n_u ≤ 256)
};

// Tree plan (exact leaf-to-root elimination, reading A12); see mabd_tree.cu.
// Internal body order: bottom groups (CTA-local subtrees, ≤ cap bodies each), then the top group; inside a group
// bodies are sorted by depth, deepest first, with per-level ranges, bodies with child joints first in each level.
// cap = TREE_CAP, or 2·TREE_CAP for trees large enough to give every SM a group at the larger size.
constexpr int TREE_CAP = 256;
constexpr int TREE_TOP_SMALL = 32;  // a top set larger than this gets a middle layer …
constexpr int TREE_MID_CAP = 7;     // … of subtrees with at most this many bodies (measured: 7 < 15 < 31 < 63)
constexpr int TREE_TSLOT = 28;  // doubles per condensed joint block (Ŝ_u packed + r̂_u), the tree exchange unit
constexpr int TREE_MAXN = 24;  // max dual rows of the child joints of one body (frontal size ≤ 24 + 6)
struct TreePlan {
  std::vector<int32_t> up_joint;     // [n] joint to the parent (−1 for a root)
  std::vector<int32_t> child_off;    // [n+1] CSR of each body's child joints (incl. anchors)
  std::vector<int32_t> child_joint;
  std::vector<int64_t> ws_off;       // [n+1] per-body doubles of (y, W) kept for the downward pass
  std::vector<int32_t> jnpts;        // [K]
  std::vector<int32_t> jchd;         // [K] child body (internal) or −1 for an anchor
  std::vector<double> jy;            // [K][12]: ȳ on the parent body (2×3), ȳ on the child / world point (2×3)
  std::vector<int32_t> group_off;    // [G+1] body ranges
  std::vector<int32_t> glev_ptr;     // [G+1] into glev_off
  std::vector<int32_t> glev_off;     // level boundaries (absolute body indices), deepest level first
  std::vector<int32_t> glev_nl;      // [levels] end of the level's bodies with child joints
  int32_t cap = TREE_CAP;            // group capacity (bodies)
  bool top_fused = false;            // the top group fits one CTA (else one launch per top level)
  int32_t n_bottom = 0;              // bottom groups (layer 0)
  int32_t n_mid = 0;                 // middle-layer groups (after the bottom ones); the top group (if any) is last
  bool has_top = false;
  int64_t ws_total = 0;
  std::vector<int64_t> fo_off;       // [n] front record offsets (bodies with child joints, and the top group)
  std::vector<int32_t> fo_str;       // [n] their stride (records interleaved per group)
  std::vector<int32_t> parent, up_row;  // [n] parent body (internal order) and the up joint's row in its front
  int64_t fo_total = 0;
  int32_t max_m = 3;                 // largest frontal matrix (rows)
  std::vector<int32_t> pt_off, pt_code, body_nn;  // per body: frontal point codes, N | nu << 8
  // multi-GPU split: the bottom groups are divided into W contiguous blocks of gpr groups;
  // each part eliminates its groups, the condensed blocks (Ŝ_u, r̂_u) of the group roots' up joints are
  // all-gathered, and every part solves the top levels redundantly
  int32_t parts = 1, part = 0, gpr = 0, rpp = 0;
  bool emulate = false;                      // W parts in one process (no NCCL): single-GPU test of the split
  std::vector<int32_t> root_off;             // [n_bottom+1] CSR: joints from a top body into each bottom group
  std::vector<int32_t> root_joint;           // those joints, by group
  std::vector<int32_t> root_slot;            // their slot in the gather buffer: part · rpp + index in part
};

// Sparse plan: constraint points, body → point incidence, and the multifrontal symbolic factorization of the
// dual (nested dissection on the bodies' initial positions; see mabd_sparse.cu).
struct SparsePlan {
  int64_t np = 0;
  std::vector<int32_t> pa, pb, inc_off, inc;
  std::vector<double> py;
  // multifrontal symbolic
  int32_t nnode = 0;
  std::vector<int32_t> epos, ipos;                       // point ↔ elimination position
  std::vector<int32_t> own_first, nown, fdim, height, parent, ch_off, ch;
  std::vector<int64_t> foff, woff;
  std::vector<int32_t> bnd_off, bnd, ea_off, ea_map;
  std::vector<int32_t> ablk, acoff, acon;
  int64_t front_doubles = 0, w_doubles = 0;
  double flops = 0.0;  // numeric factorization flops per step: 2 × (Σ nn³/6 + nn²mm/2 + nn·mm²/2), the Cholesky count
  // launch schedule, by assembly-tree height
  struct Panel { int64_t potrf, n_potrf, trsm, n_trsm, syrk, n_syrk; };  // offsets into tasks
  struct Level {
    int64_t nodes, n_nodes;        // all nodes of the level (solves), into lev_nodes
    int64_t small, n_small;        // fronts factored in shared memory, into lev_nodes
    int64_t big = 0, n_big = 0;    // fronts factored by panels, into lev_nodes
    std::vector<int64_t> fwd, n_fwd, bwd, n_bwd;  // per MF_SG-chunk group: solve tasks of the big fronts
    int64_t bwdb = 0, n_bwdb = 0;  // backward boundary-product tasks
    int32_t max_f = 0, max_f_small = 0, max_children = 0;
    std::vector<int64_t> ea, n_ea; // per child slot: (parent, column) tasks of big parents
    std::vector<Panel> panels;
  };
  std::vector<Level> levels;
  std::vector<int32_t> lev_nodes, tasks;
  int64_t zero = 0, n_zero = 0;                          // (node, column) tasks of the per-step front zeroing
  std::vector<int64_t> loff;                             // [nnode] inverse diagonal blocks of big fronts
  int64_t linv_doubles = 0;
  int32_t refine = 1;                                    // iterative-refinement passes per step (at most)
  bool syrk_dfma = false;                                // trailing updates on DFMA instead of DMMA (A/B knob)
  double refine_tol = 1e-10;                             // gate: a pass runs if max|r − Sλ| > tol · max|r|
  // five-row hinges: projected points (R13)
  std::vector<int32_t> pslot, pplist;
  std::vector<double> pdr, plim;   // plim: LIM_DOUBLES per slot (joint limits, R14)
  std::vector<double> pgc;         // PGC_DOUBLES per slot (universal / prismatic rows, R17); empty if none
  size_t o_pslot = 0, o_pdr = 0, o_pw = 0, o_pplist = 0, o_pnr = 0, o_plim = 0, o_pgc = 0, o_pg = 0;
  // line Gauss-Seidel (MABD_SOLVER_LINE_GS; gs_build in mabd_sparse.cu)
  std::vector<int32_t> gs_chain_pts, gs_chain_off, gs_color_off;
  int32_t gs_ncolor = 0, gs_sweeps = 0;
  double gs_tol = 0.0;
  size_t o_gs_pts = 0, o_gs_off = 0, o_gs_col = 0, o_gs_fac = 0, o_gs_res = 0;
  int32_t max_f = 0;
  size_t o_pa = 0, o_pb = 0, o_py = 0, o_incoff = 0, o_inc = 0, o_vec = 0, o_vv = 0, o_dqt = 0, o_iters = 0;
  size_t o_F = 0, o_foff = 0, o_fdim = 0, o_nown = 0, o_ownf = 0, o_choff = 0, o_ch = 0, o_eaoff = 0, o_eamap = 0,
         o_bndoff = 0, o_bnd = 0, o_ipos = 0, o_ablk = 0, o_acoff = 0, o_acon = 0, o_linv = 0, o_w = 0, o_woff = 0,
         o_lev = 0, o_tasks = 0, o_loff = 0;
};

// Loop breakers (the paper's Case III, MABD_SOLVER_LOOP_BREAKER; mabd_loop.cu): a forest solved by the chain or tree
// solver plus ≤ LOOP_MAX_PTS breaker points whose multipliers come from a small Schur system formed by forest runs.
constexpr int LOOP_MAX_PTS = 8;
struct LoopPlan {
  bool active = false;
  std::vector<int64_t> keep, breakers;           // joint indices (caller order)
  std::vector<int32_t> pa, pb;                   // breaker points: bodies (caller order, then internal positions)
  std::vector<double> ya, yb;                    // [np][3]
  std::vector<int32_t> fa, fb, fn;               // the forest's joints
  std::vector<double> fya, fyb;
  mabd_joints forest{};
  size_t o_save = 0, o_M = 0, o_lam = 0, o_pa = 0, o_pb = 0, o_ya = 0, o_yb = 0;
};
bool loop_split(const mabd_joints* J, int64_t n, LoopPlan* L, std::string* msg);

struct Plan {
  int64_t n = 0, n_joints = 0, n_dual_rows = 0;
  int32_t solver = 0;
  int32_t launches_per_step = 0;
  int32_t newton_iters = 1;      // Newton iterations per step (K)
  int32_t rotation = 0;          // MABD_ROTATION_* (options.rotation)
  double grav[3] = {0, 0, 0};
  // bodies
  std::vector<Material> mats;
  std::vector<int32_t> mat_id;   // [ld] (empty if one material)
  std::vector<double> mscale;    // [ld] (empty if all 1)
  std::vector<int64_t> perm;     // caller body → internal position
  std::vector<double> frame;     // [n][12] canonical body frame (Q, o) per caller body, or empty (all canonical)
  int64_t ld = 0;                // SoA stride (positions)
  std::vector<double> q_soa, qd_soa;  // [12][ld]
  // chain solver
  int64_t n_windows = 0;
  std::vector<uint32_t> slot_info;   // [ld+1]
  std::vector<double> geo;           // [ng][6]
  std::vector<int32_t> seg_flags, seg_red, long_list, left_iface;
  int64_t n_long = 0;
  bool small_chain = false;          // one window within SMALL_SLOTS slots: small_chain_kernel
  bool step_end_folded = false;      // small_chain_kernel does the step_end bookkeeping (one kernel per step)
  std::vector<BtdLevel> levels;      // levels[0] is BTD level 1 (single part)
  // multi-part chains (multi-GPU, or W parts emulated in one process): see partition_chain()
  struct Part {
    int64_t win_lo = 0, win_hi = 0, long_lo = 0, long_hi = 0;
    int32_t left_open = 0, right_open = 0;
    int64_t n1 = 0, n2 = 0;  // level-1 unknowns (long windows), unknowns of the sequential top
    bool btd1 = false;       // one BTD level (n1 > 256) before the sequential top
  };
  int32_t n_parts = 1, part_lo = 0, part_hi = 1;
  bool use_nccl = false;
  bool host_exchange = false;    // options.host_exchange: the caller all-gathers between mabd_step_exchange_begin/end
  std::vector<Part> parts;
  std::vector<int32_t> local_windows, local_long, part_left_open;
  // loop breakers (Case III) around the chain or tree solver
  LoopPlan loop;
  // tree solver
  TreePlan tree;
  // sparse solver
  SparsePlan sparse;
  // device layout (byte offsets into the workspace)
  size_t workspace_bytes = 0;
  struct Off {
    size_t q, qd, rs, z, wr, mat_id, mscale, mats, hinv, perm, io, err, frame;
    size_t slot_info, geo, seg_flags, seg_red, long_list, left_iface;
    std::vector<size_t> tops, lams;  // per BTD level: tops[0] = chain tops (n_long), lams[i] = level i+1 λ
    size_t all_tops, lam_g, plo, lwin, llong;
    std::vector<size_t> p_tops1, p_lam2, p_scr;
    size_t t_up, t_coff, t_cj, t_wsoff, t_jnpts, t_jchd, t_jy, t_goff, t_glp, t_glo, t_glnl, t_fo, t_fstr, t_f0, t_par, t_uprow, t_shat, t_lam, t_bscr,
        t_ws, t_ptoff, t_ptcode, t_nn, t_rootj, t_rslot, t_xbuf;
  } off{};
};

struct DevPtrs {
  BodyArrays b{};
  double* wr_buf = nullptr;        // [9][ld] wrench storage (b.wr points here once a wrench is set): τ, f, and the
                                   // material point f acts at (the caller's frame origin, in the canonical frame)
  double* frame = nullptr;         // [n][12] canonical frames per caller body (Plan::frame), or null
  double *loop_save = nullptr, *loop_M = nullptr, *loop_lam = nullptr, *loop_ya = nullptr, *loop_yb = nullptr;
  int32_t *loop_pa = nullptr, *loop_pb = nullptr;
  HinvBlk* hinv = nullptr;
  Material* mats = nullptr;
  int64_t* perm = nullptr;
  double* io = nullptr;
  int32_t* err = nullptr;
  uint32_t* slot_info = nullptr;
  double* geo = nullptr;
  int32_t *seg_flags = nullptr, *seg_red = nullptr, *long_list = nullptr, *left_iface = nullptr;
  std::vector<Top*> tops;
  std::vector<double*> lams;
  Top* all_tops = nullptr;
  double* lam_g = nullptr;
  int32_t *part_left_open = nullptr, *local_windows = nullptr, *local_long = nullptr;
  std::vector<Top*> p_tops1;
  std::vector<double*> p_lam2, p_scr;
  void* nccl_comm = nullptr;
  TreeArgs tree{};                   // device pointers of the tree solver
  SparseArgs sparse{};               // device pointers of the sparse solver
  const int32_t* sparse_lev = nullptr;    // level node lists of the sparse schedule
  const int32_t* sparse_tasks = nullptr;  // extend-add / panel task lists
};

// NCCL, loaded on demand (mabd_nccl.cu)
bool nccl_load(std::string* err);
int nccl_unique_id(void* out128);
int nccl_comm_init(void** comm, int world, const void* id128, int rank);
int nccl_allgather_doubles(void* comm, double* buf, size_t count_per_rank, int rank, cudaStream_t st);
int nccl_bcast_ranges(void* comm, double* base, const std::vector<std::pair<int64_t, int64_t>>& ranges,
                      int64_t ld, int ncomp, cudaStream_t st);
void nccl_comm_destroy(void* comm);
const char* nccl_err(int code);
// A step's launch sequence that hits an NCCL failure records its code (nccl_step_failed) and returns
// cudaErrorUnknown; mabd_step then takes the code (nccl_take_step_error, 0 if none) and reports MABD_ENCCL.
int nccl_step_failed(int rc);
int nccl_take_step_error();

mabd_status build_plan(const mabd_bodies* bodies, const mabd_joints* joints, const mabd_options* opts, Plan* p,
                       std::string* msg);
cudaError_t upload_plan(const Plan& p, char* ws, cudaStream_t st, DevPtrs* d);
cudaError_t prefactor_device(const Plan& p, const DevPtrs& d, double h, cudaStream_t st);
cudaError_t reset_err(const DevPtrs& d, cudaStream_t st);
cudaError_t launch_step_end(const Plan& p, const DevPtrs& d, cudaStream_t st);
// nsteps steps of a one-warp chain scene in one launch (Plan::step_end_folded only)
cudaError_t launch_steps_small(const Plan& p, const DevPtrs& d, double h, int32_t nsteps, cudaStream_t st);
cudaError_t loop_step(const Plan& p, const DevPtrs& d, const StepConsts& k, cudaStream_t st,
                      cudaError_t (*forest_step)(const Plan&, const DevPtrs&, const StepConsts&, cudaStream_t));
cudaError_t launch_step(const Plan& p, const DevPtrs& d, double h, int32_t step, cudaStream_t st, int phase = 0);

// tree solver (mabd_tree.cu)
bool tree_build(const mabd_joints* joints, int64_t n, Plan* p, std::vector<int64_t>* pos_of_body, std::string* msg);
cudaError_t tree_step(const Plan& p, const DevPtrs& d, const StepConsts& k, cudaStream_t st);
cudaError_t tree_init();
bool tree_partition(Plan* p, int W, int rank, bool emulate, std::string* msg);

// sparse solver (mabd_sparse.cu)
bool gs_build(const mabd_bodies* bodies, Plan* p, int32_t sweeps, double tol, std::string* msg);
cudaError_t gs_step(const Plan& p, const DevPtrs& d, const StepConsts& k, cudaStream_t st);
bool sparse_build(const mabd_bodies* bodies, const mabd_joints* joints, Plan* p, std::vector<int64_t>* pos_of_body,
                  std::string* msg, bool symbolic = true);
void sparse_layout(Plan* p, const std::function<size_t(size_t)>& take);
cudaError_t sparse_upload(const Plan& p, char* ws, cudaStream_t st, DevPtrs* d);
cudaError_t sparse_init();
cudaError_t sparse_step(const Plan& p, const DevPtrs& d, const StepConsts& k, cudaStream_t st);

}  // namespace mabd
