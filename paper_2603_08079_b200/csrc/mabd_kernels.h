// Kernel launch interface between the host runtime and the CUDA kernels (internal; not part of the ABI).
#pragma once
#include <cuda_runtime.h>

#include "mabd_internal.h"

namespace mabd {

struct ChainArgs {
  BodyArrays b;
  const uint32_t* slot_info;   // [NS+1] slot encoding (mabd_internal.h)
  const double* geo;           // [ng][6] (ȳ_L, ȳ_R); world points for anchor sides
  const int32_t* seg_flags;    // [nseg]
  const int32_t* seg_red;      // [nseg] ordinal among long segments, −1 otherwise
  const int32_t* seg_list;     // [n_items] segment ids of this launch, or null for 0..n_items−1
  int32_t n_items;             // segments of this launch (set by launch_chain)
  const HinvBlk* hinv_tab;     // [n_mat] prefactored H̄⁻¹ per material, or null (per-body mass scale)
  int32_t n_mats;              // entries of b.mats
  Top* top_out;                // REDUCE output, indexed by seg_red
  const double* lam_in;        // FINISH input: level-2 λ [n_long][3]
  int32_t step_end;            // small_chain_kernel: also do the step_end node's bookkeeping (Plan::step_end_folded)
  int32_t nsteps;              // small_chain_kernel with step_end: steps to run in this launch (≤ 1: one)
  StepConsts k;
};

enum : int32_t { BTD_FUSED = 0, BTD_REDUCE = 1, BTD_FINISH = 2 };

struct BtdArgs {
  const Top* top_in;           // level L−1 tops, one per unknown
  const int32_t* left_iface;   // [n_u] or null (then left(u) = u > 0)
  int64_t n_u;
  int32_t mode;
  Top* top_out;                // REDUCE: one per window
  const double* lam_in;        // FINISH: level L+1 λ, one per window
  double* lam_out;             // FUSED/FINISH: λ per unknown
  int32_t right_open;          // multi-part: the last unknown couples to the next part's first unknown
  const double* lam_remote;    // FINISH with right_open: λ of that remote unknown
  StepConsts k;
};

// Sequential reduction of one part's n ≤ 256 unknowns onto {its first unknown, the next part's first unknown}
// (multi-part chains; see mabd_chain.cu "parts").
struct SeqArgs {
  const Top* top_in;           // tops of the level below, one per unknown
  int32_t n;
  int32_t right_open;
  Top* top_out;                // the part's top
  double* scratch;             // [n][27]: D'⁻¹ (6), X (9), B (9), r' (3) per eliminated unknown
  const double* lam_ends;      // FINISH: λ of unknown 0 at [0..2], of the remote unknown at [3..5]
  double* lam_out;             // FINISH: λ per unknown
  StepConsts k;
};
cudaError_t launch_seq_top(const SeqArgs& a, cudaStream_t st);
cudaError_t launch_seq_finish(const SeqArgs& a, cudaStream_t st);

struct TreeArgs {
  BodyArrays b;
  const HinvBlk* hinv_tab;     // per material, or null (per-body mass scale)
  const int32_t* up_joint;
  const int32_t* child_off;
  const int32_t* child_joint;
  const int64_t* ws_off;
  const int32_t* jnpts;
  const int32_t* jchd;
  const double* jy;            // [K][12]
  const int32_t* group_off;
  const int32_t* glev_ptr;
  const int32_t* glev_off;
  const int32_t* glev_nl;      // [levels] end of the bodies with child joints in each level (they come first)
  double* Shat;                // [K][28] child-side condensed dual block of each joint: Ŝ lower triangle (21), r̂ (6)
  double* lam;                 // [K][6]
  double* bscr;                // [21][ld]: R, δq̃ between the passes (structure of arrays)
  double* ws;                  // per-body y, W
  double* f0;                  // per-body front records (G H_b⁻¹ Gᵀ packed lower, own right-hand side)
  const int64_t* fo_off;       // [n] record offset in f0 (−1: none)
  const int32_t* fo_str;       // [n] record stride (element e at fo_off + e·fo_str)
  const int32_t* parent;       // [n] parent body (−1: root)
  const int32_t* up_row;       // [n] row of the body's up joint in its parent's front
  int32_t group0;              // first group of this launch
  int32_t front_rows;          // largest frontal matrix (rows; shared-memory sizing)
  int32_t cap;                 // group capacity (bodies; shared-memory slots of the group kernel)
  const int32_t* pt_off;       // [n+1] per body: its frontal points in pt_code
  const int32_t* pt_code;      // 4·joint + 2·point + (child side)
  const int32_t* body_nn;      // [n] N | nu << 8
  const int32_t* root_joint;   // multi-part: joints from top bodies into bottom groups, by group
  const int32_t* root_slot;    // their slot in xbuf
  double* xbuf;                // multi-part: [parts][rpp][42] condensed root blocks (all-gather buffer)
  int64_t n;                   // bodies
  StepConsts k;
};

enum : int32_t { TREE_UP = 0, TREE_DOWN = 1, TREE_BOTH = 2, TREE_UP_LEVEL = 3, TREE_DOWN_LEVEL = 4 };

// Multifrontal Cholesky of the dual S (sparse solver, mabd_sparse.cu). Fronts are dense column-major f×f
// matrices (f = 3·(own + boundary points)); own columns first, then the boundary rows, both in elimination order.
struct MfArgs {
  double* F;                   // all fronts
  const int64_t* foff;         // [nnode] front offset (doubles)
  const int32_t* fdim;         // [nnode] f (scalar rows)
  const int32_t* nown;         // [nnode] own scalar columns (3 · own points)
  const int32_t* own_first;    // [nnode] first elimination position of the own points
  const int32_t* ch_off;       // [nnode+1] CSR of the assembly-tree children
  const int32_t* ch;
  const int32_t* ea_off;       // [nnode] offset into ea_map
  const int32_t* ea_map;       // per node: front block position in its parent of each boundary point
  const int32_t* bnd_off;      // [nnode] offset into bnd
  const int32_t* bnd;          // boundary points (elimination positions, ascending)
  const int32_t* ipos;         // elimination position → point
  const int32_t* ablk;         // [nblk][3] assembly blocks: node, row block, column block
  const int32_t* acoff;        // [nblk+1] CSR into acon
  const int32_t* acon;         // [ncon][2] contributions: 2·(row point)+side, 2·(column point)+side
  int64_t nblk;
  double* linv;                // inverse of every 64×64 diagonal Cholesky block of the large fronts
  const int64_t* loff;         // [nnode] offset into linv (chunk c of node at loff + 4096·c)
  double* wvec;                // [Σf] per-node solve vectors
  const int64_t* woff;         // [nnode]
};

// Line Gauss-Seidel on the dual (the paper's Case IV; R10): the joint
// points are covered by "chains" (paths in the body graph: consecutive points share a body, no other two do), whose
// dual blocks are block tridiagonal; chains are coloured so that one colour's chains share no body. A sweep relaxes
// the colours in turn, every chain of a colour solved exactly (block Thomas) in parallel, one thread per chain.
struct GsArgs {
  const int32_t* chain_pts;    // [np] points in chain order (chains contiguous, colours contiguous)
  const int32_t* chain_off;    // [nchain+1] into chain_pts
  const int32_t* color_off;    // [ncolor+1] chain ranges per colour
  double* fac;                 // [24][np] per chain position: D'⁻¹ (6, sym), L (9), B (9, coupling to the next)
  unsigned long long* resmax;  // [1 + 2·max_sweeps] (doubles ≥ 0 as bits): [0] max|r|; sweep s: [1 + 2s] max|r − Sλ|,
                               // [2 + 2s] max|Sλ| (the stopping scale of a warm start)
  int32_t ncolor, max_sweeps;
  double tol;                  // stop when max|residual| ≤ tol · max|r|
};

// a projected slot's limit record (plim): [0] lo, [1] hi, [2..4] u_a, [5..7] u_b, [8..10] ȳ_a0 (pivot on body a),
// [11..13] â (unit axis, body a), [14] ρ (> 0 marks a limit slot; 0: the hinge rows of a five-row hinge)
constexpr int LIM_DOUBLES = 15;
// universal / prismatic joints (R17): "general" slots of ≤ 2 rows; constant per row: type (0 unused,
// 1 'point': (A_a d)·(x_a(ȳ_a) − x_b(ȳ_b)) with the slot point's ȳ, 2 'dir': (A_a d)·(A_b e)), d (3), e (3), pad
constexpr int PGC_ROW = 8, PGC_DOUBLES = 2 * PGC_ROW;
// per Newton iteration: for row i, side σ the row's world coefficients w (point part), v, dd (direction part) at
// 18 i + 9 σ; the value at the linearisation point c0[i] at 36 + i
constexpr int PG_DOUBLES = 38;
struct SparseArgs {
  BodyArrays b;
  const HinvBlk* hinv_tab;     // per material, or null (per-body mass scale)
  int64_t n, np;               // bodies, constraint points (3 dual rows each)
  const int32_t* pa;           // [np] body on side a
  const int32_t* pb;           // [np] body on side b or −1 (world)
  const double* py;            // [np][6] ȳ_a, ȳ_b (world point when pb < 0)
  // five-row hinges (R13): the second axis point of such a joint is "projected": its rows are
  // [w0; w1; dummy] with w_i = R_a ΔR_H[row i]ᵀ (i = x̃, z̃) re-evaluated every step, the dummy row decoupled
  // (S = 1, r = 0, λ = 0) so the 3×3 block structure stays
  const int32_t* pslot;        // [np] slot of a projected point, or −1 (null: no projected points)
  const double* pdr;           // [nproj][6] ΔR_H rows x and z (body a's canonical frame); limits: unused
  double* pw;                  // [nproj][6] w0, w1 of this step
  int32_t* pnr;                // [nproj] rows in use this step (2: hinge rows; limits: 1 active, 0 inactive);
                               // the rows beyond are decoupled dummies (S = 1, r = 0, λ = 0)
  const int32_t* pplist;       // [nproj] the projected points
  const double* plim;          // [nproj][LIM_DOUBLES] joint limits (R14), or unused (hinge rows)
  const double* pgc;           // [nproj][PGC_DOUBLES] general-slot rows (R17), type 0 for other slots; or null
  double* pg;                  // [nproj][PG_DOUBLES] general-slot rows at the linearisation point
  int64_t nproj;
  const int32_t* inc_off;      // [n+1] CSR body → incident points (2·point + side)
  const int32_t* inc;
  double *rhs, *lam, *res, *dl, *yy;  // component-major [3][np]: r = C(q̃), λ, residual, correction, solve scratch
  double* vv;                  // [12][n]
  double* dqt;                 // [12][n] δq̃ of the step (predict → rhs, update)
  int32_t* iters;              // [0] refinement passes run in the last step, [1] gate of the current pass
  unsigned long long* rmax;    // [2] max|r − Sλ|, max|r| (bit patterns) for the refinement gate
  const int32_t* gate;         // non-null in a refinement pass's solve kernels: skip when *gate
  double refine_tol;
  MfArgs mf;
  GsArgs gs;
  StepConsts k;
};

size_t cr_smem_bytes();
cudaError_t chain_kernels_init();
cudaError_t launch_chain(const ChainArgs& a, int nblocks, bool finish, cudaStream_t st);
cudaError_t launch_small_chain(const ChainArgs& a, cudaStream_t st);
cudaError_t launch_btd(const BtdArgs& a, int nblocks, cudaStream_t st);
cudaError_t launch_hinv_table(const Material* mats, int nm, double ih2, HinvBlk* out, cudaStream_t st);
cudaError_t launch_gather(const double* q, const double* qd, int64_t ld, const int64_t* perm, int64_t n,
                          const double* frame, double* qo, double* qdo, cudaStream_t st);
cudaError_t launch_scatter_rows(double* dst, int64_t ld, const int64_t* perm, int64_t n, const double* src, int nc,
                                cudaStream_t st);
cudaError_t launch_scatter(double* q, double* qd, int64_t ld, const int64_t* perm, int64_t n, const double* frame,
                           const double* qi, const double* qdi, cudaStream_t st);
cudaError_t launch_wrench_point(double* wr, int64_t ld, const int64_t* perm, int64_t n, const double* frame,
                                cudaStream_t st);

}  // namespace mabd
