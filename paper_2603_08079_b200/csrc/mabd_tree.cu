// Tree solver of the M-ABD step on sm_100a: exact leaf-to-root elimination of the dual (reading A12;
// the exact form of the paper's ABD-ABA, Alg. 2).
//
// Every joint k hangs from a "parent" body p_k and has a child body c_k (or the world, for an anchor);
// C_k = x_p(ȳ_p) − x_c(ȳ_c) (or − p_world), 3 rows per point (ball: 1 point, linear hinge: 2 points).
// Up (deepest bodies first), for body b with child joints X and up joint u, the frontal matrix
//   F = G H_b⁻¹ Gᵀ + diag(Ŝ_k, k ∈ X),  G = stacked ±Γ(ȳ) rows of the points on b,  H_b⁻¹ = diag₄(R)H̄⁻¹diag₄(Rᵀ)
// (blocks ±R P(ȳ,ȳ') Rᵀ, P the constant 3×3 kernels of mabd_device.cuh) is factored on X:
//   Ŝ_u = F_uu − F_uX F_XX⁻¹ F_Xu,  r̂_u = r_u − F_uX F_XX⁻¹ r_X        (condensed child side of joint u)
// Down (root first): λ_X = F_XX⁻¹(r_X − F_Xu λ_u), then qⁿ⁺¹ = q̃ − diag₄(R)H̄⁻¹Σ±Γᵀ Rᵀλ.
// The dual graph of a tree is chordal in this order, so the elimination has no fill (PROBE in SURVEY A12).
//
// Parallel schedule: bodies are grouped into CTA-local subtrees (layer 0, ≤ cap bodies), an
// optional middle layer of ≤ 7-body subtrees of the rest (TREE_MID_CAP), and a top group. One CTA per group runs stages 1-2 and
// the front records a thread per body, the upward levels a warp per body (Gauss-Jordan in registers), the
// downward levels a thread per body, and stage 4; a top group too large for one CTA runs one launch per level.
// Across ranks: each rank takes a contiguous block of the CTA-local subtrees, eliminates
// them, and shares the condensed blocks (Ŝ_u, r̂_u) of the joints into the top through one all-gather; every
// rank then solves the top levels redundantly and finishes its own subtrees.
#include <cuda_runtime.h>

#include <algorithm>
#include <climits>
#include <cstring>
#include <string>
#include <vector>

#include "mabd_device.cuh"
#include "mabd_plan.h"

namespace mabd {

__device__ __forceinline__ void treport(const StepConsts& k, int32_t flag) {
  atomicOr(k.err, flag);
  atomicMin(k.err + 1, k.step_index);
}

// body_nn word: N (child-joint rows) | nu (up-joint rows) << 8 | ext << 16 (the parent lies outside the body's group)
__device__ __forceinline__ int nn_N(int nn) { return nn & 255; }
__device__ __forceinline__ int nn_nu(int nn) { return (nn >> 8) & 255; }
__device__ __forceinline__ bool nn_ext(int nn) { return (nn >> 16) & 1; }

// Per-body shared-memory slots of a CTA-local group [g0, g1): upward, the condensed child side of the body's up
// joint (Ŝ_u lower triangle in tri6 order, then r̂_u); downward, λ_u. A body whose parent lies outside the group
// (ext) also publishes its slot to global memory (Shat: [joint][TSLOT], same layout) and reads λ_u from lam.
// s == nullptr: no slots (the per-level launches of a large top group: everything through global memory).
constexpr int TSLOT = TREE_TSLOT;
__device__ __forceinline__ int tri6(int r, int c) { return r >= c ? r * (r + 1) / 2 + c : c * (c + 1) / 2 + r; }
struct TSlots {
  double* s;
  int g0, g1;
  __device__ __forceinline__ double* at(int b) const { return s + (size_t)(b - g0) * TSLOT; }
  __device__ __forceinline__ double* local(uint32_t i) const { return s + (size_t)i * TSLOT; }
};

// Where the condensed block / λ of each child-joint point of a body lives (uint32, frontal point order):
//   CS_LOCAL  the child body is in the same group: payload = (local index << 1) | point, its slot
//   CS_GLOBAL the child body is in another group: payload = (joint << 1) | point, Shat / lam
//   CS_ANCHOR no child body (world anchor): payload = (joint << 1) | point, λ in lam
enum : uint32_t { CS_LOCAL = 0u, CS_GLOBAL = 1u << 30, CS_ANCHOR = 2u << 30, CS_KIND = 3u << 30 };
constexpr int TNP = TREE_MAXN / 3;  // child-joint points per body (max)
struct TMeta {
  int32_t nn, u;
  int64_t fo, ws;   // front record in f0 (−1: none), y / W in ws
  int64_t pf;       // the parent's front record when the parent is in the same group (−1: publish to Shat)
  int32_t pr, pT;   // row of the up joint in the parent's front; start of the parent's right-hand side
  uint32_t cs[TNP];
  int32_t any_global;  // some child lies in another group (its condensed block is read from Shat)
  int32_t fs;          // record stride: the group's records are interleaved (element e of a record at fo + e·fs)
};

__device__ TMeta tree_meta(const TreeArgs& a, int b, int g0, int g1) {
  TMeta m;
  m.nn = a.body_nn[b];
  m.u = a.up_joint[b];
  m.fo = a.fo_off[b];
  m.fs = a.fo_str[b];
  m.ws = a.ws_off[b];
  const int32_t* pc = a.pt_code + a.pt_off[b];
  const int N = nn_N(m.nn);
  const int p = a.parent[b];
  m.pf = -1;
  m.pr = a.up_row[b];
  m.pT = 0;
  if (p >= g0 && p < g1) {
    const int pn = a.body_nn[p], Mp = nn_N(pn) + nn_nu(pn);
    m.pf = a.fo_off[p];
    m.pT = Mp * (Mp + 1) / 2;
  }
  m.any_global = 0;
#pragma unroll
  for (int i = 0; i < TNP; ++i) {
    uint32_t v = 0;
    if (3 * i < N) {
      const int code = pc[i];
      const uint32_t kp = (uint32_t)(code >> 1);  // (joint << 1) | point
      const int c = a.jchd[code >> 2];
      v = c < 0 ? (CS_ANCHOR | kp) : (c >= g0 && c < g1) ? ((uint32_t)(c - g0) << 1 | (kp & 1u)) : (CS_GLOBAL | kp);
      if ((v & CS_KIND) == CS_GLOBAL) m.any_global = 1;
    }
    m.cs[i] = v;
  }
  return m;
}

__device__ const double kZeroSlot[TSLOT] = {};  // the condensed block of an anchor (none)

// Entry t of a condensed block (tri6 index < 21: Ŝ_u row r ≥ column c; 21 + r: r̂_u row r) added into the parent's
// front record: Ŝ_u lands on the parent's diagonal block of joint u (rows pr.., packed lower), r̂_u on its
// right-hand side. Each entry has exactly one writer (its child), after the parent's record was written.
__device__ __forceinline__ int64_t tree_push_at(const TMeta& m, int r, int c, bool rhs) {
  const int row = m.pr + r;
  return m.pf + (int64_t)m.fs * (rhs ? m.pT + row : row * (row + 1) / 2 + m.pr + c);  // same group: same stride
}

// Body b's front record (element e at f0[fo + e·fs], interleaved with the group's other records so that a thread per
// body writes them coalesced): the packed lower triangle of F = G H_b⁻¹ Gᵀ (M×M, (i, j) at i(i+1)/2 + j),
// then its own side of the right-hand side (M): +x_b(ȳ) (child-joint points; − p_world for an anchor),
// −x_b(ȳ) (up-joint points), at q̃. With slots, the condensed blocks of leaf children in the group (already in
// their slots) are added here; other children's are added later (pushed by the child, or read from Shat).
__device__ void tree_assemble(const TreeArgs& a, int b, const TMeta& m, const double* R, const double* qt,
                              const HinvBlk& H, const TSlots& sl, const TMeta* meta) {
  const int N = nn_N(m.nn), M = N + nn_nu(m.nn), npt = M / 3, T = M * (M + 1) / 2;
  const int32_t* pc = a.pt_code + a.pt_off[b];
  double* f = a.f0 + m.fo;
  const int64_t fs = m.fs;
  // every point's code, ȳ and world point first (independent loads, two round trips in all)
  constexpr int NPT = TNP + 2;
  int code[NPT];
  double yy[NPT][6];
  const double* leaf[NPT];  // a leaf child's slot (child-joint points), or null
  for (int i = 0; i < npt; ++i) {
    code[i] = pc[i];
    leaf[i] = nullptr;
    if (sl.s != nullptr && 3 * i < N) {
      const uint32_t c = m.cs[i];
      const uint32_t id = (c & ~CS_KIND) >> 1;
      if ((c & CS_KIND) == CS_LOCAL && nn_N(meta[id].nn) == 0) leaf[i] = sl.local(id);
    }
  }
  for (int i = 0; i < npt; ++i) {
    const double* yi = a.jy + 12 * (int64_t)(code[i] >> 2) + 6 * (code[i] & 1) + 3 * ((code[i] >> 1) & 1);
#pragma unroll
    for (int e = 0; e < 3; ++e) {
      yy[i][e] = yi[e];
      yy[i][3 + e] = (code[i] & 1) ? 0.0 : yi[6 + e];  // anchor world point (child side of a parent point)
    }
  }
  for (int i = 0; i < npt; ++i) {
    const int ci = code[i];
    const int si = ci & 1, pi = (ci >> 1) & 1;
    const double* yi = yy[i];
    double x[3];
    point_pos(qt, yi, x);
    const bool anchor = !si && a.jchd[ci >> 2] < 0;
    const double* li = leaf[i];
#pragma unroll
    for (int e = 0; e < 3; ++e)
      f[fs * (T + 3 * i + e)] = si ? -x[e] : (anchor ? x[e] - yi[3 + e] : x[e] + (li ? li[21 + 3 * pi + e] : 0.0));
    for (int j = 0; j <= i; ++j) {
      const int cj = code[j];
      const double* yj = yy[j];
      double P[9], Bk[9];
      pblock(H, yi, yj, P);
      rot_conj(R, P, Bk);
      const double sg = ((ci ^ cj) & 1) ? -1.0 : 1.0;
      const bool same = li != nullptr && (ci >> 2) == (cj >> 2);  // both points of the same leaf child's joint
      const int pj = (cj >> 1) & 1;
#pragma unroll
      for (int r = 0; r < 3; ++r)
#pragma unroll
        for (int c = 0; c < 3; ++c)
          if (i > j || r >= c)
            f[fs * ((3 * i + r) * (3 * i + r + 1) / 2 + 3 * j + c)] =
                sg * Bk[3 * r + c] + (same ? li[tri6(3 * pi + r, 3 * pj + c)] : 0.0);
    }
  }
}

// Stages 1-2 of body b (no tree dependency): R, q̃ and H_b⁻¹'s blocks out, R and δq̃ → bscr.
__device__ void tree_predict_core(const TreeArgs& a, int b, double* R, double* qt, HinvBlk& H) {
  const StepConsts& k = a.k;
  const int64_t ld = a.b.ld;
  double q[12], qd[12], dqt[12];
#pragma unroll
  for (int c = 0; c < 12; ++c) {
    q[c] = a.b.q[c * ld + b];
    qd[c] = a.b.qd[c * ld + b];
  }
  const int mid = a.b.mat_id ? a.b.mat_id[b] : 0;
  const double msc = a.b.mscale ? a.b.mscale[b] : 1.0;
  const Material M = a.b.mats[mid];
  if (a.hinv_tab)
    H = a.hinv_tab[mid];
  else
    hinv_blocks(M, msc, k.ih2, H);
  double W[9];
  const double* Wp = load_wrench(a.b, b, W);
  if (!(k.lp ? predict_body<true>(q, qd, M, msc, H, k.ih, k.grav, R, dqt, Wp)
             : predict_body<false>(q, qd, M, msc, H, k.ih, k.grav, R, dqt, Wp)))
    treport(k, ERR_NONFINITE);
  double* sc = a.bscr + b;  // [21][ld]: component c at sc[c·ld]
#pragma unroll
  for (int c = 0; c < 9; ++c) sc[c * ld] = R[c];
#pragma unroll
  for (int c = 0; c < 12; ++c) sc[(9 + c) * ld] = dqt[c];
#pragma unroll
  for (int c = 0; c < 12; ++c) qt[c] = q[c] + dqt[c];
}

// R, q̃ = qⁿ + δq̃ (bscr) and the blocks of H_b⁻¹ of body b after its stages 1-2.
__device__ void tree_reload(const TreeArgs& a, int b, double* R, double* qt, HinvBlk& H) {
  const int64_t ld = a.b.ld;
  const double* sc = a.bscr + b;  // [21][ld]: component c at sc[c·ld]
#pragma unroll
  for (int c = 0; c < 9; ++c) R[c] = sc[c * ld];
#pragma unroll
  for (int c = 0; c < 12; ++c) qt[c] = a.b.q[c * ld + b] + sc[(9 + c) * ld];
  const int mid = a.b.mat_id ? a.b.mat_id[b] : 0;
  if (a.hinv_tab)
    H = a.hinv_tab[mid];
  else
    hinv_blocks(a.b.mats[mid], a.b.mscale ? a.b.mscale[b] : 1.0, a.k.ih2, H);
}

// A leaf (no child joints) of a group condenses its up joint right away: N = 0 leaves nothing to eliminate, so
// Ŝ_u = F_uu = Σ (−1)² R P(ȳ_i, ȳ_j) Rᵀ over the up joint's child-side points and r̂_u = r_u = −x_b(ȳ_i) at q̃
// → its slot (and Shat when the parent is in another group).
__device__ void tree_leaf(const TreeArgs& a, int b, const TMeta& m, const TSlots& sl, const double* R,
                          const double* qt, const HinvBlk& H) {
  const int nu = nn_nu(m.nn);
  if (nu == 0) return;
  const double* yc = a.jy + 12 * (int64_t)m.u + 6;
  double* o = sl.at(b);
  for (int pi = 0; pi < nu / 3; ++pi) {
    for (int pj = 0; pj <= pi; ++pj) {
      double P[9], Bk[9];
      pblock(H, yc + 3 * pi, yc + 3 * pj, P);
      rot_conj(R, P, Bk);
#pragma unroll
      for (int r = 0; r < 3; ++r)
#pragma unroll
        for (int c = 0; c < 3; ++c)
          if (3 * pi + r >= 3 * pj + c) o[tri6(3 * pi + r, 3 * pj + c)] = Bk[3 * r + c];
    }
    double x[3];
    point_pos(qt, yc + 3 * pi, x);
#pragma unroll
    for (int e = 0; e < 3; ++e) o[21 + 3 * pi + e] = -x[e];
  }
  if (nn_ext(m.nn)) {
    double* g = a.Shat + TSLOT * (int64_t)m.u;
    for (int t = 0; t < TSLOT - 1; ++t) g[t] = o[t];
  }
}

#ifdef MABD_EXP_TCLOCK  // developer probe: global-timer marks of every CTA's phases (read by mabd_dbg_tclk)
constexpr int TCLK_SLOTS = 64, TCLK_CTAS = 512;
__device__ unsigned long long g_tclk[3 * TCLK_CTAS * TCLK_SLOTS];
#define TMARK(slot)                                                                                        \
  do {                                                                                                     \
    if (threadIdx.x == 0 && blockIdx.x < TCLK_CTAS && (slot) < TCLK_SLOTS) {                               \
      unsigned long long t_;                                                                               \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                                               \
      g_tclk[(MODE * TCLK_CTAS + blockIdx.x) * TCLK_SLOTS + (slot)] = t_;                                  \
    }                                                                                                      \
  } while (0)
#else
#define TMARK(slot)
#endif
#ifdef MABD_EXP_TCLOCK
__device__ __forceinline__ void tmark_at(int slot) {  // CTA 0, mode slot range 40..59 of mode 0's CTA 0 row
  unsigned long long t_;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));
  g_tclk[slot] = t_;
}
#define EMARK(cond, slot) \
  if (cond) tmark_at(slot)
#else
#define EMARK(cond, slot)
#endif

// Upward elimination at body b by one warp, in registers: lane j holds column j of the augmented front [F | r]
// (lane M: r), read from the front record, plus the children's condensed blocks (Ŝ_c on their diagonal blocks,
// r̂_c on their right-hand-side rows). Gauss-Jordan over the N child-joint columns, pivot column broadcast by
// shuffles; F is symmetric positive definite on X, so no pivoting is needed. Afterwards the columns hold
//   rows < N:  F_XX⁻¹ F_Xu = W (lanes N..M−1),  F_XX⁻¹ r_X = y (lane M)
//   rows ≥ N:  Ŝ_u = F_uu − F_uX F_XX⁻¹ F_Xu (lanes N..M−1),  r̂_u = r_u − F_uX F_XX⁻¹ r_X (lane M).
// MX: the front size rounded up to a multiple of 6, so that every loop is fully unrolled (register indices).
template <int MX>
__device__ __forceinline__ void tree_elim(const TreeArgs& a, int b, int lane, const TMeta* mp, const TSlots& sl,
                                          double* colbuf) {
  const StepConsts& k = a.k;
  const int nn = mp->nn, N = nn_N(nn), nu = nn_nu(nn), M = N + nu, u = mp->u;
  const double* f = a.f0 + mp->fo;
  const int64_t fs = mp->fs;
  const int T = M * (M + 1) / 2, tl = lane * (lane + 1) / 2;
#ifdef MABD_EXP_TCLOCK
  const bool probe = blockIdx.x == 0 && lane == 0 && b == sl.g1 - 1 && sl.s != nullptr;
#endif
  EMARK(probe, 40);
  double v[MX];
#pragma unroll
  for (int i = 0; i < MX; ++i) {
    double x = 0.0;
    if (i < M && lane <= M) x = f[fs * (lane == M ? T + i : (i >= lane ? i * (i + 1) / 2 + lane : tl + i))];
    v[i] = x;
  }
  EMARK(probe && v[0] != 1e300, 41);
  if (mp->any_global && (lane < N || lane == M)) {  // condensed blocks of children in other groups (Shat); the
                                                    // children in this group pushed theirs into the record
    const uint32_t cj = lane < N ? mp->cs[lane / 3] : 0u;
    const int rj = 3 * (int)(cj & 1u) + lane % 3;
#pragma unroll
    for (int i = 0; i < MX; ++i) {
      const uint32_t ci = i < N ? mp->cs[i / 3] : CS_ANCHOR;
      const uint32_t kind = ci & CS_KIND, id = (ci & ~CS_KIND) >> 1;
      const double* src = kind == CS_GLOBAL ? a.Shat + TSLOT * (int64_t)id : kZeroSlot;
      const int ri = 3 * (int)(ci & 1u) + i % 3;
      const double x = src[lane == M ? 21 + ri : tri6(ri, rj)];
      v[i] += (lane == M || ((ci ^ cj) & ~1u) == 0u) ? x : 0.0;  // same child joint as this column
    }
  }
  // the parent's record entries this lane will add to (static addresses, no other writer): loaded now, so the
  // push at the end is a plain store instead of a read-modify-write on the critical path
  const int cu = lane - N;  // this lane's column of u (0 ≤ cu < nu), or nu for the right-hand side
  const bool pushes = u >= 0 && mp->pf >= 0 && cu >= 0 && cu <= nu;
  double pre[6];
#pragma unroll
  for (int r = 0; r < 6; ++r)
    pre[r] = (pushes && r < nu && (cu == nu || r >= cu)) ? a.f0[tree_push_at(*mp, r, cu, cu == nu)] : 0.0;
  // Pivot loop kept rolled (code size: every step runs the same instructions): the registers rotate by one row per
  // step so that the pivot row is always v[0]; after N steps, v[i] holds original row (i + N) mod MX, i.e.
  // rows N..M−1 (Ŝ_u / r̂_u) at v[0..nu) and rows 0..N−1 (W / y) at v[MX−N..MX).
  // Pivots in 3×3 blocks (a joint point's rows; N is a multiple of 3): block K = rows kb..kb+2 (v[0..2] after the
  // rotation), columns in lanes kb..kb+2. Per lane (column j): t = F_KK⁻¹ F_Kj, F_ij −= F_iK t for i ∉ K, and the
  // block's rows become t: three scalar Gauss-Jordan steps at once, one broadcast and one reciprocal instead of three.
  // The pivot lanes write their columns row-interleaved (row i of the three at colbuf[4i..4i+2]) so that every
  // lane reads a row's three coefficients with one 16-byte and one 8-byte broadcast load.
  bool ok = true;
  for (int kb = 0; kb < N; kb += 3) {
    const int pl = lane - kb;
    if (pl >= 0 && pl < 3) {
#pragma unroll
      for (int i = 0; i < MX; ++i) colbuf[4 * i + pl] = v[i];
    }
    __syncwarp();
    double B[9];  // F_KK, row-major: B[3a + b] = F[kb + a][kb + b]
#pragma unroll
    for (int a3 = 0; a3 < 3; ++a3) {
      const double2 w = *reinterpret_cast<const double2*>(colbuf + 4 * a3);
      B[3 * a3] = w.x;
      B[3 * a3 + 1] = w.y;
      B[3 * a3 + 2] = colbuf[4 * a3 + 2];
    }
    const double C00 = B[4] * B[8] - B[5] * B[7], C01 = B[5] * B[6] - B[3] * B[8], C02 = B[3] * B[7] - B[4] * B[6];
    const double det = B[0] * C00 + B[1] * C01 + B[2] * C02;
    ok = ok && B[0] > 0.0 && B[0] * B[4] - B[1] * B[3] > 0.0 && det > 0.0;
    const double id = fast_rcp(det > 0.0 ? det : 1.0);
    // adj(B) rows: adj[a][b] = cofactor C[b][a]
    const double C10 = B[2] * B[7] - B[1] * B[8], C11 = B[0] * B[8] - B[2] * B[6], C12 = B[1] * B[6] - B[0] * B[7];
    const double C20 = B[1] * B[5] - B[2] * B[4], C21 = B[2] * B[3] - B[0] * B[5], C22 = B[0] * B[4] - B[1] * B[3];
    double t0 = (C00 * v[0] + C10 * v[1] + C20 * v[2]) * id;
    double t1 = (C01 * v[0] + C11 * v[1] + C21 * v[2]) * id;
    double t2 = (C02 * v[0] + C12 * v[1] + C22 * v[2]) * id;
    {  // one refinement step: the adjugate solve alone loses accuracy on stiff hinge blocks
      const double r0 = v[0] - (B[0] * t0 + B[1] * t1 + B[2] * t2);
      const double r1 = v[1] - (B[3] * t0 + B[4] * t1 + B[5] * t2);
      const double r2 = v[2] - (B[6] * t0 + B[7] * t1 + B[8] * t2);
      t0 += (C00 * r0 + C10 * r1 + C20 * r2) * id;
      t1 += (C01 * r0 + C11 * r1 + C21 * r2) * id;
      t2 += (C02 * r0 + C12 * r1 + C22 * r2) * id;
    }
#pragma unroll
    for (int i = 3; i < MX; ++i) {  // rows beyond M are zero and stay zero
      const double2 w = *reinterpret_cast<const double2*>(colbuf + 4 * i);
      const double c2 = colbuf[4 * i + 2];
      v[i - 3] = v[i] - (w.x * t0 + w.y * t1 + c2 * t2);
    }
    v[MX - 3] = t0;
    v[MX - 2] = t1;
    v[MX - 1] = t2;
    __syncwarp();  // every lane has read the block before the next block's pivot lanes overwrite it
  }
  EMARK(probe && v[MX - 1] != 1e300, 43);
  if (!ok && lane == 0) treport(k, ERR_SINGULAR);
  if (cu < 0 || cu > nu) return;
  double* ws = a.ws + mp->ws;  // y [N], W [N][nu] (row-major)
#pragma unroll
  for (int i = 0; i < MX; ++i) {
    const int r = i - (MX - N);  // row r < N of y / W
    if (r >= 0) ws[cu == nu ? r : N + r * nu + cu] = v[i];
  }
  if (u >= 0) {  // condensed child side of the up joint → the parent's record, or Shat (parent in another group)
    const TMeta& m = *mp;
#pragma unroll
    for (int r = 0; r < 6; ++r) {
      if (r >= nu) break;
      const double x = v[r];
      if (cu == nu || r >= cu) {
        if (m.pf >= 0)
          a.f0[tree_push_at(m, r, cu, cu == nu)] = pre[r] + x;
        else
          a.Shat[TSLOT * (int64_t)u + (cu == nu ? 21 + r : tri6(r, cu))] = x;
      }
    }
  } else if (sl.s == nullptr && cu == nu) {  // root of the per-level schedule: λ_X = y
#pragma unroll
    for (int i = 0; i < MX; ++i) {
      const int r = i - (MX - N);
      if (r >= 0) {
        const uint32_t kp = mp->cs[r / 3] & ~CS_KIND;
        a.lam[6 * (int64_t)(kp >> 1) + 3 * (kp & 1u) + r % 3] = v[i];
      }
    }
  }
}

__device__ __forceinline__ void tree_up_warp(const TreeArgs& a, int b, int lane, const TMeta* mp, const TSlots& sl,
                                             double* colbuf) {
  const int M = nn_N(mp->nn) + nn_nu(mp->nn);
  switch ((M + 5) / 6) {  // the front size rounded up to a multiple of 6 rows
    case 0:
    case 1: tree_elim<6>(a, b, lane, mp, sl, colbuf); break;
    case 2: tree_elim<12>(a, b, lane, mp, sl, colbuf); break;
    case 3: tree_elim<18>(a, b, lane, mp, sl, colbuf); break;
    case 4: tree_elim<24>(a, b, lane, mp, sl, colbuf); break;
    default: tree_elim<30>(a, b, lane, mp, sl, colbuf); break;
  }
  EMARK(blockIdx.x == 0 && lane == 0 && b == sl.g1 - 1 && sl.s != nullptr, 44);
  __syncwarp();
}

// λ_u of body b (zero-padded to 6 rows): its slot (the parent is in the group) or global memory.
__device__ __forceinline__ void tree_lambda_up(const TreeArgs& a, int b, const TMeta& m, const TSlots& sl,
                                               double* lu) {
  const int nu = nn_nu(m.nn);
  const double* src = (sl.s == nullptr || nn_ext(m.nn)) ? a.lam + 6 * (int64_t)m.u : sl.at(b);
#pragma unroll
  for (int r = 0; r < 6; ++r) lu[r] = r < nu ? src[r] : 0.0;
}

// λ of child-joint point i of a body (source code c), 3 rows
__device__ __forceinline__ double* tree_lam_at(const TreeArgs& a, const TSlots& sl, uint32_t c) {
  const uint32_t id = (c & ~CS_KIND) >> 1, pp = c & 1u;
  return (c & CS_KIND) == CS_LOCAL ? sl.local(id) + 3 * pp : a.lam + 6 * (int64_t)id + 3 * pp;
}

// Downward step at a body with child joints (one thread): λ_X = y − W λ_u → the child bodies' slots (or lam).
// NP child points (exact size: every load unconditional and issued together).
template <int NP>
__device__ __forceinline__ void tree_lambda_np(const TreeArgs& a, const TMeta& m, const TSlots& sl, const double* ws,
                                               const double* lu) {
  constexpr int N = 3 * NP;
  const int nu = nn_nu(m.nn);
  double lx[N];
#pragma unroll
  for (int r = 0; r < N; ++r) {
    double v = ws[r];
#pragma unroll
    for (int c = 0; c < 6; ++c) v -= ws[N + r * nu + (c < nu ? c : 0)] * lu[c];  // lu[c ≥ nu] = 0
    lx[r] = v;
  }
#pragma unroll
  for (int i = 0; i < NP; ++i) {
    double* d = tree_lam_at(a, sl, m.cs[i]);
#pragma unroll
    for (int e = 0; e < 3; ++e) d[e] = lx[3 * i + e];
  }
}

__device__ void tree_lambda(const TreeArgs& a, int b, const TMeta& m, const TSlots& sl) {
  const double* ws = a.ws + m.ws;
  double lu[6];
  tree_lambda_up(a, b, m, sl, lu);
  switch (nn_N(m.nn) / 3) {
    case 1: tree_lambda_np<1>(a, m, sl, ws, lu); break;
    case 2: tree_lambda_np<2>(a, m, sl, ws, lu); break;
    case 3: tree_lambda_np<3>(a, m, sl, ws, lu); break;
    case 4: tree_lambda_np<4>(a, m, sl, ws, lu); break;
    case 5: tree_lambda_np<5>(a, m, sl, ws, lu); break;
    case 6: tree_lambda_np<6>(a, m, sl, ws, lu); break;
    case 7: tree_lambda_np<7>(a, m, sl, ws, lu); break;
    case 8: tree_lambda_np<8>(a, m, sl, ws, lu); break;
    default: break;
  }
}

// Stage 4 at body b once every λ of its joints is known (one thread): qⁿ⁺¹ = q̃ − diag₄(R)H̄⁻¹ Σ ±Γᵀ Rᵀλ.
__device__ void tree_update(const TreeArgs& a, int b, const TMeta& m, const TSlots& sl) {
  const StepConsts& k = a.k;
  const int64_t ld = a.b.ld;
  const int N = nn_N(m.nn), nu = nn_nu(m.nn);
  const int32_t* pcode = a.pt_code + a.pt_off[b];
  const double* sc = a.bscr + b;  // [21][ld]: component c at sc[c·ld]
  double R[9];
#pragma unroll
  for (int c = 0; c < 9; ++c) R[c] = sc[c * ld];
  HinvBlk H;
  {
    const int mid = a.b.mat_id ? a.b.mat_id[b] : 0;
    if (a.hinv_tab)
      H = a.hinv_tab[mid];
    else
      hinv_blocks(a.b.mats[mid], a.b.mscale ? a.b.mscale[b] : 1.0, k.ih2, H);
  }
  double lu[6];
  tree_lambda_up(a, b, m, sl, lu);
  double gq[12];
#pragma unroll
  for (int c = 0; c < 12; ++c) gq[c] = 0.0;
  if (N > 0) {
#pragma unroll
    for (int i = 0; i < TNP; ++i) {  // child-joint points (this body is their parent side, sign +); loads unguarded
      const int ii = 3 * i < N ? i : 0;
      const int code = pcode[ii];
      const double* lam = tree_lam_at(a, sl, m.cs[ii]);
      const double s = 3 * i < N ? 1.0 : 0.0;
      const double l3[3] = {s * lam[0], s * lam[1], s * lam[2]};
      double w[3];
      mat3t_vec(R, l3, w);
      add_point_force(gq, a.jy + 12 * (int64_t)(code >> 2) + 3 * ((code >> 1) & 1), w, 1.0);
    }
  }
#pragma unroll
  for (int pp = 0; pp < 2; ++pp) {  // up-joint points (this body is their child side, sign −)
    if (3 * pp >= nu) break;
    double w[3];
    mat3t_vec(R, lu + 3 * pp, w);
    add_point_force(gq, a.jy + 12 * (int64_t)m.u + 6 + 3 * pp, w, -1.0);
  }
  double uu[12];
  hinv_apply(H, gq, uu);
  // every load before the first store: q, q̇ and bscr may alias as far as the compiler knows, so a load after a
  // store would wait for it (12 serialized round trips)
  double q[12], dq[12];
#pragma unroll
  for (int c = 0; c < 12; ++c) {
    q[c] = a.b.q[c * ld + b];
    dq[c] = sc[(9 + c) * ld];
  }
#pragma unroll
  for (int kb = 0; kb < 4; ++kb) {
    double c3[3];
    mat3_vec(R, uu + 3 * kb, c3);
#pragma unroll
    for (int e = 0; e < 3; ++e) dq[3 * kb + e] -= c3[e];  // δq = δq̃ − correction
  }
  if (k.niter == 1) {
#pragma unroll
    for (int c = 0; c < 12; ++c) {
      a.b.q[c * ld + b] = q[c] + dq[c];
      a.b.qd[c * ld + b] = dq[c] * k.ih;
    }
  } else {  // K > 1: v ← v − δq/h + h·grav (launch_step in mabd_plan.cu)
    double v[12];
#pragma unroll
    for (int c = 0; c < 12; ++c) v[c] = a.b.qd[c * ld + b];
#pragma unroll
    for (int c = 0; c < 12; ++c) {
      a.b.q[c * ld + b] = q[c] + dq[c];
      a.b.qd[c * ld + b] = v[c] - dq[c] * k.ih + (c >= 9 ? k.h * k.grav[c - 9] : 0.0);
    }
  }
}

// One level of a large top group over the whole GPU (no slots: everything through global memory): upward a warp
// per body, downward a thread per body (λ of its child joints, then stage 4).
__global__ void __launch_bounds__(512) tree_level_kernel(TreeArgs a, int mode) {
  __shared__ TMeta sm[16];
  __shared__ __align__(16) double colbuf[16][4 * (TREE_MAXN + 6)];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  const int l = a.group0;
  const TSlots none{nullptr, 0, 0};
  if (mode == TREE_UP_LEVEL) {
    const int b = a.glev_off[l] + blockIdx.x * nw + warp;
    if (b >= a.glev_off[l + 1]) return;
    if (lane == 0) sm[warp] = tree_meta(a, b, 0, 0);
    __syncwarp();
    tree_up_warp(a, b, lane, &sm[warp], none, colbuf[warp]);
  } else {
    const int b = a.glev_off[l] + blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= a.glev_off[l + 1]) return;
    const TMeta m = tree_meta(a, b, 0, 0);
    tree_lambda(a, b, m, none);
    tree_update(a, b, m, none);
  }
}



// A CTA-local group (one CTA per group; the top group as a single CTA when it fits). Shared memory: the slots and
// the per-body metadata of the group. Upward: stages 1-2 with the front records (or, for leaves, the condensed
// blocks) of every body at once, then the levels with child joints, deepest first, a warp per body (those bodies
// come first in each level: [glev_off[l], glev_nl[l])). Downward: λ level by level, shallowest first, a thread
// per body, then stage 4 for every body at once.
// UP launches of the bottom groups carry extra CTAs (blockIdx.x ≥ ngroups) that prepare the top section
// [top0, n): stages 1-2 and front records, a thread per body, on the SMs the groups leave idle. The groups of the
// top section (prepared != 0) then only load their metadata in the first phase.
#ifndef MABD_TREE_THREADS
#define MABD_TREE_THREADS 512
#endif
constexpr int TREE_THREADS = MABD_TREE_THREADS;  // threads per group CTA (≥ cap: one body per thread in phase A)
template <int MODE>
__global__ void __launch_bounds__(TREE_THREADS, 1) tree_group_kernel(TreeArgs a, int ngroups, int top0, int prepared) {
  extern __shared__ double tsm[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  if ((int)blockIdx.x >= ngroups) {
    const int b = top0 + ((int)blockIdx.x - ngroups) * blockDim.x + threadIdx.x;
    if (b < a.n) {
      double R[9], qt[12];
      HinvBlk H;
      tree_predict_core(a, b, R, qt, H);
      const TMeta m = tree_meta(a, b, 0, 0);
      if (m.fo >= 0) tree_assemble(a, b, m, R, qt, H, TSlots{nullptr, 0, 0}, nullptr);
    }
    return;
  }
  const int g = a.group0 + blockIdx.x;
  const int g0 = a.group_off[g], g1 = a.group_off[g + 1];
  const int l0 = a.glev_ptr[g], l1 = a.glev_ptr[g + 1] - 1;  // levels l ∈ [l0, l1), deepest first
  const TSlots sl{tsm, g0, g1};
  TMeta* meta = reinterpret_cast<TMeta*>(tsm + (size_t)a.cap * TSLOT);
  double* colbuf = reinterpret_cast<double*>(meta + a.cap) + (size_t)warp * 4 * (TREE_MAXN + 6);  // pivot block
  TMARK(0);
  // one body per thread (a group has at most cap ≤ blockDim bodies): stages 1-2 and the leaves' condensed blocks,
  // then (after the leaves' slots are complete) the front records of the bodies with child joints
  const int bb = g0 + threadIdx.x;
  const bool mine = bb < g1, prep = MODE != TREE_DOWN && !prepared;
  if (mine) {
    const TMeta m = tree_meta(a, bb, g0, g1);
    meta[bb - g0] = m;
    if (prep) {
      double R[9], qt[12];
      HinvBlk H;
      tree_predict_core(a, bb, R, qt, H);
      if (nn_N(m.nn) == 0) tree_leaf(a, bb, m, sl, R, qt, H);
    }
  }
  __syncthreads();
  TMARK(31);
  if (prep) {
    if (mine && nn_N(meta[bb - g0].nn) > 0) {  // R, q̃, H_b⁻¹ reloaded (not held across the barrier)
      double R[9], qt[12];
      HinvBlk H;
      tree_reload(a, bb, R, qt, H);
      tree_assemble(a, bb, meta[bb - g0], R, qt, H, sl, meta);
    }
    __syncthreads();
  }
  TMARK(1);
  if (MODE != TREE_DOWN) {
    for (int l = l0; l < l1; ++l) {
      const int e = a.glev_nl[l];
      if (e == a.glev_off[l]) continue;  // leaves only (uniform across the CTA)
      for (int b = a.glev_off[l] + warp; b < e; b += nw) tree_up_warp(a, b, lane, meta + (b - g0), sl, colbuf);
      __syncthreads();
      TMARK(2 + l - l0);
    }
  }
  if (MODE != TREE_UP) {
    TMARK(32);
    for (int l = l1 - 1; l >= l0; --l) {
      const int e = a.glev_nl[l];
      if (e == a.glev_off[l]) continue;
      for (int b = a.glev_off[l] + threadIdx.x; b < e; b += blockDim.x) tree_lambda(a, b, meta[b - g0], sl);
      __syncthreads();
      TMARK(33 + l1 - 1 - l);
    }
    for (int b = g0 + threadIdx.x; b < g1; b += blockDim.x) tree_update(a, b, meta[b - g0], sl);
    __syncthreads();
    TMARK(63);
  }
}

// Multi-part split: the condensed child side (slot layout, TSLOT doubles) of every joint from a top body into a
// bottom group, packed by the part owning the group into its block of the all-gather buffer, then unpacked by every
// part into Shat for the top section. Root entries [r0, r1) are those of a part's groups.
__global__ void tree_pack_kernel(TreeArgs a, int r0, int r1) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const int r = r0 + i / TSLOT, e = i % TSLOT;
  if (r >= r1) return;
  const int u = a.root_joint[r];
  a.xbuf[(size_t)a.root_slot[r] * TSLOT + e] = a.Shat[TSLOT * (int64_t)u + e];
}
__global__ void tree_unpack_kernel(TreeArgs a, int nroot) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const int r = i / TSLOT, e = i % TSLOT;
  if (r >= nroot) return;
  a.Shat[TSLOT * (int64_t)a.root_joint[r] + e] = a.xbuf[(size_t)a.root_slot[r] * TSLOT + e];
}

constexpr size_t TREE_SMEM_MAX = 227 * 1024;  // dynamic shared memory per CTA (sm_100a opt-in maximum)

// Shared memory of the group kernel: slots and metadata for cap bodies.
size_t tree_group_smem(int cap) {
  return (sizeof(double) * TSLOT + sizeof(TMeta)) * (size_t)cap + sizeof(double) * 4 * (TREE_MAXN + 6) * (TREE_THREADS / 32);
}

template <int MODE>
static cudaError_t launch_group(const TreeArgs& a, int g_lo, int g_hi, const TreePlan& t, cudaStream_t st,
                                bool prepare_top = false) {
  const int ng = std::max(0, g_hi - g_lo);
  const int top0 = t.group_off[t.n_bottom];
  const int nprep = prepare_top ? (int)((a.n - top0 + TREE_THREADS - 1) / TREE_THREADS) : 0;
  if (ng + nprep == 0) return cudaSuccess;
  TreeArgs b = a;
  b.group0 = g_lo;
  const int prepared = g_lo >= t.n_bottom ? 1 : 0;
  tree_group_kernel<MODE><<<ng + nprep, TREE_THREADS, tree_group_smem(t.cap), st>>>(b, ng, top0, prepared);
  return cudaGetLastError();
}


cudaError_t tree_step(const Plan& p, const DevPtrs& d, const StepConsts& k, cudaStream_t st) {
  TreeArgs a = d.tree;
  a.k = k;
  const TreePlan& t = p.tree;
  cudaError_t e;
  // bottom groups of this process: all of them, or this rank's block when the tree is split across ranks
  const bool split = t.parts > 1 && !t.emulate;
  const int g_lo = split ? std::min(t.n_bottom, t.part * t.gpr) : 0;
  const int g_hi = split ? std::min(t.n_bottom, (t.part + 1) * t.gpr) : t.n_bottom;
  const bool top_section = t.n_mid > 0 || t.has_top;
  if (!top_section) return k.phase == 2 ? cudaSuccess : launch_group<TREE_BOTH>(a, g_lo, g_hi, t, st);
  if (k.phase != 2 && (e = launch_group<TREE_UP>(a, g_lo, g_hi, t, st, true))) return e;
  if (t.parts > 1) {  // exchange of the group roots' condensed blocks (one all-gather; emulated: every part local)
    const int q0 = split ? t.part : 0, q1 = split ? t.part + 1 : t.parts;
    for (int q = q0; q < q1 && k.phase != 2; ++q) {
      const int lo = std::min(t.n_bottom, q * t.gpr), hi = std::min(t.n_bottom, (q + 1) * t.gpr);
      const int r0 = t.root_off[lo], r1 = t.root_off[hi];
      if (r1 > r0) tree_pack_kernel<<<(unsigned)(((r1 - r0) * TSLOT + 255) / 256), 256, 0, st>>>(a, r0, r1);
    }
    if (k.phase == 1) return cudaGetLastError();  // host exchange: the caller all-gathers xbuf now
    if (split && t.rpp > 0 && p.use_nccl) {
      const int rc = nccl_allgather_doubles(d.nccl_comm, a.xbuf, (size_t)t.rpp * TSLOT, t.part, st);
      if (rc != 0) return nccl_step_failed(rc), cudaErrorUnknown;  // mabd_step reports MABD_ENCCL
    }
    const int nroot = t.root_off[t.n_bottom];
    if (nroot > 0) tree_unpack_kernel<<<(unsigned)((nroot * TSLOT + 255) / 256), 256, 0, st>>>(a, nroot);
  }
  const int m0 = t.n_bottom, m1 = t.n_bottom + t.n_mid, gt = m1;  // middle groups [m0, m1), top group gt
  if (!t.has_top) {  // the middle groups are whole trees of the top section
    if ((e = launch_group<TREE_BOTH>(a, m0, m1, t, st))) return e;
  } else {
    if ((e = launch_group<TREE_UP>(a, m0, m1, t, st))) return e;
    if (t.top_fused) {  // the top group as one CTA: up, down and stage 4 in one launch
      if ((e = launch_group<TREE_BOTH>(a, gt, gt + 1, t, st))) return e;
    } else {  // a large top group: one launch per level over the whole GPU (a body per warp up, per thread down)
      const int l0 = t.glev_ptr[gt], l1 = t.glev_ptr[gt + 1] - 1;
      const int wpc = 4;  // warps per CTA of the upward level launches
      for (int l = l0; l < l1; ++l) {
        const int nb = t.glev_off[l + 1] - t.glev_off[l];
        a.group0 = l;
        tree_level_kernel<<<(nb + wpc - 1) / wpc, 32 * wpc, 0, st>>>(a, TREE_UP_LEVEL);
      }
      for (int l = l1 - 1; l >= l0; --l) {
        const int nb = t.glev_off[l + 1] - t.glev_off[l];
        a.group0 = l;
        tree_level_kernel<<<(nb + 127) / 128, 128, 0, st>>>(a, TREE_DOWN_LEVEL);
      }
      if ((e = cudaGetLastError())) return e;
    }
    if ((e = launch_group<TREE_DOWN>(a, m0, m1, t, st))) return e;
  }
  return launch_group<TREE_DOWN>(a, g_lo, g_hi, t, st);
}

// Split across W ranks (or W emulated parts): contiguous blocks of gpr bottom groups; the joints from top bodies
// into each group, with their gather-buffer slots (rpp per part).
bool tree_partition(Plan* p, int W, int rank, bool emulate, std::string* msg) {
  TreePlan& t = p->tree;
  t.parts = W;
  t.part = rank;
  t.emulate = emulate;
  t.gpr = std::max(1, (t.n_bottom + W - 1) / W);
  if (!emulate && t.n_bottom < W)
    return *msg = "tree split: fewer CTA-local subtrees than ranks (run as replicas)", false;
  const int64_t n = p->n, top0 = t.n_bottom < (int)t.group_off.size() ? t.group_off[t.n_bottom] : n;
  std::vector<int32_t> group_of(n, -1);
  for (int g = 0; g < t.n_bottom; ++g)
    for (int b = t.group_off[g]; b < t.group_off[g + 1]; ++b) group_of[b] = g;
  std::vector<std::vector<int32_t>> per(std::max(1, t.n_bottom));
  for (int64_t pb = top0; pb < n; ++pb)  // child joints of top bodies whose child lies in a bottom group
    for (int j = t.child_off[pb]; j < t.child_off[pb + 1]; ++j) {
      const int cj = t.child_joint[j];
      const int cb = t.jchd[cj];
      if (cb >= 0 && group_of[cb] >= 0) per[group_of[cb]].push_back(cj);
    }
  t.root_off.assign(t.n_bottom + 1, 0);
  t.root_joint.clear();
  for (int g = 0; g < t.n_bottom; ++g) {
    std::sort(per[g].begin(), per[g].end());
    t.root_joint.insert(t.root_joint.end(), per[g].begin(), per[g].end());
    t.root_off[g + 1] = (int32_t)t.root_joint.size();
  }
  t.rpp = 0;
  t.root_slot.assign(t.root_joint.size(), 0);
  for (int q = 0; q < W; ++q) {
    const int lo = std::min(t.n_bottom, q * t.gpr), hi = std::min(t.n_bottom, (q + 1) * t.gpr);
    t.rpp = std::max(t.rpp, t.root_off[hi] - t.root_off[lo]);
  }
  for (int q = 0; q < W; ++q) {
    const int lo = std::min(t.n_bottom, q * t.gpr), hi = std::min(t.n_bottom, (q + 1) * t.gpr);
    for (int r = t.root_off[lo]; r < t.root_off[hi]; ++r) t.root_slot[r] = q * t.rpp + (r - t.root_off[lo]);
  }
  p->launches_per_step += 3;
  return true;
}

#ifdef MABD_EXP_TCLOCK
extern "C" int mabd_dbg_tclk(unsigned long long* out, int n) {
  const int m = std::min<int>(n, 3 * TCLK_CTAS * TCLK_SLOTS);
  return (int)cudaMemcpyFromSymbol(out, g_tclk, sizeof(unsigned long long) * m);
}
#endif

cudaError_t tree_init() {
  cudaError_t e;
  if ((e = cudaFuncSetAttribute(tree_group_kernel<TREE_UP>, cudaFuncAttributeMaxDynamicSharedMemorySize, TREE_SMEM_MAX)))
    return e;
  if ((e = cudaFuncSetAttribute(tree_group_kernel<TREE_DOWN>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                TREE_SMEM_MAX)))
    return e;
  return cudaFuncSetAttribute(tree_group_kernel<TREE_BOTH>, cudaFuncAttributeMaxDynamicSharedMemorySize, TREE_SMEM_MAX);
}

// ============================================================================ host: topology and ordering
bool tree_build(const mabd_joints* J, int64_t n, Plan* p, std::vector<int64_t>* pos_of_body, std::string* msg) {
  for (int64_t k = 0; J->kind && k < J->n_joints; ++k)
    if (J->kind[k] != 0) return *msg = "nonlinear joints (five-row hinges, universal, prismatic) need the sparse solver", false;
  const int64_t K = J->n_joints;
  // union-find over inter-body joints: a repeated connection is a cycle
  std::vector<int64_t> uf(n);
  for (int64_t i = 0; i < n; ++i) uf[i] = i;
  auto find = [&](int64_t x) {
    while (uf[x] != x) x = uf[x] = uf[uf[x]];
    return x;
  };
  std::vector<int64_t> pt_off(K + 1, 0);
  std::vector<std::vector<std::pair<int64_t, int64_t>>> adj(n);  // (neighbour, joint)
  for (int64_t k = 0; k < K; ++k) {
    pt_off[k + 1] = pt_off[k] + J->npts[k];
    const int64_t a = J->body_a[k], b = J->body_b[k];
    if (b < 0) continue;
    const int64_t ra = find(a), rb = find(b);
    if (ra == rb) return *msg = "cycle in the joint graph (tree solver)", false;
    uf[ra] = rb;
    adj[a].push_back({b, k});
    adj[b].push_back({a, k});
  }
  // root every component at a centre (repeated leaf peeling) to minimise the depth
  std::vector<int64_t> deg(n);
  for (int64_t i = 0; i < n; ++i) deg[i] = (int64_t)adj[i].size();
  std::vector<int64_t> comp_root(n, -1);
  {
    std::vector<int64_t> layer;
    std::vector<int64_t> d2 = deg;
    std::vector<char> peeled(n, 0);
    for (int64_t i = 0; i < n; ++i)
      if (d2[i] <= 1) layer.push_back(i);
    std::vector<int64_t> order_peel;
    while (!layer.empty()) {
      std::vector<int64_t> next;
      for (int64_t v : layer) {
        peeled[v] = 1;
        order_peel.push_back(v);
        for (auto& e : adj[v])
          if (!peeled[e.first] && --d2[e.first] == 1) next.push_back(e.first);
      }
      layer.swap(next);
    }
    // the last peeled body of each component is a centre
    for (auto it = order_peel.rbegin(); it != order_peel.rend(); ++it) {
      const int64_t c = find(*it);
      if (comp_root[c] < 0) comp_root[c] = *it;
    }
  }
  std::vector<int64_t> parent(n, -1), upj(n, -1), depth(n, 0), bfs;
  bfs.reserve(n);
  std::vector<char> seen(n, 0);
  for (int64_t i = 0; i < n; ++i) {
    const int64_t r = comp_root[find(i)];
    if (seen[r]) continue;
    seen[r] = 1;
    size_t h = bfs.size();
    bfs.push_back(r);
    while (h < bfs.size()) {
      const int64_t v = bfs[h++];
      for (auto& e : adj[v])
        if (!seen[e.first]) {
          seen[e.first] = 1;
          parent[e.first] = v;
          upj[e.first] = e.second;
          depth[e.first] = depth[v] + 1;
          bfs.push_back(e.first);
        }
    }
  }
  // subtree sizes and groups
  std::vector<int64_t> size(n, 1);
  for (auto it = bfs.rbegin(); it != bfs.rend(); ++it)
    if (parent[*it] >= 0) size[parent[*it]] += size[*it];
  // bodies carrying child joints (real children or anchors): the ones with something to eliminate
  std::vector<char> nonleaf(n, 0);
  for (int64_t k = 0; k < K; ++k) {
    const int64_t a = J->body_a[k], b = J->body_b[k];
    nonleaf[(b < 0 || (parent[b] == a && upj[b] == k)) ? a : b] = 1;
  }
  // group capacity: the larger groups once the tree gives every SM (148 on B200) one of them
  const int cap = n > 148LL * TREE_CAP ? 2 * TREE_CAP : TREE_CAP;
  std::vector<int64_t> local_roots;
  for (int64_t v : bfs)
    if (size[v] <= cap && (parent[v] < 0 || size[parent[v]] > cap)) local_roots.push_back(v);
  // children lists for subtree collection
  std::vector<std::vector<int64_t>> kids(n);
  for (int64_t v : bfs)
    if (parent[v] >= 0) kids[parent[v]].push_back(v);
  std::vector<std::vector<int64_t>> groups;
  std::vector<int64_t> cur;
  for (int64_t r : local_roots) {
    std::vector<int64_t> sub{r};
    for (size_t h = 0; h < sub.size(); ++h)
      for (int64_t c : kids[sub[h]]) sub.push_back(c);
    if (cur.size() + sub.size() > (size_t)cap) {
      groups.push_back(cur);
      cur.clear();
    }
    cur.insert(cur.end(), sub.begin(), sub.end());
  }
  if (!cur.empty()) groups.push_back(cur);
  TreePlan& t = p->tree;
  t = TreePlan();
  t.cap = cap;
  t.n_bottom = (int32_t)groups.size();
  std::vector<int64_t> top;
  for (int64_t v : bfs)
    if (size[v] > cap) top.push_back(v);
  if (top.size() > (size_t)TREE_TOP_SMALL && top.size() <= (size_t)cap) {
    // middle layer: subtrees of the top set with ≤ TREE_MID_CAP bodies (one CTA each), below a small top
    std::vector<char> in_top(n, 0);
    for (int64_t v : top) in_top[v] = 1;
    std::vector<int64_t> size_t_(n, 0);
    for (auto it = bfs.rbegin(); it != bfs.rend(); ++it)
      if (in_top[*it]) {
        size_t_[*it] += 1;
        if (parent[*it] >= 0) size_t_[parent[*it]] += size_t_[*it];
      }
    std::vector<char> taken(n, 0);
    std::vector<int64_t> mcur;
    for (int64_t v : top) {
      if (size_t_[v] > TREE_MID_CAP || (parent[v] >= 0 && size_t_[parent[v]] <= TREE_MID_CAP)) continue;
      std::vector<int64_t> sub{v};
      for (size_t h = 0; h < sub.size(); ++h)
        for (int64_t c : kids[sub[h]])
          if (in_top[c]) sub.push_back(c);
      if (mcur.size() + sub.size() > (size_t)TREE_MID_CAP) {
        groups.push_back(mcur);
        ++t.n_mid;
        mcur.clear();
      }
      for (int64_t c : sub) taken[c] = 1;
      mcur.insert(mcur.end(), sub.begin(), sub.end());
    }
    if (!mcur.empty()) {
      groups.push_back(mcur);
      ++t.n_mid;
    }
    std::vector<int64_t> rest;
    for (int64_t v : top)
      if (!taken[v]) rest.push_back(v);
    top.swap(rest);
  }
  if (!top.empty()) {
    groups.push_back(top);
    t.has_top = true;
    t.top_fused = top.size() <= (size_t)cap;
  }
  // internal order: groups in sequence, each sorted by depth (deepest first). Level ranges: group g owns
  // levels l ∈ [glev_ptr[g], glev_ptr[g+1]−1), level l spans bodies [glev_off[l], glev_off[l+1]).
  pos_of_body->assign(n, -1);
  std::vector<int64_t> body_of(n);
  int64_t pos = 0;
  std::vector<int32_t> gid(n, -1);
  t.group_off.push_back(0);
  for (size_t gi = 0; gi < groups.size(); ++gi) {
    auto& gvec = groups[gi];
    std::stable_sort(gvec.begin(), gvec.end(), [&](int64_t x, int64_t y) {
      return depth[x] != depth[y] ? depth[x] > depth[y] : nonleaf[x] > nonleaf[y];
    });
    t.glev_ptr.push_back((int32_t)t.glev_off.size());
    for (size_t i = 0; i < gvec.size(); ++i) {
      if (i == 0 || depth[gvec[i]] != depth[gvec[i - 1]]) {
        t.glev_off.push_back((int32_t)(pos + i));
        t.glev_nl.push_back((int32_t)(pos + i));
      }
      if (nonleaf[gvec[i]]) t.glev_nl.back() = (int32_t)(pos + i + 1);
      (*pos_of_body)[gvec[i]] = pos + (int64_t)i;
      body_of[pos + i] = gvec[i];
      gid[gvec[i]] = (int32_t)gi;
    }
    pos += (int64_t)gvec.size();
    t.glev_off.push_back((int32_t)pos);  // terminator of the group's last level
    t.glev_nl.push_back((int32_t)pos);   // (keeps glev_nl indexable like glev_off)
    t.group_off.push_back((int32_t)pos);
    if ((int)gi >= t.n_bottom)  // the top section is prepared by UP0: every body has a front record
      for (size_t l = t.glev_ptr.back(); l + 1 < t.glev_off.size(); ++l) t.glev_nl[l] = t.glev_off[l + 1];
  }
  t.glev_ptr.push_back((int32_t)t.glev_off.size());
  // joints
  t.jnpts.assign(K, 0);
  t.jchd.assign(K, -1);
  t.jy.assign(12 * K, 0.0);
  std::vector<int64_t> jpar(K, -1);
  int64_t rows = 0;
  for (int64_t k = 0; k < K; ++k) {
    const int64_t a = J->body_a[k], b = J->body_b[k];
    const int np = J->npts[k];
    t.jnpts[k] = np;
    rows += 3 * np;
    const double* ya = J->ybar_a + 3 * pt_off[k];
    const double* yb = J->ybar_b + 3 * pt_off[k];
    const double *yp, *yc;
    if (b < 0) {
      jpar[k] = a;
      yp = ya;
      yc = yb;
    } else if (parent[b] == a && upj[b] == k) {
      jpar[k] = a;
      t.jchd[k] = (int32_t)(*pos_of_body)[b];
      yp = ya;
      yc = yb;
    } else {
      jpar[k] = b;
      t.jchd[k] = (int32_t)(*pos_of_body)[a];
      yp = yb;
      yc = ya;
    }
    for (int q = 0; q < 3 * np; ++q) {
      t.jy[12 * k + q] = yp[q];
      t.jy[12 * k + 6 + q] = yc[q];
    }
  }
  p->n_dual_rows = rows;
  // per internal body: up joint, child joints, workspace
  t.up_joint.assign(n, -1);
  std::vector<std::vector<int32_t>> cj(n);
  for (int64_t k = 0; k < K; ++k) cj[(*pos_of_body)[jpar[k]]].push_back((int32_t)k);
  t.child_off.assign(n + 1, 0);
  t.ws_off.assign(n + 1, 0);
  t.fo_off.assign(n, -1);
  t.fo_str.assign(n, 0);
  t.fo_total = 0;
  std::vector<int64_t> recsz(n, 0);
  t.pt_off.clear();
  t.pt_code.clear();
  t.body_nn.clear();
  for (int64_t i = 0; i < n; ++i) {
    const int64_t v = body_of[i];
    t.up_joint[i] = (int32_t)upj[v];
    int N = 0;
    for (int32_t kk : cj[i]) N += 3 * t.jnpts[kk];
    if (N > TREE_MAXN) return *msg = "a body carries more than 24 child-joint rows (tree solver limit)", false;
    const int nu = upj[v] >= 0 ? 3 * t.jnpts[upj[v]] : 0;
    t.child_off[i + 1] = t.child_off[i] + (int32_t)cj[i].size();
    for (int32_t kk : cj[i]) t.child_joint.push_back(kk);
    t.ws_off[i + 1] = t.ws_off[i] + N + (int64_t)N * nu;
    const bool rec = N > 0 || i >= t.group_off[t.n_bottom];  // front record needed (incl. the whole top section)
    recsz[i] = rec ? (int64_t)(N + nu) * (N + nu + 1) / 2 + N + nu : 0;
    t.max_m = std::max(t.max_m, N + nu);
    // frontal point list: child joints' points (parent side, +), then the up joint's (child side, −);
    // code = 4·joint + 2·point + (1 for the child side)
    t.pt_off.push_back((int32_t)t.pt_code.size());
    for (int32_t kk : cj[i])
      for (int q = 0; q < t.jnpts[kk]; ++q) t.pt_code.push_back(4 * kk + 2 * q);
    if (upj[v] >= 0)
      for (int q = 0; q < t.jnpts[upj[v]]; ++q) t.pt_code.push_back(4 * (int32_t)upj[v] + 2 * q + 1);
    const bool ext = parent[v] >= 0 && gid[parent[v]] != gid[v];
    t.body_nn.push_back((int32_t)(N | (nu << 8) | (ext ? 1 << 16 : 0)));
  }
  t.pt_off.push_back((int32_t)t.pt_code.size());
  t.ws_total = t.ws_off[n];
  for (size_t g = 0; g + 1 < t.group_off.size(); ++g) {  // records interleaved per group
    int32_t cnt = 0;
    int64_t mx = 0;
    for (int b = t.group_off[g]; b < t.group_off[g + 1]; ++b)
      if (recsz[b] > 0) {
        ++cnt;
        mx = std::max(mx, recsz[b]);
      }
    int32_t rho = 0;
    for (int b = t.group_off[g]; b < t.group_off[g + 1]; ++b)
      if (recsz[b] > 0) {
        t.fo_off[b] = t.fo_total + rho++;
        t.fo_str[b] = cnt;
      }
    t.fo_total += mx * cnt;
  }
  t.parent.assign(n, -1);
  t.up_row.assign(n, 0);
  for (int64_t i = 0; i < n; ++i) {  // each child's up-joint rows in its parent's front (child joints in order)
    int row = 0;
    for (int32_t kk : cj[i]) {
      if (t.jchd[kk] >= 0) {
        t.parent[t.jchd[kk]] = (int32_t)i;
        t.up_row[t.jchd[kk]] = row;
      }
      row += 3 * t.jnpts[kk];
    }
  }
  p->ld = n;
  {  // UP0 (+ top-section preparation), [UP1], top, [DOWN1], DOWN0 — or one launch of whole-tree groups
    const int gt = t.n_bottom + t.n_mid;  // the top group's index
    int top_levels = 0;
    if (t.has_top) top_levels = t.glev_ptr[gt + 1] - 1 - t.glev_ptr[gt];
    const int top_launches = !t.has_top ? 0 : t.top_fused ? 1 : 2 * top_levels;
    if (t.n_mid == 0 && !t.has_top)
      p->launches_per_step = 1;
    else if (t.n_mid > 0)
      p->launches_per_step = 2 + (t.has_top ? 2 + top_launches : 1);
    else
      p->launches_per_step = 2 + top_launches;
  }
  return true;
}

}  // namespace mabd
