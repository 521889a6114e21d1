// Sparse (loops / irregular networks) solver of the M-ABD step on sm_100a: a multifrontal Cholesky
// factorization of the dual, refactored every step, with iterative refinement against the exact dual.
//
// The dual S λ = r, S = ∇C̃ H̃⁻¹ ∇C̃ᵀ, r = C(q̃) (P:563-566 with the footnote P:459), is solved "by any
// linear solver like Cholesky". Its sparsity pattern is constant, its values are not: the 3×3 block
// between constraint points p and q that share body j is s_p s_q R_j P_j(ȳ_p, ȳ_q) R_jᵀ, with the constant
// kernel P_j = Γ(ȳ_p) H̄_j⁻¹ Γ(ȳ_q)ᵀ and the body rotation R_j of this step (reading A1). So:
//   create (host, once):  nested-dissection ordering of the points from the bodies' initial positions, the
//                         assembly tree, front structures, extend-add maps, and the launch schedule;
//   every step (device):  assemble S into the fronts, factor them level by level (leaves first; small fronts
//                         in shared memory, large ones by 64-wide panels: POTRF → TRSM → SYRK), then forward
//                         and backward substitution, then two passes of iterative refinement with the exact
//                         matrix-free product S·x (bodies: v_j = H_j⁻¹ Σ s Γᵀx; points: Σ s Γ v).
// Nested dissection (geometric): the bodies of a region are split at the median of their widest coordinate;
// points joining bodies of both halves form the separator. Two points are coupled in S only if they share a
// body, so the halves' points are uncoupled and the separator is eliminated after both. Everything is fp64;
// there are no floating-point atomics (extend-add runs one child slot per launch), so the step is
// deterministic.
#include <cuda_runtime.h>

#include <algorithm>
#include <array>
#include <cstdlib>
#include <cmath>
#include <cstring>
#include <functional>
#include <numeric>
#include <string>
#include <vector>

#include "mabd_device.cuh"
#include "mabd_plan.h"

namespace mabd {

constexpr int SP_THREADS = 256;
constexpr int MF_NB = 64;          // panel width and tile size of the large-front path
#ifndef MF_SG
#define MF_SG 2               // 64-chunks per triangular-solve launch of the large fronts
#endif
constexpr int MF_ZC = 16;          // columns per CTA of the per-step lower-triangle zeroing of large fronts
#ifndef MF_SMALL_F
#define MF_SMALL_F 96
#endif
#ifndef MF_LEAF_P
#define MF_LEAF_P 8
#endif
constexpr int MF_SMALL = MF_SMALL_F;  // fronts with f ≤ MF_SMALL are factored in shared memory by one CTA
constexpr int MF_LEAF_PTS = MF_LEAF_P;  // nested dissection stops at regions of ≤ this many points
constexpr int MF_REFINE = 1;       // iterative-refinement passes per step (default; each gated, see below)
constexpr double MF_REFINE_TOL = 1e-10;  // a pass runs only if max|r − Sλ| > this · max|r| (refine_gate_kernel)

__device__ __forceinline__ void sreport(const StepConsts& k, int32_t flag) {
  atomicOr(k.err, flag);
  atomicMin(k.err + 1, k.step_index);
}

// ============================================================================ per-body stages (a1, a2, a5)
// bodies: predict; R → rs scratch, δq̃ → dqt
__global__ void sparse_predict_kernel(SparseArgs a) {
  const int64_t ld = a.b.ld;
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < a.n; j += (int64_t)gridDim.x * blockDim.x) {
    double q[12], qd[12], R[9], dqt[12];
#pragma unroll
    for (int c = 0; c < 12; ++c) {
      q[c] = a.b.q[c * ld + j];
      qd[c] = a.b.qd[c * ld + j];
    }
    const int mid = a.b.mat_id ? a.b.mat_id[j] : 0;
    const double msc = a.b.mscale ? a.b.mscale[j] : 1.0;
    const Material M = a.b.mats[mid];
    HinvBlk H;
    if (a.hinv_tab)
      H = a.hinv_tab[mid];
    else
      hinv_blocks(M, msc, a.k.ih2, H);
    double W[9];
    const double* Wp = load_wrench(a.b, j, W);
    if (!(a.k.lp ? predict_body<true>(q, qd, M, msc, H, a.k.ih, a.k.grav, R, dqt, Wp)
                 : predict_body<false>(q, qd, M, msc, H, a.k.ih, a.k.grav, R, dqt, Wp)))
      sreport(a.k, ERR_NONFINITE);
#pragma unroll
    for (int c = 0; c < 9; ++c) a.b.rs[c * ld + j] = R[c];
#pragma unroll
    for (int c = 0; c < 12; ++c) a.dqt[c * ld + j] = dqt[c];
  }
}

__device__ __forceinline__ void body_hinv(const SparseArgs& a, int64_t j, HinvBlk& H) {
  const int mid = a.b.mat_id ? a.b.mat_id[j] : 0;
  if (a.hinv_tab)
    H = a.hinv_tab[mid];
  else
    hinv_blocks(a.b.mats[mid], a.b.mscale ? a.b.mscale[j] : 1.0, a.k.ih2, H);
}
__device__ __forceinline__ void body_R(const SparseArgs& a, int64_t j, double* R) {
#pragma unroll
  for (int c = 0; c < 9; ++c) R[c] = a.b.rs[c * a.b.ld + j];
}

// projected point (five-row hinge): v ← [w0·v, w1·v, 0] (its rows), and the transpose x ← w0 x0 + w1 x1
__device__ __forceinline__ void project_rows(const SparseArgs& a, int64_t p, double* v) {
  const double* w = a.pw + 6 * (int64_t)a.pslot[p];
  const double v0 = w[0] * v[0] + w[1] * v[1] + w[2] * v[2];
  const double v1 = w[3] * v[0] + w[4] * v[1] + w[5] * v[2];
  v[0] = v0;
  v[1] = v1;
  v[2] = 0.0;
}
__device__ __forceinline__ void project_cols(const SparseArgs& a, int64_t p, double* x) {
  const double* w = a.pw + 6 * (int64_t)a.pslot[p];
  const double x0 = x[0], x1 = x[1];
#pragma unroll
  for (int e = 0; e < 3; ++e) x[e] = w[e] * x0 + w[3 + e] * x1;
}

// general slots (universal / prismatic joints, R17): each row is a scalar in body a's joint frame with
// R ≈ A, linearised at the iterate with its exact gradient; per side its coefficients are, in the world frame,
// w (a point part, at the slot point's ȳ) and v ⊗ dd (a direction part): J_side = [w ȳ_c + v dd_c (c = 0..2); w].
__device__ __forceinline__ int gen_slot(const SparseArgs& a, int64_t p) {
  if (!a.pgc || !a.pslot) return -1;
  const int s = a.pslot[p];
  return (s >= 0 && a.pgc[(int64_t)PGC_DOUBLES * s] != 0.0) ? s : -1;
}
__device__ __forceinline__ void gen_row_world(const SparseArgs& a, int64_t p, int s, int i, int side, double* o) {
  const double* g = a.pg + (int64_t)PG_DOUBLES * s + 18 * i + 9 * side;
  const double* y = a.py + 6 * p + 3 * side;
#pragma unroll
  for (int c = 0; c < 3; ++c)
#pragma unroll
    for (int r = 0; r < 3; ++r) o[3 * c + r] = g[r] * y[c] + g[3 + r] * g[6 + c];
#pragma unroll
  for (int r = 0; r < 3; ++r) o[9 + r] = g[r];
}
__device__ __forceinline__ double dot12(const double* x, const double* y) {
  double s = 0.0;
#pragma unroll
  for (int c = 0; c < 12; ++c) s += x[c] * y[c];
  return s;
}
__device__ __forceinline__ void to_body12(const double* R, const double* w, double* b) {
#pragma unroll
  for (int kb = 0; kb < 4; ++kb) mat3t_vec(R, w + 3 * kb, b + 3 * kb);
}
// row e of point p on `side` as a body-frame 12-vector (any point: plain, hinge / limit rows, general rows), with
// the side's sign; rows beyond a slot's count are zero
__device__ void row_body(const SparseArgs& a, int64_t p, int e, int side, const double* R, double* o) {
#pragma unroll
  for (int c = 0; c < 12; ++c) o[c] = 0.0;
  const int gs = gen_slot(a, p);
  if (gs >= 0) {
    if (e < a.pnr[gs]) {
      double w[12];
      gen_row_world(a, p, gs, e, side, w);
      to_body12(R, w, o);
    }
    return;
  }
  double wv[3] = {0.0, 0.0, 0.0};
  if (a.pslot && a.pslot[p] >= 0) {
    const int sl = a.pslot[p];
    if (e >= a.pnr[sl]) return;
    const double* w = a.pw + 6 * (int64_t)sl + 3 * e;
    wv[0] = w[0];
    wv[1] = w[1];
    wv[2] = w[2];
  } else {
    wv[e] = 1.0;
  }
  double wl[3];
  mat3t_vec(R, wv, wl);
  add_point_force(o, a.py + 6 * p + 3 * side, wl, side == 0 ? 1.0 : -1.0);
}
// a general slot's rows at the linearisation point (A, t of the iterate in q): 'dir' (A_a d)·(A_b e): side a
// v = A_b e, dd = d; side b v = A_a d, dd = e. 'point' (A_a d)·(x_a − x_b): side a w = A_a d, v = x_a − x_b (the
// frame's rotation term), dd = d; side b w = −A_a d. c0 = the row's value.
__device__ void gen_rows(const SparseArgs& a, int s, int64_t p) {
  const int64_t ld = a.b.ld, ja = a.pa[p], jb = a.pb[p];
  double Aa[9], Ab[9], ta[3], tb[3];
#pragma unroll
  for (int r = 0; r < 3; ++r) {
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      Aa[3 * r + c] = a.b.q[(3 * c + r) * ld + ja];
      Ab[3 * r + c] = jb >= 0 ? a.b.q[(3 * c + r) * ld + jb] : (r == c ? 1.0 : 0.0);
    }
    ta[r] = a.b.q[(9 + r) * ld + ja];
    tb[r] = jb >= 0 ? a.b.q[(9 + r) * ld + jb] : 0.0;
  }
  int nr = 0;
  for (int i = 0; i < 2; ++i) {
    const double* c = a.pgc + (int64_t)PGC_DOUBLES * s + PGC_ROW * i;
    const int type = (int)c[0];
    double* g = a.pg + (int64_t)PG_DOUBLES * s + 18 * i;
#pragma unroll
    for (int e = 0; e < 18; ++e) g[e] = 0.0;
    a.pg[(int64_t)PG_DOUBLES * s + 36 + i] = 0.0;
    if (type == 0) continue;
    nr = i + 1;
    double wa[3], xb[3];
    mat3_vec(Aa, c + 1, wa);
    double c0 = 0.0;
    if (type == 2) {
      mat3_vec(Ab, c + 4, xb);
#pragma unroll
      for (int r = 0; r < 3; ++r) {
        g[3 + r] = xb[r];
        g[6 + r] = c[1 + r];
        g[12 + r] = wa[r];
        g[15 + r] = c[4 + r];
        c0 += wa[r] * xb[r];
      }
    } else {
      const double* ya = a.py + 6 * p;
      const double* yb = ya + 3;
      double xa[3];
      mat3_vec(Aa, ya, xa);
      if (jb >= 0)
        mat3_vec(Ab, yb, xb);
#pragma unroll
      for (int r = 0; r < 3; ++r) {
        xa[r] += ta[r];
        xb[r] = jb >= 0 ? xb[r] + tb[r] : yb[r];
        const double off = xa[r] - xb[r];
        g[r] = wa[r];
        g[3 + r] = off;
        g[6 + r] = c[1 + r];
        g[9 + r] = -wa[r];
        c0 += wa[r] * off;
      }
    }
    a.pg[(int64_t)PG_DOUBLES * s + 36 + i] = c0;
  }
  a.pnr[s] = nr;
}

// per step (Newton iteration), at its linearisation point (R in rs):
//  hinge rows: w_i = R_a ΔR_H[i]ᵀ of the second axis point (R13);
//  joint limits (R14): θ = atan2(a_w·(u_aw × u_bw), u_aw·u_bw); inside [lo, hi] the slot is inactive (no rows);
//  beyond, the violated bound θ̂ gives the row w₀ = t, t = unit(a_w × R_a Rot(â, θ̂) u_a), at body a's point
//  ȳ₃ₐ = ȳ_a0 + ρ Rot(â, θ̂) u_a (written into py; body b's point ȳ_b0 + ρ u_b is constant).
__global__ void proj_rows_kernel(SparseArgs a) {
  const int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (s >= a.nproj) return;
  const int64_t p = a.pplist[s];
  if (a.pgc && a.pgc[(int64_t)PGC_DOUBLES * s] != 0.0) {  // universal / prismatic rows (R17)
    gen_rows(a, (int)s, p);
    return;
  }
  double R[9];
  body_R(a, a.pa[p], R);
  double* w = a.pw + 6 * s;
  const double* L = a.plim + (int64_t)LIM_DOUBLES * s;
  if (!(L[14] > 0.0)) {  // hinge rows (ρ = 0 marks a non-limit slot)
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      const double* d = a.pdr + 6 * s + 3 * i;
#pragma unroll
      for (int c = 0; c < 3; ++c) w[3 * i + c] = R[3 * c] * d[0] + R[3 * c + 1] * d[1] + R[3 * c + 2] * d[2];
    }
    a.pnr[s] = 2;
    return;
  }
  const double* ax = L + 11;
  double aw[3], uaw[3], ubw[3];
  mat3_vec(R, ax, aw);
  mat3_vec(R, L + 2, uaw);
  if (a.pb[p] >= 0) {
    double Rb[9];
    body_R(a, a.pb[p], Rb);
    mat3_vec(Rb, L + 5, ubw);
  } else {
#pragma unroll
    for (int e = 0; e < 3; ++e) ubw[e] = L[5 + e];
  }
  const double cx = uaw[1] * ubw[2] - uaw[2] * ubw[1], cy = uaw[2] * ubw[0] - uaw[0] * ubw[2],
               cz = uaw[0] * ubw[1] - uaw[1] * ubw[0];
  const double th = atan2(aw[0] * cx + aw[1] * cy + aw[2] * cz, uaw[0] * ubw[0] + uaw[1] * ubw[1] + uaw[2] * ubw[2]);
  const double lo = L[0], hi = L[1];
#pragma unroll
  for (int e = 0; e < 6; ++e) w[e] = 0.0;
  if (th >= lo && th <= hi) {
    a.pnr[s] = 0;
    return;
  }
  const double thh = th > hi ? hi : lo;
  // Rot(â, θ̂) u_a = u_a cos θ̂ + (â × u_a) sin θ̂ + â (â·u_a)(1 − cos θ̂), in body a's frame
  const double* ua = L + 2;
  const double c = cos(thh), sn = sin(thh), ad = ax[0] * ua[0] + ax[1] * ua[1] + ax[2] * ua[2];
  const double axu[3] = {ax[1] * ua[2] - ax[2] * ua[1], ax[2] * ua[0] - ax[0] * ua[2], ax[0] * ua[1] - ax[1] * ua[0]};
  double ur[3], urw[3];
#pragma unroll
  for (int e = 0; e < 3; ++e) ur[e] = ua[e] * c + axu[e] * sn + ax[e] * ad * (1.0 - c);
  double* py = const_cast<double*>(a.py) + 6 * p;  // body a's point of this iteration
#pragma unroll
  for (int e = 0; e < 3; ++e) py[e] = L[8 + e] + L[14] * ur[e];
  mat3_vec(R, ur, urw);
  double t[3] = {aw[1] * urw[2] - aw[2] * urw[1], aw[2] * urw[0] - aw[0] * urw[2], aw[0] * urw[1] - aw[1] * urw[0]};
  const double it = rsqrt(t[0] * t[0] + t[1] * t[1] + t[2] * t[2]);
#pragma unroll
  for (int e = 0; e < 3; ++e) w[e] = t[e] * it;
  a.pnr[s] = 1;
}

// points: r = C(q̃) (q̃ = qⁿ + δq̃)
__global__ void sparse_rhs_kernel(SparseArgs a) {
  const int64_t ld = a.b.ld;
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < a.np; p += (int64_t)gridDim.x * blockDim.x) {
    double r[3] = {0, 0, 0};
    const int gs = gen_slot(a, p);
    if (gs >= 0) {  // general rows: c0 + J δq̃ (linearised at the iterate)
      for (int e = 0; e < a.pnr[gs]; ++e) {
        r[e] = a.pg[(int64_t)PG_DOUBLES * gs + 36 + e];
        for (int side = 0; side < 2; ++side) {
          const int64_t j = side == 0 ? a.pa[p] : a.pb[p];
          if (j < 0) continue;
          double w[12], d[12];
          gen_row_world(a, p, gs, e, side, w);
#pragma unroll
          for (int c = 0; c < 12; ++c) d[c] = a.dqt[c * ld + j];
          r[e] += dot12(w, d);
        }
      }
#pragma unroll
      for (int e = 0; e < 3; ++e) a.rhs[e * a.np + p] = r[e];
      continue;
    }
    for (int side = 0; side < 2; ++side) {
      const int64_t j = side == 0 ? a.pa[p] : a.pb[p];
      const double* y = a.py + 6 * p + 3 * side;
      const double sg = side == 0 ? 1.0 : -1.0;
      if (j < 0) {  // world point
#pragma unroll
        for (int e = 0; e < 3; ++e) r[e] += sg * y[e];
        continue;
      }
      double qt[12], x[3];
#pragma unroll
      for (int c = 0; c < 12; ++c) qt[c] = a.b.q[c * ld + j] + a.dqt[c * ld + j];
      point_pos(qt, y, x);
#pragma unroll
      for (int e = 0; e < 3; ++e) r[e] += sg * x[e];
    }
    if (a.pslot && a.pslot[p] >= 0) project_rows(a, p, r);
#pragma unroll
    for (int e = 0; e < 3; ++e) a.rhs[e * a.np + p] = r[e];
  }
}

// v_j = H_j⁻¹ Σ s Γ(ȳ)ᵀ x_p over the points incident to body j (x: [3][np] component-major)
__device__ __forceinline__ void body_apply(const SparseArgs& a, int64_t j, const double* x, double* out12) {
  double g[12];
#pragma unroll
  for (int c = 0; c < 12; ++c) g[c] = 0.0;
  double R[9];
  body_R(a, j, R);
  for (int i = a.inc_off[j]; i < a.inc_off[j + 1]; ++i) {
    const int32_t e = a.inc[i];
    const int64_t p = e >> 1;
    const int side = e & 1;
    const int gs = gen_slot(a, p);
    if (gs >= 0) {  // general rows: g += x_e J_e (body frame)
      for (int r = 0; r < a.pnr[gs]; ++r) {
        double wr[12], wb[12];
        gen_row_world(a, p, gs, r, side, wr);
        to_body12(R, wr, wb);
        const double xe = x[r * a.np + p];
#pragma unroll
        for (int c = 0; c < 12; ++c) g[c] += xe * wb[c];
      }
      continue;
    }
    double w[3], wl[3];
#pragma unroll
    for (int c = 0; c < 3; ++c) w[c] = x[c * a.np + p];
    if (a.pslot && a.pslot[p] >= 0) project_cols(a, p, w);
    mat3t_vec(R, w, wl);  // body frame
    add_point_force(g, a.py + 6 * p + 3 * side, wl, side == 0 ? 1.0 : -1.0);
  }
  HinvBlk H;
  body_hinv(a, j, H);
  double u[12];
  hinv_apply(H, g, u);
#pragma unroll
  for (int kb = 0; kb < 4; ++kb) mat3_vec(R, u + 3 * kb, out12 + 3 * kb);
}

// matrix-free S·x, pass 1 (bodies): V = H⁻¹ Jᵀ x
__device__ __forceinline__ bool refine_gated(const SparseArgs& a) { return a.gate && *a.gate; }

__global__ void mv_body_kernel(SparseArgs a, const double* x) {
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < a.n; j += (int64_t)gridDim.x * blockDim.x) {
    double v[12];
    body_apply(a, j, x, v);
#pragma unroll
    for (int c = 0; c < 12; ++c) a.vv[c * a.n + j] = v[c];
  }
}
// pass 2 (points): res = rhs − J V
__global__ void mv_point_kernel(SparseArgs a) {
  double mres = 0.0, mrhs = 0.0;
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < a.np; p += (int64_t)gridDim.x * blockDim.x) {
    double s[3] = {0, 0, 0};
    const int gs = gen_slot(a, p);
    if (gs >= 0) {  // general rows: J V; dummy rows S = 1
      const int nr = a.pnr[gs];
      for (int e = 0; e < 3; ++e) {
        if (e >= nr) {
          s[e] = a.lam[e * a.np + p];
          continue;
        }
        for (int side = 0; side < 2; ++side) {
          const int64_t j = side == 0 ? a.pa[p] : a.pb[p];
          if (j < 0) continue;
          double w[12], v[12];
          gen_row_world(a, p, gs, e, side, w);
#pragma unroll
          for (int c = 0; c < 12; ++c) v[c] = a.vv[c * a.n + j];
          s[e] += dot12(w, v);
        }
      }
    } else {
    for (int side = 0; side < 2; ++side) {
      const int64_t j = side == 0 ? a.pa[p] : a.pb[p];
      if (j < 0) continue;
      const double* y = a.py + 6 * p + 3 * side;
      const double sg = side == 0 ? 1.0 : -1.0;
#pragma unroll
      for (int e = 0; e < 3; ++e)
        s[e] += sg * (a.vv[(0 + e) * a.n + j] * y[0] + a.vv[(3 + e) * a.n + j] * y[1] +
                      a.vv[(6 + e) * a.n + j] * y[2] + a.vv[(9 + e) * a.n + j]);
    }
    if (a.pslot && a.pslot[p] >= 0) {  // rows w·(J V); the dummy rows' S = 1 (the refinement's x is λ)
      project_rows(a, p, s);
      const int nr = a.pnr[a.pslot[p]];
      for (int e = nr; e < 3; ++e) s[e] = a.lam[e * a.np + p];
    }
    }
#pragma unroll
    for (int e = 0; e < 3; ++e) {
      const double r = a.rhs[e * a.np + p];
      a.res[e * a.np + p] = r - s[e];
      mres = fmax(mres, fabs(r - s[e]));
      mrhs = fmax(mrhs, fabs(r));
    }
  }
  // max |res| and max |rhs| for the refinement gate (non-negative doubles order like their bit patterns)
  for (int o = 16; o > 0; o >>= 1) {
    mres = fmax(mres, __shfl_xor_sync(0xffffffffu, mres, o));
    mrhs = fmax(mrhs, __shfl_xor_sync(0xffffffffu, mrhs, o));
  }
  if ((threadIdx.x & 31) == 0) {
    atomicMax(a.rmax, (unsigned long long)__double_as_longlong(mres));
    atomicMax(a.rmax + 1, (unsigned long long)__double_as_longlong(mrhs));
  }
}
// Refinement gate (pass `it`): the pass runs only if the residual of the current λ exceeds refine_tol · max|r|
// (a backward-stable factorization of a well-conditioned S already leaves a residual at rounding level, and the
// pass would change nothing); a NaN residual runs it (the non-finite check sees the result). iters[0] = passes run.
__global__ void refine_gate_kernel(SparseArgs a, int it) {
  const double mres = __longlong_as_double((long long)a.rmax[0]), mrhs = __longlong_as_double((long long)a.rmax[1]);
  const int skip = (it > 0 && a.iters[1]) || mres <= a.refine_tol * mrhs;
  a.iters[1] = skip;
  a.rmax[2] = (unsigned long long)__double_as_longlong(mres / mrhs);  // developer probe (mabd_dbg_refine_ratio)
  a.iters[0] = (it == 0 ? 0 : a.iters[0]) + (skip ? 0 : 1);
  a.rmax[0] = a.rmax[1] = 0ull;
}
__global__ void axpy_kernel(double* y, const double* x, int64_t n, const int32_t* gate) {
  if (*gate) return;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    y[i] += x[i];
}

// bodies: qⁿ⁺¹ = q̃ − H⁻¹ Jᵀ λ, q̇ⁿ⁺¹ = δq/h
__global__ void sparse_update_kernel(SparseArgs a) {
  const int64_t ld = a.b.ld;
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < a.n; j += (int64_t)gridDim.x * blockDim.x) {
    double v[12];
    body_apply(a, j, a.lam, v);
    // every load before the first store (q, q̇ and δq̃ may alias as far as the compiler knows)
    double q[12], dq[12];
#pragma unroll
    for (int c = 0; c < 12; ++c) {
      q[c] = a.b.q[c * ld + j];
      dq[c] = a.dqt[c * ld + j] - v[c];
    }
    if (a.k.niter == 1) {
#pragma unroll
      for (int c = 0; c < 12; ++c) {
        a.b.q[c * ld + j] = q[c] + dq[c];
        a.b.qd[c * ld + j] = dq[c] * a.k.ih;
      }
    } else {  // K > 1: v ← v − δq/h + h·grav (launch_step in mabd_plan.cu)
      double w[12];
#pragma unroll
      for (int c = 0; c < 12; ++c) w[c] = a.b.qd[c * ld + j];
#pragma unroll
      for (int c = 0; c < 12; ++c) {
        a.b.q[c * ld + j] = q[c] + dq[c];
        a.b.qd[c * ld + j] = w[c] - dq[c] * a.k.ih + (c >= 9 ? a.k.h * a.k.grav[c - 9] : 0.0);
      }
    }
  }
}

// ============================================================================ numeric factorization
// Assembly of the original entries: one thread per 3×3 block (row point q, column point p, both in the front of
// the node owning p): S_qp = Σ_{shared bodies j} s_q s_p R_j P_j(ȳ_q, ȳ_p) R_jᵀ.
// Fronts are column-major and every factorization and solve kernel reads and writes only their lower triangle
// (rows r ≥ column c), so a step zeroes only that part: f(f+1)/2 instead of f² doubles per front (the upper part
// is zeroed once at upload and never touched). task = (node, first column of a run of MF_ZC columns; a small front
// is one task).
__global__ void __launch_bounds__(SP_THREADS) mf_zero_kernel(SparseArgs a, const int32_t* tasks) {
  const MfArgs& m = a.mf;
  const int node = tasks[2 * blockIdx.x], c0 = tasks[2 * blockIdx.x + 1];
  const int64_t f = m.fdim[node];
  double* F = m.F + m.foff[node];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t c1 = f <= MF_SMALL ? f : (f < c0 + MF_ZC ? f : (int64_t)(c0 + MF_ZC));  // a small front: one task
  for (int64_t c = c0 + warp; c < c1; c += SP_THREADS / 32) {
    double* col = F + c * f;
    for (int64_t r = c + lane; r < f; r += 32) col[r] = 0.0;
  }
}

__global__ void mf_assemble_kernel(SparseArgs a) {
  const MfArgs& m = a.mf;
  for (int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; b < m.nblk;
       b += (int64_t)gridDim.x * blockDim.x) {
    const int node = m.ablk[3 * b], rb = m.ablk[3 * b + 1], cb = m.ablk[3 * b + 2];
    double S[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
    int prow = -1, pcol = -1;
    if (m.acoff[b] < m.acoff[b + 1]) {
      prow = m.acon[2 * m.acoff[b]] >> 1;
      pcol = m.acon[2 * m.acoff[b] + 1] >> 1;
    }
    if (prow >= 0 && (gen_slot(a, prow) >= 0 || gen_slot(a, pcol) >= 0)) {  // general rows: J_r H⁻¹ J_cᵀ by rows
      for (int c = m.acoff[b]; c < m.acoff[b + 1]; ++c) {
        const int re = m.acon[2 * c], ce = m.acon[2 * c + 1];
        const int sr = re & 1, sc = ce & 1;
        const int64_t j = sr == 0 ? a.pa[prow] : a.pb[prow];
        double R[9];
        body_R(a, j, R);
        HinvBlk H;
        body_hinv(a, j, H);
        double u[3][12];
        for (int f = 0; f < 3; ++f) {
          double cv[12];
          row_body(a, pcol, f, sc, R, cv);
          hinv_apply(H, cv, u[f]);
        }
        for (int e = 0; e < 3; ++e) {
          double rv[12];
          row_body(a, prow, e, sr, R, rv);
          for (int f = 0; f < 3; ++f) S[3 * e + f] += dot12(rv, u[f]);
        }
      }
      if (prow == pcol) {
        const int sl = a.pslot[prow];
        if (sl >= 0)
          for (int e = a.pnr[sl]; e < 3; ++e) S[4 * e] = 1.0;  // dummy rows: S = 1, decoupled
      }
    } else {
    for (int c = m.acoff[b]; c < m.acoff[b + 1]; ++c) {
      const int re = m.acon[2 * c], ce = m.acon[2 * c + 1];
      const int pr = re >> 1, sr = re & 1, pc = ce >> 1, sc = ce & 1;
      prow = pr;
      pcol = pc;
      const int64_t j = sr == 0 ? a.pa[pr] : a.pb[pr];
      const double sg = (sr == sc) ? 1.0 : -1.0;
      double R[9], P[9], T[9];
      body_R(a, j, R);
      HinvBlk H;
      body_hinv(a, j, H);
      pblock(H, a.py + 6 * pr + 3 * sr, a.py + 6 * pc + 3 * sc, P);
      rot_conj(R, P, T);
#pragma unroll
      for (int e = 0; e < 9; ++e) S[e] += sg * T[e];
    }
    if (a.pslot && prow >= 0) {  // projected points: S ← T_r S T_cᵀ (+1 on a projected point's dummy row)
      const bool pjr = a.pslot[prow] >= 0, pjc = a.pslot[pcol] >= 0;
      if (pjr)
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          double col[3] = {S[c], S[3 + c], S[6 + c]};
          project_rows(a, prow, col);
          S[c] = col[0]; S[3 + c] = col[1]; S[6 + c] = col[2];
        }
      if (pjc)
#pragma unroll
        for (int r = 0; r < 3; ++r) project_rows(a, pcol, S + 3 * r);
      if (pjr && prow == pcol)
        for (int e = a.pnr[a.pslot[prow]]; e < 3; ++e) S[4 * e] = 1.0;  // dummy rows: S = 1, decoupled
    }
    }
    double* F = m.F + m.foff[node];
    const int64_t f = m.fdim[node];
#pragma unroll
    for (int r = 0; r < 3; ++r)
#pragma unroll
      for (int c = 0; c < 3; ++c) F[(3 * cb + c) * f + 3 * rb + r] = S[3 * r + c];
  }
}

__device__ __forceinline__ int mapped(const int32_t* map, int i) { return 3 * map[i / 3] + i % 3; }

// Small fronts (f ≤ MF_SMALL): one CTA loads the front into shared memory, extend-adds its children's update
// matrices, runs the partial (right-looking) Cholesky of its own columns, and writes L and its own update back.
__global__ void __launch_bounds__(SP_THREADS) mf_small_kernel(SparseArgs a, const int32_t* nodes) {
  extern __shared__ double sF[];
  const MfArgs& m = a.mf;
  const int node = nodes[blockIdx.x];
  const int f = m.fdim[node], n = m.nown[node];
  double* F = m.F + m.foff[node];
  for (int i = threadIdx.x; i < f * f; i += blockDim.x) sF[i] = F[i];
  __syncthreads();
  for (int ci = m.ch_off[node]; ci < m.ch_off[node + 1]; ++ci) {
    const int c = m.ch[ci];
    const int fc = m.fdim[c], nc = m.nown[c], mc = fc - nc;
    const double* Fc = m.F + m.foff[c];
    const int32_t* map = m.ea_map + m.ea_off[c];
    const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;  // 16 × 16 tile over (row i, column j): no division
    for (int j = ty; j < mc; j += 16) {
      const int pj = mapped(map, j);
      const double* src = Fc + (int64_t)(nc + j) * fc + nc;
      for (int i = j + tx; i < mc; i += 16) sF[pj * f + mapped(map, i)] += src[i];
    }
    __syncthreads();
  }
  // unscaled (L D Lᵀ) elimination: step k reads column k, which it does not write, and updates the columns
  // j > k with S_ij −= S_ik S_jk / S_kk — one barrier per column; the columns are scaled by 1/√D_k afterwards
  __shared__ double isd[MF_SMALL];
  const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;
  for (int k = 0; k < n; ++k) {
    double d = sF[k * f + k];
    if (!(d > 0.0)) {
      if (threadIdx.x == 0) sreport(a.k, ERR_SINGULAR);
      d = 1.0;
      if (threadIdx.x == 0) sF[k * f + k] = 1.0;
    }
    const double id = 1.0 / d;
    for (int j = k + 1 + ty; j < f; j += 16) {  // column j, rows i ≥ j
      const double ljk = sF[k * f + j] * id;
      for (int i = j + tx; i < f; i += 16) sF[j * f + i] -= sF[k * f + i] * ljk;
    }
    __syncthreads();
  }
  for (int k = threadIdx.x; k < n; k += blockDim.x) isd[k] = 1.0 / sqrt(sF[k * f + k]);
  __syncthreads();
  for (int i = threadIdx.x; i < f * f; i += blockDim.x) {
    const int c = i / f, r = i % f;
    if (r >= c) F[i] = c < n ? sF[i] * isd[c] : sF[i];  // L_rc = S_rc / √D_c (the diagonal: √D_c); update as is
  }
}

// Extend-add into large parents, one child slot per launch: task = (parent, child column j).
__global__ void __launch_bounds__(128) mf_ea_kernel(SparseArgs a, const int32_t* tasks, int slot) {
  const MfArgs& m = a.mf;
  const int node = tasks[2 * blockIdx.x], j = tasks[2 * blockIdx.x + 1];
  const int c = m.ch[m.ch_off[node] + slot];
  const int fc = m.fdim[c], nc = m.nown[c], mc = fc - nc;
  const int64_t f = m.fdim[node];
  const int32_t* map = m.ea_map + m.ea_off[c];
  const double* src = m.F + m.foff[c] + (int64_t)(nc + j) * fc + nc;
  double* dst = m.F + m.foff[node] + mapped(map, j) * f;
  // four entries per round, every load before the stores (dst and src may alias as far as the compiler knows)
  const int st = blockDim.x;
  int i = j + threadIdx.x;
  for (; i + 3 * st < mc; i += 4 * st) {
    int64_t d[4];
    double x[4], y[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      d[u] = mapped(map, i + u * st);
      x[u] = src[i + u * st];
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) y[u] = dst[d[u]];
#pragma unroll
    for (int u = 0; u < 4; ++u) dst[d[u]] = y[u] + x[u];
  }
  for (; i < mc; i += st) dst[mapped(map, i)] += src[i];
}

// Panel step 1: Cholesky of the kb×kb diagonal block at k0, and its inverse L⁻¹ (kept per front and chunk: the
// TRSM of this panel and the triangular solves use it). Blocked by 8×8: warp 0 factors a diagonal block, the CTA
// solves the block column below against it (forward substitution per row) and applies the rank-8 trailing update.
// The inverse is formed afterwards by recursive doubling: the eight 8×8 diagonal inverses at once, then blocks of
// 16, 32, 64 with X21 = −X22 (L21 X11) (two CTA-wide products per level instead of a serial sweep over block rows).
constexpr int PB = 8;
__global__ void __launch_bounds__(SP_THREADS) mf_potrf_kernel(SparseArgs a, const int32_t* tasks, int k0) {
  extern __shared__ double psm[];
  double(*L)[MF_NB + 1] = reinterpret_cast<double(*)[MF_NB + 1]>(psm);
  double(*X)[MF_NB + 1] = reinterpret_cast<double(*)[MF_NB + 1]>(psm + MF_NB * (MF_NB + 1));
  __shared__ double dinv[MF_NB];  // 1 / L_jj
  const MfArgs& m = a.mf;
  const int node = tasks[blockIdx.x];
  const int n = m.nown[node];
  const int64_t f = m.fdim[node];
  const int kb = min(MF_NB, n - k0);
  double* F = m.F + m.foff[node];
  const int tid = threadIdx.x, tx = tid % 16, ty = tid / 16, lane = tid & 31, warp = tid >> 5;
  // load the lower part; pad to 64 with an identity block (rows/cols ≥ kb) so every block step is 8 wide
  for (int idx = tid; idx < MF_NB * MF_NB; idx += blockDim.x) {
    const int r = idx % MF_NB, c = idx / MF_NB;
    double v = 0.0;
    if (r < kb && c < kb) {
      if (r >= c) v = F[(k0 + c) * f + k0 + r];
    } else if (r == c) {
      v = 1.0;
    }
    L[r][c] = v;
    X[r][c] = 0.0;
  }
  __syncthreads();
  const int nbk = (kb + PB - 1) / PB;
  for (int bk = 0; bk < nbk; ++bk) {
    const int c0 = PB * bk;
    if (warp == 0) {  // 8×8 diagonal block: Cholesky (1 / L_jj kept)
      for (int j = 0; j < PB; ++j) {
        double d = L[c0 + j][c0 + j];
        if (!(d > 0.0)) {
          if (lane == 0) sreport(a.k, ERR_SINGULAR);
          d = 1.0;
        }
        const double isd = fast_rsqrt(d), sd = d * isd;
        __syncwarp();
        if (lane == 0) {
          L[c0 + j][c0 + j] = sd;
          dinv[c0 + j] = isd;
        }
        if (lane > j && lane < PB) L[c0 + lane][c0 + j] *= isd;
        __syncwarp();
        {  // trailing of the block: (i, l), j < l ≤ i < 8; 28 pairs at most
          const int i = j + 1 + lane / PB, l = j + 1 + lane % PB;
          if (i < PB && l <= i) L[c0 + i][c0 + l] -= L[c0 + i][c0 + j] * L[c0 + l][c0 + j];
          const int i2 = i + 4;  // lanes cover rows j+1..j+4 and j+5..j+8
          if (i2 < PB && l <= i2) L[c0 + i2][c0 + l] -= L[c0 + i2][c0 + j] * L[c0 + l][c0 + j];
        }
        __syncwarp();
      }
    }
    __syncthreads();
    // block column below: L[r, c0:c0+8] ← L[r, c0:c0+8] L_bb⁻ᵀ, forward substitution (one thread per row)
    for (int r = c0 + PB + tid; r < MF_NB; r += blockDim.x) {
      double v[PB];
#pragma unroll
      for (int e = 0; e < PB; ++e) v[e] = L[r][c0 + e];
#pragma unroll
      for (int c = 0; c < PB; ++c) {
        double acc = v[c];
#pragma unroll
        for (int e = 0; e < c; ++e) acc -= v[e] * L[c0 + c][c0 + e];
        v[c] = acc * dinv[c0 + c];
      }
#pragma unroll
      for (int e = 0; e < PB; ++e) L[r][c0 + e] = v[e];
    }
    __syncthreads();
    // rank-8 trailing update of the lower part: rows and columns ≥ c0+8
    for (int r = c0 + PB + ty; r < MF_NB; r += 16) {
      double lr[PB];
#pragma unroll
      for (int e = 0; e < PB; ++e) lr[e] = L[r][c0 + e];
      for (int c = c0 + PB + tx; c <= r; c += 16) {
        double acc = 0.0;
#pragma unroll
        for (int e = 0; e < PB; ++e) acc += lr[e] * L[c][c0 + e];
        L[r][c] -= acc;
      }
    }
    __syncthreads();
  }
  for (int idx = tid; idx < kb * kb; idx += blockDim.x) {
    const int r = idx % kb, c = idx / kb;
    if (r >= c) F[(k0 + c) * f + k0 + r] = L[r][c];
  }
  // the eight 8×8 diagonal inverses (padding blocks are identities): thread (b, j) forms column j of block b
  if (tid < MF_NB) {
    const int c0 = PB * (tid / PB), j = tid % PB;
    for (int i = 0; i < PB; ++i) {
      double v = (i == j) ? 1.0 : 0.0;
      for (int l = j; l < i; ++l) v -= L[c0 + i][c0 + l] * X[c0 + l][c0 + j];
      X[c0 + i][c0 + j] = i >= j ? v / L[c0 + i][c0 + i] : 0.0;
    }
  }
  __syncthreads();
  // recursive doubling: pairs of s×s diagonal blocks at p, p + s: X21 = −X22 T with T = L21 X11; T is parked
  // transposed in X's upper part (X[p + j][p + s + i], never read as part of the inverse; masked on output)
  for (int s = PB; s < MF_NB; s *= 2) {
    const int ne = (MF_NB / (2 * s)) * s * s;
    for (int e = tid; e < ne; e += blockDim.x) {
      const int p = (e / (s * s)) * 2 * s, i = (e % (s * s)) / s, j = e % s;
      double acc = 0.0;
      for (int l = j; l < s; ++l) acc += L[p + s + i][p + l] * X[p + l][p + j];  // X11 lower: l ≥ j
      X[p + j][p + s + i] = acc;
    }
    __syncthreads();
    for (int e = tid; e < ne; e += blockDim.x) {
      const int p = (e / (s * s)) * 2 * s, i = (e % (s * s)) / s, j = e % s;
      double acc = 0.0;
      for (int l = 0; l <= i; ++l) acc += X[p + s + i][p + s + l] * X[p + j][p + s + l];  // X22 lower: l ≤ i
      X[p + s + i][p + j] = -acc;
    }
    __syncthreads();
  }
  double* out = m.linv + m.loff[node] + (int64_t)(k0 / MF_NB) * MF_NB * MF_NB;
  for (int idx = tid; idx < MF_NB * MF_NB; idx += blockDim.x) {
    const int r = idx / MF_NB, c = idx % MF_NB;
    out[idx] = (r < kb && c < kb && c <= r) ? X[r][c] : 0.0;
  }
}

// Panel step 2: rows r0..r0+63 of the panel: X = B L⁻ᵀ (B = F[r, k0:k0+kb]); task = (node, r0, potrf slot).
__global__ void __launch_bounds__(SP_THREADS) mf_trsm_kernel(SparseArgs a, const int32_t* tasks, int k0) {
  extern __shared__ double tsm[];
  double(*Li)[MF_NB + 1] = reinterpret_cast<double(*)[MF_NB + 1]>(tsm);
  double(*Bs)[MF_NB + 1] = reinterpret_cast<double(*)[MF_NB + 1]>(tsm + MF_NB * (MF_NB + 1));
  const MfArgs& m = a.mf;
  const int node = tasks[3 * blockIdx.x], r0 = tasks[3 * blockIdx.x + 1];
  const int n = m.nown[node];
  const int64_t f = m.fdim[node];
  const int kb = min(MF_NB, n - k0);
  const int rows = min((int64_t)MF_NB, f - r0);
  double* F = m.F + m.foff[node];
  const double* li = m.linv + m.loff[node] + (int64_t)(k0 / MF_NB) * MF_NB * MF_NB;
  const int tid = threadIdx.x;
  for (int idx = tid; idx < MF_NB * MF_NB; idx += blockDim.x) {
    const int r = idx % MF_NB, l = idx / MF_NB;
    Li[idx / MF_NB][idx % MF_NB] = li[idx];
    Bs[r][l] = (r < rows && l < kb) ? F[(k0 + l) * f + r0 + r] : 0.0;
  }
  __syncthreads();
  const int tx = tid % 16, ty = tid / 16;
  double acc[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = 0.0;
  for (int l = 0; l < kb; ++l) {
    double bv[4], lv[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) bv[i] = Bs[ty + 16 * i][l];
#pragma unroll
    for (int j = 0; j < 4; ++j) lv[j] = Li[tx + 16 * j][l];  // Linv[c][l], zero above the diagonal
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) acc[i][j] = fma(bv[i], lv[j], acc[i][j]);
  }
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int r = ty + 16 * i, c = tx + 16 * j;
      if (r < rows && c < kb) F[(k0 + c) * f + r0 + r] = acc[i][j];
    }
}

// Panel step 3: trailing update C[r0.., c0..] −= P_r P_cᵀ with the panel P = F[:, kbeg:kbeg+kcnt] (lower tiles
// only; one or two panels, see the plan); task = (node, r0, c0, kbeg, kcnt). 64 threads, 8×8 outputs each (rows tx + 8i, columns ty + 8j); the panel is staged 16
// columns at a time through a double-buffered cp.async pipeline (loads of chunk c+1 overlap the DFMAs of c).
__device__ __forceinline__ void cp_async8(double* dst, const double* src, bool valid) {
  const uint32_t d = (uint32_t)__cvta_generic_to_shared(dst);
  const int sz = valid ? 8 : 0;  // zero-fill outside the front / panel
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(d), "l"(src), "r"(sz) : "memory");
}
__global__ void __launch_bounds__(64) mf_syrk_kernel(SparseArgs a, const int32_t* tasks) {
  __shared__ double As[2][16][MF_NB];
  __shared__ double Bs[2][16][MF_NB];
  const MfArgs& m = a.mf;
  const int32_t* tk = tasks + 5 * blockIdx.x;
  const int node = tk[0], r0 = tk[1], c0 = tk[2], k0 = tk[3], kb = tk[4];
  const int64_t f = m.fdim[node];
  double* F = m.F + m.foff[node];
  const int tid = threadIdx.x, tx = tid % 8, ty = tid / 8;
  auto stage = [&](int buf, int kk) {
#pragma unroll
    for (int t = 0; t < 16; ++t) {
      const int idx = tid + 64 * t;
      const int r = idx % MF_NB, kc = idx / MF_NB;
      const bool kin = kk + kc < kb;
      const double* col = F + (k0 + kk + (kin ? kc : 0)) * f;
      cp_async8(&As[buf][kc][r], col + (r0 + r < f ? r0 + r : 0), kin && r0 + r < f);
      cp_async8(&Bs[buf][kc][r], col + (c0 + r < f ? c0 + r : 0), kin && c0 + r < f);
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  // the accumulators start from the trailing block itself (every load before the first store: a final
  // col[r] −= acc read-modify-write on possibly aliasing columns would serialize its round trips)
  double acc[8][8];
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    const int c = c0 + ty + 8 * j;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int r = r0 + tx + 8 * i;
      acc[i][j] = (c < f && r < f && r >= c) ? F[(int64_t)c * f + r] : 0.0;
    }
  }
  const int nch = (kb + 15) / 16;
  stage(0, 0);
  for (int ch = 0; ch < nch; ++ch) {
    const int buf = ch & 1;
    if (ch + 1 < nch) {
      stage(buf ^ 1, (ch + 1) * 16);
      asm volatile("cp.async.wait_group 1;" ::: "memory");
    } else {
      asm volatile("cp.async.wait_group 0;" ::: "memory");
    }
    __syncthreads();
#pragma unroll 4
    for (int k = 0; k < 16; ++k) {
      double av[8], bv[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) av[i] = As[buf][k][tx + 8 * i];
#pragma unroll
      for (int j = 0; j < 8; ++j) bv[j] = Bs[buf][k][ty + 8 * j];
#pragma unroll
      for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[i][j] = fma(-av[i], bv[j], acc[i][j]);
    }
    __syncthreads();  // this buffer is refilled two chunks later
  }
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    const int c = c0 + ty + 8 * j;
    if (c >= f) continue;
    double* col = F + (int64_t)c * f;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int r = r0 + tx + 8 * i;
      if (r < f && r >= c) col[r] = acc[i][j];
    }
  }
}

// The same update on the fp64 tensor cores (mma.sync m8n8k4 .f64 = DMMA: 256 FMAs per warp instruction, so the
// issue slots the DFMA version spends on 8×8 outer products go free; measured peak 37.0 TFLOP/s vs 34.1 for DFMA,
// tools/dmma_peak.cu). 128 threads = 2×2 warps of 32×32 per 64×64 tile; the panel is staged as above (16 columns
// per stage, row stride 72 doubles: the fragment loads — 8 rows × 4 columns per warp — hit distinct banks).
// Fragments (PTX ISA, m8n8k4 .f64): a0 = A[g][t], b0 = B[t][g], c_e = C[g][2t + e] (g = lane / 4, t = lane % 4).
constexpr int SYRK_LD = MF_NB + 8;
__global__ void __launch_bounds__(128) mf_syrk_mma_kernel(SparseArgs a, const int32_t* tasks) {
  __shared__ __align__(16) double As[2][16][SYRK_LD];
  __shared__ __align__(16) double Bs[2][16][SYRK_LD];
  const MfArgs& m = a.mf;
  const int32_t* tk = tasks + 5 * blockIdx.x;
  const int node = tk[0], r0 = tk[1], c0 = tk[2], k0 = tk[3], kb = tk[4];
  const int64_t f = m.fdim[node];
  double* F = m.F + m.foff[node];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, t = lane & 3;
  const int wr = 32 * (warp >> 1), wc = 32 * (warp & 1);  // the warp's 32×32 sub-tile
  auto stage = [&](int buf, int kk) {
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int idx = tid + 128 * u;
      const int r = idx % MF_NB, kc = idx / MF_NB;
      const bool kin = kk + kc < kb;
      const double* col = F + (k0 + kk + (kin ? kc : 0)) * f;
      cp_async8(&As[buf][kc][r], col + (r0 + r < f ? r0 + r : 0), kin && r0 + r < f);
      cp_async8(&Bs[buf][kc][r], col + (c0 + r < f ? c0 + r : 0), kin && c0 + r < f);
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  // a diagonal tile's strictly upper sub-tile (warp rows 0-31, columns 32-63) holds nothing of the lower part
  const bool idle = r0 == c0 && wr < wc;
  double acc[4][4][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int r = r0 + wr + 8 * i + g, c = c0 + wc + 8 * j + 2 * t + e;
        acc[i][j][e] = (!idle && c < f && r < f && r >= c) ? F[(int64_t)c * f + r] : 0.0;
      }
  const int nch = (kb + 15) / 16;
  stage(0, 0);
  for (int ch = 0; ch < nch; ++ch) {
    const int buf = ch & 1;
    if (ch + 1 < nch) {
      stage(buf ^ 1, (ch + 1) * 16);
      asm volatile("cp.async.wait_group 1;" ::: "memory");
    } else {
      asm volatile("cp.async.wait_group 0;" ::: "memory");
    }
    __syncthreads();
    if (!idle) {
#pragma unroll
      for (int k = 0; k < 16; k += 4) {
        double av[4], bv[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) av[i] = -As[buf][k + t][wr + 8 * i + g];
#pragma unroll
        for (int j = 0; j < 4; ++j) bv[j] = Bs[buf][k + t][wc + 8 * j + g];
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j)
            asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                         : "+d"(acc[i][j][0]), "+d"(acc[i][j][1])
                         : "d"(av[i]), "d"(bv[j]));
      }
    }
    __syncthreads();  // this buffer is refilled two chunks later
  }
  if (idle) return;
#pragma unroll
  for (int j = 0; j < 4; ++j)
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const int c = c0 + wc + 8 * j + 2 * t + e;
      if (c >= f) continue;
      double* col = F + (int64_t)c * f;
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int r = r0 + wr + 8 * i + g;
        if (r < f && r >= c) col[r] = acc[i][j][e];
      }
    }
}

// ============================================================================ triangular solves
// Forward, one CTA per front of a level: w = [own rhs; 0] + children's boundary vectors; y = L11⁻¹ w_own
// (blocked by 64; the diagonal block is solved by warp 0 in shared memory); w_bnd −= L21 y. y goes to dst
// (point order), w_bnd stays in the node's solve vector for the parent.
__global__ void __launch_bounds__(SP_THREADS) mf_fwd_kernel(SparseArgs a, const int32_t* nodes, const double* src,
                                                           double* dst) {
  if (refine_gated(a)) return;
  extern __shared__ double sm[];
  const MfArgs& m = a.mf;
  const int node = nodes[blockIdx.x];
  const int n = m.nown[node];
  const int64_t f = m.fdim[node];
  double* w = sm;
  double* Ld = sm + ((f + 1) & ~1);  // [MF_NB][MF_NB + 1]
  const double* F = m.F + m.foff[node];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int first = m.own_first[node];
  for (int i = tid; i < f; i += blockDim.x)
    w[i] = i < n ? src[(i % 3) * a.np + m.ipos[first + i / 3]] : 0.0;
  __syncthreads();
  for (int ci = m.ch_off[node]; ci < m.ch_off[node + 1]; ++ci) {
    const int c = m.ch[ci];
    const int fc = m.fdim[c], nc = m.nown[c];
    const int32_t* map = m.ea_map + m.ea_off[c];
    const double* wc = m.wvec + m.woff[c];
    for (int i = tid; i < fc - nc; i += blockDim.x) w[mapped(map, i)] += wc[nc + i];
    __syncthreads();
  }
  for (int k0 = 0; k0 < n; k0 += MF_NB) {
    const int kb = min(MF_NB, n - k0);
    for (int idx = tid; idx < kb * kb; idx += blockDim.x) {
      const int r = idx % kb, c = idx / kb;
      const double v = F[(k0 + c) * f + k0 + r];
      Ld[r * (MF_NB + 1) + c] = r == c ? 1.0 / v : v;  // the diagonal as its reciprocal (no division in the chain)
    }
    __syncthreads();
    if (warp == 0) {
      for (int j = 0; j < kb; ++j) {
        const double xj = w[k0 + j] * Ld[j * (MF_NB + 1) + j];
        __syncwarp();
        if (lane == 0) w[k0 + j] = xj;
        for (int i = j + 1 + lane; i < kb; i += 32) w[k0 + i] -= Ld[i * (MF_NB + 1) + j] * xj;
        __syncwarp();
      }
    }
    __syncthreads();
    for (int64_t r = k0 + kb + tid; r < f; r += blockDim.x) {
      double s = 0.0;
      for (int j = 0; j < kb; ++j) s += F[(k0 + j) * f + r] * w[k0 + j];
      w[r] -= s;
    }
    __syncthreads();
  }
  for (int i = tid; i < n; i += blockDim.x) dst[(i % 3) * a.np + m.ipos[first + i / 3]] = w[i];
  double* wv = m.wvec + m.woff[node];
  for (int64_t i = n + tid; i < f; i += blockDim.x) wv[i] = w[i];
}

// Backward, one CTA per front, top level first: z = y_own − L21ᵀ x_bnd (x_bnd from the ancestors' solution),
// then L11ᵀ x_own = z by 64-blocks from the last. x goes to sol (point order).
__global__ void __launch_bounds__(SP_THREADS) mf_bwd_kernel(SparseArgs a, const int32_t* nodes, const double* ysrc,
                                                           double* sol) {
  if (refine_gated(a)) return;
  extern __shared__ double sm[];
  const MfArgs& m = a.mf;
  const int node = nodes[blockIdx.x];
  const int n = m.nown[node];
  const int64_t f = m.fdim[node];
  double* x = sm;
  double* Ld = sm + ((f + 1) & ~1);
  const double* F = m.F + m.foff[node];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
  const int first = m.own_first[node];
  const int32_t* bnd = m.bnd + m.bnd_off[node];
  for (int64_t i = tid; i < f; i += blockDim.x) {
    const int p = i < n ? m.ipos[first + i / 3] : m.ipos[bnd[(i - n) / 3]];
    x[i] = (i < n ? ysrc : sol)[(i % 3) * a.np + p];
  }
  __syncthreads();
  for (int i = warp; i < n; i += nw) {  // z_i = y_i − Σ_r L[r][i] x_r over boundary rows
    const double* col = F + (int64_t)i * f;
    double s = 0.0;
    for (int64_t r = n + lane; r < f; r += 32) s += col[r] * x[r];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_down_sync(0xffffffffu, s, o);
    if (lane == 0) x[i] -= s;
  }
  __syncthreads();
  const int nchunk = (n + MF_NB - 1) / MF_NB;
  for (int cidx = nchunk - 1; cidx >= 0; --cidx) {
    const int k0 = cidx * MF_NB, kb = min(MF_NB, n - k0);
    for (int idx = tid; idx < kb * kb; idx += blockDim.x) {
      const int r = idx % kb, c = idx / kb;
      const double v = F[(k0 + c) * f + k0 + r];
      Ld[r * (MF_NB + 1) + c] = r == c ? 1.0 / v : v;  // the diagonal as its reciprocal
    }
    __syncthreads();
    if (warp == 0) {
      for (int j = kb - 1; j >= 0; --j) {
        const double xj = x[k0 + j] * Ld[j * (MF_NB + 1) + j];
        __syncwarp();
        if (lane == 0) x[k0 + j] = xj;
        for (int i = lane; i < j; i += 32) x[k0 + i] -= Ld[j * (MF_NB + 1) + i] * xj;
        __syncwarp();
      }
    }
    __syncthreads();
    for (int i = warp; i < k0; i += nw) {  // earlier own entries: x_i −= Σ_{r in chunk} L[r][i] x_r
      const double* col = F + (int64_t)i * f + k0;
      double s = 0.0;
      for (int r = lane; r < kb; r += 32) s += col[r] * x[k0 + r];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) s += __shfl_down_sync(0xffffffffu, s, o);
      if (lane == 0) x[i] -= s;
    }
    __syncthreads();
  }
  for (int i = tid; i < n; i += blockDim.x) sol[(i % 3) * a.np + m.ipos[first + i / 3]] = x[i];
}

// ---- triangular solves of large fronts, parallel over 64-row / 64-column tiles, one launch per group of MF_SG 64-chunks
// Forward init: w = [own rhs; 0] + the children's boundary vectors (into the node's solve vector).
__global__ void __launch_bounds__(SP_THREADS) mf_fwd_init_kernel(SparseArgs a, const int32_t* nodes, const double* src) {
  if (refine_gated(a)) return;
  const MfArgs& m = a.mf;
  const int node = nodes[blockIdx.x];
  const int n = m.nown[node];
  const int64_t f = m.fdim[node];
  const int first = m.own_first[node];
  double* w = m.wvec + m.woff[node];
  for (int64_t i = threadIdx.x; i < f; i += blockDim.x)
    w[i] = i < n ? src[(i % 3) * a.np + m.ipos[first + i / 3]] : 0.0;
  __syncthreads();
  for (int ci = m.ch_off[node]; ci < m.ch_off[node + 1]; ++ci) {
    const int c = m.ch[ci];
    const int fc = m.fdim[c], nc = m.nown[c];
    const int32_t* map = m.ea_map + m.ea_off[c];
    const double* wc = m.wvec + m.woff[c];
    for (int i = threadIdx.x; i < fc - nc; i += blockDim.x) w[mapped(map, i)] += wc[nc + i];
    __syncthreads();
  }
}

// Forward group of MF_SG chunks from c0 (chunks of 64 own columns; one launch per group instead of per chunk):
// every CTA forms the group's y redundantly, chunk by chunk, y_s = L_ss⁻¹ (w_s − Σ_{t<s} L_st y_t) with the
// L_st blocks read from the front (L2-resident, 32 KB per pair); the writer task stores y, the others update
// their 64 rows below the group: w_r −= Σ_{j in group} L[r][j] y_j. task = (node, r0 or −1, writer flag).
__global__ void __launch_bounds__(SP_THREADS) mf_fwd_chunk_kernel(SparseArgs a, const int32_t* tasks, int c0,
                                                                 double* dst) {
  if (refine_gated(a)) return;
  __shared__ double yc[MF_SG * MF_NB];
  __shared__ double wl[MF_NB];
  __shared__ double part[4][MF_NB];
  const MfArgs& m = a.mf;
  const int node = tasks[3 * blockIdx.x], r0 = tasks[3 * blockIdx.x + 1], writer = tasks[3 * blockIdx.x + 2];
  const int n = m.nown[node];
  const int64_t f = m.fdim[node];
  const int k00 = c0 * MF_NB, cols = min(MF_SG * MF_NB, n - k00);
  const double* F = m.F + m.foff[node];
  double* w = m.wvec + m.woff[node];
  const int tid = threadIdx.x, i = tid % MF_NB, g = tid / MF_NB;
  for (int s = 0; s * MF_NB < cols; ++s) {
    const int k0 = k00 + s * MF_NB, kb = min(MF_NB, n - k0);
    {  // w_s − Σ_{t<s} L_st y_t: row k0+i, 4 threads per row over the group's earlier columns
      double acc = 0.0;
      if (i < kb)
        for (int j = g; j < s * MF_NB; j += 4) acc += F[(int64_t)(k00 + j) * f + k0 + i] * yc[j];
      part[g][i] = acc;
    }
    __syncthreads();
    if (tid < MF_NB) wl[tid] = tid < kb ? w[k0 + tid] - (part[0][tid] + part[1][tid] + part[2][tid] + part[3][tid]) : 0.0;
    __syncthreads();
    {  // y_s[i] = Σ_j Linv[i][j] wl[j]: 4 threads per row
      const double* li = m.linv + m.loff[node] + (int64_t)(c0 + s) * MF_NB * MF_NB;
      double acc = 0.0;
      if (i < kb)
        for (int j = g * 16; j < min(kb, g * 16 + 16); ++j) acc += li[i * MF_NB + j] * wl[j];
      part[g][i] = acc;
    }
    __syncthreads();
    if (tid < MF_NB) yc[s * MF_NB + tid] = part[0][tid] + part[1][tid] + part[2][tid] + part[3][tid];
    __syncthreads();
  }
  if (writer)
    for (int j = tid; j < cols; j += blockDim.x) {
      const int e = k00 + j;
      dst[(e % 3) * a.np + m.ipos[m.own_first[node] + e / 3]] = yc[j];
    }
  if (r0 < 0) return;
  const int64_t r = r0 + i;
  double acc = 0.0;
  if (r < f)
    for (int j = g; j < cols; j += 4) acc += F[(int64_t)(k00 + j) * f + r] * yc[j];
  part[g][i] = acc;
  __syncthreads();
  if (tid < MF_NB && r0 + tid < f) w[r0 + tid] -= part[0][tid] + part[1][tid] + part[2][tid] + part[3][tid];
}

// Backward init: the node's vector ← [y_own; x_bnd] (x_bnd from the ancestors' solution).
__global__ void __launch_bounds__(SP_THREADS) mf_bwd_init_kernel(SparseArgs a, const int32_t* nodes, const double* ysrc,
                                                                const double* sol) {
  if (refine_gated(a)) return;
  const MfArgs& m = a.mf;
  const int node = nodes[blockIdx.x];
  const int n = m.nown[node];
  const int64_t f = m.fdim[node];
  const int first = m.own_first[node];
  const int32_t* bnd = m.bnd + m.bnd_off[node];
  double* x = m.wvec + m.woff[node];
  for (int64_t i = threadIdx.x; i < f; i += blockDim.x) {
    const int p = i < n ? m.ipos[first + i / 3] : m.ipos[bnd[(i - n) / 3]];
    x[i] = (i < n ? ysrc : sol)[(i % 3) * a.np + p];
  }
}

// Backward boundary product: z_i = y_i − Σ_{r ≥ n} L[r][i] x_r for the 64 own columns of a tile; task = (node, t0).
__global__ void __launch_bounds__(SP_THREADS) mf_bwd_bnd_kernel(SparseArgs a, const int32_t* tasks) {
  if (refine_gated(a)) return;
  const MfArgs& m = a.mf;
  const int node = tasks[2 * blockIdx.x], t0 = tasks[2 * blockIdx.x + 1];
  const int n = m.nown[node];
  const int64_t f = m.fdim[node];
  const double* F = m.F + m.foff[node];
  double* x = m.wvec + m.woff[node];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int cc = warp; cc < MF_NB; cc += SP_THREADS / 32) {
    const int i = t0 + cc;
    if (i >= n) break;
    const double* col = F + (int64_t)i * f;
    double s = 0.0;
    for (int64_t r = n + lane; r < f; r += 32) s += col[r] * x[r];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_down_sync(0xffffffffu, s, o);
    if (lane == 0) x[i] -= s;
  }
}

// Backward group of MF_SG chunks from c0 (the last group first; inside it the last chunk first): every CTA forms
// x_s = L_ss⁻ᵀ (z_s − Σ_{t>s} L_tsᵀ x_t) redundantly; the writer stores x, the others update the 64 earlier own
// columns of their tile: z_i −= Σ_{r in group} L[r][i] x_r. task = (node, t0 or −1, writer).
__global__ void __launch_bounds__(SP_THREADS) mf_bwd_chunk_kernel(SparseArgs a, const int32_t* tasks, int c0,
                                                                 double* sol) {
  if (refine_gated(a)) return;
  __shared__ double xc[MF_SG * MF_NB];
  __shared__ double zl[MF_NB];
  __shared__ double part[4][MF_NB];
  const MfArgs& m = a.mf;
  const int node = tasks[3 * blockIdx.x], t0 = tasks[3 * blockIdx.x + 1], writer = tasks[3 * blockIdx.x + 2];
  const int n = m.nown[node];
  const int64_t f = m.fdim[node];
  const int k00 = c0 * MF_NB, cols = min(MF_SG * MF_NB, n - k00);
  const double* F = m.F + m.foff[node];
  double* x = m.wvec + m.woff[node];
  const int tid = threadIdx.x;
  const int cc = tid / 4, g4 = tid % 4;  // column cc of a 64-column block, 4 threads per column
  for (int s = (cols - 1) / MF_NB; s >= 0; --s) {
    const int k0 = k00 + s * MF_NB, kb = min(MF_NB, n - k0);
    {  // z_s − Σ_{t>s} L_tsᵀ x_t: column k0+cc over the group's later rows
      double acc = 0.0;
      if (cc < kb) {
        const double* col = F + (int64_t)(k0 + cc) * f + k00;
        for (int r = (s + 1) * MF_NB + g4; r < cols; r += 4) acc += col[r] * xc[r];
      }
      acc += __shfl_down_sync(0xffffffffu, acc, 2, 4);
      acc += __shfl_down_sync(0xffffffffu, acc, 1, 4);
      if (g4 == 0) zl[cc] = cc < kb ? x[k0 + cc] - acc : 0.0;
    }
    __syncthreads();
    {  // x_s[i] = Σ_{j ≥ i} Linv[j][i] zl[j]
      const double* li = m.linv + m.loff[node] + (int64_t)(c0 + s) * MF_NB * MF_NB;
      const int i = tid % MF_NB, g = tid / MF_NB;
      double acc = 0.0;
      if (i < kb)
        for (int j = max(i, g * 16); j < min(kb, g * 16 + 16); ++j) acc += li[j * MF_NB + i] * zl[j];
      part[g][i] = acc;
    }
    __syncthreads();
    if (tid < MF_NB) xc[s * MF_NB + tid] = part[0][tid] + part[1][tid] + part[2][tid] + part[3][tid];
    __syncthreads();
  }
  if (writer)
    for (int j = tid; j < cols; j += blockDim.x) {
      const int e = k00 + j;
      sol[(e % 3) * a.np + m.ipos[m.own_first[node] + e / 3]] = xc[j];
    }
  if (t0 < 0) return;
  const int i = t0 + cc;
  double acc = 0.0;
  const double* col = F + (int64_t)i * f + k00;
  for (int r = g4; r < cols; r += 4) acc += col[r] * xc[r];
  acc += __shfl_down_sync(0xffffffffu, acc, 2, 4);
  acc += __shfl_down_sync(0xffffffffu, acc, 1, 4);
  if (g4 == 0 && i < k00) x[i] -= acc;
}

// ============================================================================ host side: launches
constexpr int PANEL_SMEM = 2 * MF_NB * (MF_NB + 1) * (int)sizeof(double);

cudaError_t sparse_init() {
  int dev = 0, v = 0;
  cudaError_t e;
  if ((e = cudaGetDevice(&dev))) return e;
  if ((e = cudaDeviceGetAttribute(&v, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev))) return e;
  auto opt_in = [&](const void* fn) {  // all of the opt-in shared memory beyond the kernel's static part
    cudaFuncAttributes fa;
    cudaError_t r = cudaFuncGetAttributes(&fa, fn);
    if (r == cudaSuccess)
      r = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, v - (int)fa.sharedSizeBytes);
    return r;
  };
  if ((e = opt_in((const void*)mf_small_kernel))) return e;
  if ((e = opt_in((const void*)mf_fwd_kernel))) return e;
  if ((e = opt_in((const void*)mf_bwd_kernel))) return e;
  if ((e = cudaFuncSetAttribute(mf_potrf_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, PANEL_SMEM))) return e;
  if ((e = cudaFuncSetAttribute(mf_trsm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, PANEL_SMEM))) return e;
  return cudaSuccess;
}

static size_t solve_smem(int max_f) { return sizeof(double) * (((max_f + 1) & ~1) + MF_NB * (MF_NB + 1)); }

static int grid_for(int64_t n) { return (int)std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, 148 * 16)); }

static cudaError_t mf_solve(const SparsePlan& sp, const SparseArgs& a, const int32_t* LN, const int32_t* T,
                            const double* src, double* dst, cudaStream_t st) {
  const int nl = (int)sp.levels.size();
  for (int l = 0; l < nl; ++l) {  // forward: leaves first
    const auto& L = sp.levels[l];
    if (L.n_small)
      mf_fwd_kernel<<<(unsigned)L.n_small, SP_THREADS, solve_smem(L.max_f_small), st>>>(a, LN + L.small, src, a.yy);
    if (L.n_big) {
      mf_fwd_init_kernel<<<(unsigned)L.n_big, SP_THREADS, 0, st>>>(a, LN + L.big, src);
      for (size_t c = 0; c < L.fwd.size(); ++c)
        mf_fwd_chunk_kernel<<<(unsigned)L.n_fwd[c], SP_THREADS, 0, st>>>(a, T + L.fwd[c], (int)c * MF_SG, a.yy);
    }
  }
  for (int l = nl - 1; l >= 0; --l) {  // backward: root first
    const auto& L = sp.levels[l];
    if (L.n_small)
      mf_bwd_kernel<<<(unsigned)L.n_small, SP_THREADS, solve_smem(L.max_f_small), st>>>(a, LN + L.small, a.yy, dst);
    if (L.n_big) {
      mf_bwd_init_kernel<<<(unsigned)L.n_big, SP_THREADS, 0, st>>>(a, LN + L.big, a.yy, dst);
      if (L.n_bwdb) mf_bwd_bnd_kernel<<<(unsigned)L.n_bwdb, SP_THREADS, 0, st>>>(a, T + L.bwdb);
      for (int c = (int)L.bwd.size() - 1; c >= 0; --c)
        mf_bwd_chunk_kernel<<<(unsigned)L.n_bwd[c], SP_THREADS, 0, st>>>(a, T + L.bwd[c], c * MF_SG, dst);
    }
  }
  return cudaGetLastError();
}

cudaError_t sparse_step(const Plan& p, const DevPtrs& d, const StepConsts& k, cudaStream_t st) {
  SparseArgs a = d.sparse;
  a.k = k;
  const SparsePlan& sp = p.sparse;
  sparse_predict_kernel<<<grid_for(a.n), 256, 0, st>>>(a);
  if (sp.np == 0) {
    sparse_update_kernel<<<grid_for(a.n), 256, 0, st>>>(a);
    return cudaGetLastError();
  }
  if (a.nproj) proj_rows_kernel<<<(unsigned)((a.nproj + 127) / 128), 128, 0, st>>>(a);
  sparse_rhs_kernel<<<grid_for(a.np), 256, 0, st>>>(a);
  cudaError_t e;
#ifdef MF_ZERO_FULL
  if ((e = cudaMemsetAsync(a.mf.F, 0, sizeof(double) * sp.front_doubles, st))) return e;
#else
  if (sp.n_zero) mf_zero_kernel<<<(unsigned)sp.n_zero, SP_THREADS, 0, st>>>(a, d.sparse_tasks + sp.zero);
#endif
  mf_assemble_kernel<<<grid_for(a.mf.nblk), 256, 0, st>>>(a);
  const int32_t* LN = d.sparse_lev;
  const int32_t* T = d.sparse_tasks;
  for (const auto& L : sp.levels) {
    if (L.n_small)
      mf_small_kernel<<<(unsigned)L.n_small, SP_THREADS, sizeof(double) * L.max_f_small * L.max_f_small, st>>>(
          a, LN + L.small);
    for (size_t s = 0; s < L.ea.size(); ++s)
      if (L.n_ea[s]) mf_ea_kernel<<<(unsigned)L.n_ea[s], 128, 0, st>>>(a, T + L.ea[s], (int)s);
    for (size_t pi = 0; pi < L.panels.size(); ++pi) {
      const auto& P = L.panels[pi];
      const int k0 = (int)pi * MF_NB;
      if (P.n_potrf) mf_potrf_kernel<<<(unsigned)P.n_potrf, SP_THREADS, PANEL_SMEM, st>>>(a, T + P.potrf, k0);
      if (P.n_trsm) mf_trsm_kernel<<<(unsigned)P.n_trsm, SP_THREADS, PANEL_SMEM, st>>>(a, T + P.trsm, k0);
      if (P.n_syrk) {
        if (sp.syrk_dfma)
          mf_syrk_kernel<<<(unsigned)P.n_syrk, 64, 0, st>>>(a, T + P.syrk);
        else
          mf_syrk_mma_kernel<<<(unsigned)P.n_syrk, 128, 0, st>>>(a, T + P.syrk);
      }
    }
  }
  if ((e = cudaGetLastError())) return e;
  if ((e = mf_solve(sp, a, LN, T, a.rhs, a.lam, st))) return e;
  for (int it = 0; it < sp.refine; ++it) {  // iterative refinement against the exact S (matrix-free)
    mv_body_kernel<<<grid_for(a.n), 256, 0, st>>>(a, a.lam);
    mv_point_kernel<<<grid_for(a.np), 256, 0, st>>>(a);
    refine_gate_kernel<<<1, 1, 0, st>>>(a, it);
    SparseArgs g = a;
    g.gate = a.iters + 1;
    if ((e = mf_solve(sp, g, LN, T, a.res, a.dl, st))) return e;
    axpy_kernel<<<grid_for(3 * a.np), 256, 0, st>>>(a.lam, a.dl, 3 * a.np, g.gate);
  }
  sparse_update_kernel<<<grid_for(a.n), 256, 0, st>>>(a);
  return cudaGetLastError();
}

// ============================================================================ line Gauss-Seidel (Case IV)
// S_pq for two joint points: Σ over the bodies j they share of s_p s_q R_j P_j(ȳ_p, ȳ_q) R_jᵀ.
__device__ void gs_block(const SparseArgs& a, int32_t p, int32_t q, double* S) {
#pragma unroll
  for (int e = 0; e < 9; ++e) S[e] = 0.0;
  for (int sp = 0; sp < 2; ++sp) {
    const int32_t j = sp == 0 ? a.pa[p] : a.pb[p];
    if (j < 0) continue;
    for (int sq = 0; sq < 2; ++sq) {
      const int32_t jq = sq == 0 ? a.pa[q] : a.pb[q];
      if (jq != j) continue;
      double R[9], P[9], T[9];
      body_R(a, j, R);
      HinvBlk H;
      body_hinv(a, j, H);
      pblock(H, a.py + 6 * p + 3 * sp, a.py + 6 * q + 3 * sq, P);
      rot_conj(R, P, T);
      const double sg = (sp == sq) ? 1.0 : -1.0;
#pragma unroll
      for (int e = 0; e < 9; ++e) S[e] += sg * T[e];
    }
  }
}

__device__ __forceinline__ double* gs_fac(const SparseArgs& a, int64_t pos, int comp) {
  return a.gs.fac + (int64_t)comp * a.np + pos;
}

// Per step, one thread per chain: assemble the chain's diagonal and coupling blocks and factor them (block Thomas:
// D'_0 = D_0, L_k = B_{k−1}ᵀ D'_{k−1}⁻¹, D'_k = D_k − L_k B_{k−1}); keeps D'⁻¹, L, B per position.
__global__ void gs_factor_kernel(SparseArgs a, int32_t nchain) {
  const int32_t c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= nchain) return;
  const int32_t lo = a.gs.chain_off[c], hi = a.gs.chain_off[c + 1];
  double Lp[9], Bp[9], Dpi[6];
  for (int32_t k = lo; k < hi; ++k) {
    const int32_t p = a.gs.chain_pts[k];
    double D[9];
    gs_block(a, p, p, D);
    if (k > lo) {  // L = Bpᵀ Dpi, D −= L Bp
      double Dif[9];
      full_from_sym(Dpi, Dif);
      mat3_mul_at(Bp, Dif, Lp);
      double T[9];
      mat3_mul(Lp, Bp, T);
#pragma unroll
      for (int e = 0; e < 9; ++e) D[e] -= T[e];
    } else {
#pragma unroll
      for (int e = 0; e < 9; ++e) Lp[e] = 0.0;
    }
    double Ds[6];
    Ds[0] = D[0]; Ds[1] = 0.5 * (D[1] + D[3]); Ds[2] = 0.5 * (D[2] + D[6]);
    Ds[3] = D[4]; Ds[4] = 0.5 * (D[5] + D[7]); Ds[5] = D[8];
    if (!sym_inv_spd(Ds, Dpi)) sreport(a.k, ERR_SINGULAR);
    if (k + 1 < hi)
      gs_block(a, p, a.gs.chain_pts[k + 1], Bp);
    else
#pragma unroll
      for (int e = 0; e < 9; ++e) Bp[e] = 0.0;
#pragma unroll
    for (int e = 0; e < 6; ++e) *gs_fac(a, k, e) = Dpi[e];
#pragma unroll
    for (int e = 0; e < 9; ++e) {
      *gs_fac(a, k, 6 + e) = Lp[e];
      *gs_fac(a, k, 15 + e) = Bp[e];
    }
  }
}

__device__ __forceinline__ void atomic_max_pos(unsigned long long* slot, double v) {
  atomicMax(slot, (unsigned long long)__double_as_longlong(v));  // v ≥ 0: the bit patterns order like the values
}

// max |r| over the points (the residual scale of the stopping test)
__global__ void gs_rmax_kernel(SparseArgs a) {
  double m = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < 3 * a.np; i += (int64_t)gridDim.x * blockDim.x)
    m = fmax(m, fabs(a.rhs[i]));
  for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) atomic_max_pos(a.gs.resmax, m);
}

// Stopping test before sweep `sweep`: sweep − 1's residual max|r − Sλ| ≤ tol · max(max|r|, max|Sλ|) (the second
// scale matters for a warm start, where the joints are nearly satisfied but λ and Sλ are not small).
__device__ __forceinline__ bool gs_converged(const SparseArgs& a, int sweep) {
  if (sweep == 0) return false;
  const double r0 = __longlong_as_double((long long)a.gs.resmax[0]);
  const double rs = __longlong_as_double((long long)a.gs.resmax[2 * sweep - 1]);
  const double sv = __longlong_as_double((long long)a.gs.resmax[2 * sweep]);
  return rs <= a.gs.tol * fmax(r0, sv);
}

// One colour of sweep `sweep`, one thread per chain of the colour: the chain's residual res = r − (J H̃⁻¹Jᵀλ) from the
// per-body v = H̃⁻¹Jᵀλ (kept current), the exact chain solve S_cc δ = res (forward / backward Thomas), λ += δ, and
// v_j += H̃_j⁻¹ Σ s Γᵀδ for the chain's bodies (no other chain of the colour touches them). The residual before the
// update feeds the stopping test of the next sweep; a converged step skips the remaining sweeps.
__global__ void gs_color_kernel(SparseArgs a, int32_t color, int32_t sweep) {
  if (gs_converged(a, sweep)) return;
  const int32_t c = a.gs.color_off[color] + blockIdx.x * blockDim.x + threadIdx.x;
  double rmax = 0.0, smax = 0.0;
  if (c < a.gs.color_off[color + 1]) {
    const int32_t lo = a.gs.chain_off[c], hi = a.gs.chain_off[c + 1];
    double y[3] = {0, 0, 0};
    for (int32_t k = lo; k < hi; ++k) {  // forward: y_k = res_k − L_k y_{k−1}
      const int32_t p = a.gs.chain_pts[k];
      double r[3], sl[3] = {0, 0, 0};  // sl = (S λ)_p = (J v)_p
      for (int side = 0; side < 2; ++side) {
        const int64_t j = side == 0 ? a.pa[p] : a.pb[p];
        if (j < 0) continue;
        const double* yb = a.py + 6 * p + 3 * side;
        const double sg = side == 0 ? 1.0 : -1.0;
#pragma unroll
        for (int e = 0; e < 3; ++e)
          sl[e] += sg * (a.vv[(0 + e) * a.n + j] * yb[0] + a.vv[(3 + e) * a.n + j] * yb[1] +
                         a.vv[(6 + e) * a.n + j] * yb[2] + a.vv[(9 + e) * a.n + j]);
      }
#pragma unroll
      for (int e = 0; e < 3; ++e) r[e] = a.rhs[e * a.np + p] - sl[e];
      rmax = fmax(rmax, fmax(fabs(r[0]), fmax(fabs(r[1]), fabs(r[2]))));
      smax = fmax(smax, fmax(fabs(sl[0]), fmax(fabs(sl[1]), fabs(sl[2]))));
      double L[9], t[3];
#pragma unroll
      for (int e = 0; e < 9; ++e) L[e] = *gs_fac(a, k, 6 + e);
      mat3_vec(L, y, t);
#pragma unroll
      for (int e = 0; e < 3; ++e) {
        y[e] = r[e] - t[e];
        a.yy[e * a.np + p] = y[e];
      }
    }
    double x[3] = {0, 0, 0};
    for (int32_t k = hi - 1; k >= lo; --k) {  // backward: x_k = D'_k⁻¹ (y_k − B_k x_{k+1}); λ += x; v += H̃⁻¹Jᵀx
      const int32_t p = a.gs.chain_pts[k];
      double B[9], Di[6], t[3], v[3];
#pragma unroll
      for (int e = 0; e < 9; ++e) B[e] = *gs_fac(a, k, 15 + e);
#pragma unroll
      for (int e = 0; e < 6; ++e) Di[e] = *gs_fac(a, k, e);
      mat3_vec(B, x, t);
#pragma unroll
      for (int e = 0; e < 3; ++e) v[e] = a.yy[e * a.np + p] - t[e];
      sym_vec(Di, v, x);
#pragma unroll
      for (int e = 0; e < 3; ++e) a.lam[e * a.np + p] += x[e];
      for (int side = 0; side < 2; ++side) {
        const int64_t j = side == 0 ? a.pa[p] : a.pb[p];
        if (j < 0) continue;
        double R[9], g[12], u[12], wl[3], dv[3];
        body_R(a, j, R);
#pragma unroll
        for (int e = 0; e < 12; ++e) g[e] = 0.0;
        mat3t_vec(R, x, wl);
        add_point_force(g, a.py + 6 * p + 3 * side, wl, side == 0 ? 1.0 : -1.0);
        HinvBlk H;
        body_hinv(a, j, H);
        hinv_apply(H, g, u);
#pragma unroll
        for (int kb = 0; kb < 4; ++kb) {
          mat3_vec(R, u + 3 * kb, dv);
#pragma unroll
          for (int e = 0; e < 3; ++e) a.vv[(3 * kb + e) * a.n + j] += dv[e];
        }
      }
    }
  }
  for (int o = 16; o > 0; o >>= 1) {
    rmax = fmax(rmax, __shfl_xor_sync(0xffffffffu, rmax, o));
    smax = fmax(smax, __shfl_xor_sync(0xffffffffu, smax, o));
  }
  if ((threadIdx.x & 31) == 0) {
    atomic_max_pos(a.gs.resmax + 1 + 2 * sweep, rmax);
    atomic_max_pos(a.gs.resmax + 2 + 2 * sweep, smax);
  }
}

// sweeps run (the first whose starting residual met the tolerance, else max_sweeps) → iters[0] (mabd_solver_stats)
__global__ void gs_count_kernel(SparseArgs a) {
  int s = 1;
  while (s <= a.gs.max_sweeps && !gs_converged(a, s)) ++s;
  a.iters[0] = min(s, a.gs.max_sweeps);
}

cudaError_t gs_step(const Plan& p, const DevPtrs& d, const StepConsts& k, cudaStream_t st) {
  SparseArgs a = d.sparse;
  a.k = k;
  const SparsePlan& sp = p.sparse;
  sparse_predict_kernel<<<grid_for(a.n), 256, 0, st>>>(a);
  if (sp.np > 0) {
    sparse_rhs_kernel<<<grid_for(a.np), 256, 0, st>>>(a);
    cudaError_t e;
    if ((e = cudaMemsetAsync(a.gs.resmax, 0, sizeof(unsigned long long) * (1 + 2 * sp.gs_sweeps), st))) return e;
    gs_rmax_kernel<<<grid_for(3 * a.np), 256, 0, st>>>(a);
    const int32_t nch = (int32_t)(sp.gs_chain_off.size() - 1);
    gs_factor_kernel<<<(unsigned)((nch + 127) / 128), 128, 0, st>>>(a, nch);
    mv_body_kernel<<<grid_for(a.n), 256, 0, st>>>(a, a.lam);  // v = H̃⁻¹Jᵀλ of the warm start (last step's λ)
    for (int s2 = 0; s2 < sp.gs_sweeps; ++s2)
      for (int c = 0; c < sp.gs_ncolor; ++c) {
        const int32_t nc = sp.gs_color_off[c + 1] - sp.gs_color_off[c];
        gs_color_kernel<<<(unsigned)((nc + 127) / 128), 128, 0, st>>>(a, c, s2);
      }
    gs_count_kernel<<<1, 1, 0, st>>>(a);
  }
  sparse_update_kernel<<<grid_for(a.n), 256, 0, st>>>(a);
  return cudaGetLastError();
}

// ============================================================================ host side: symbolic analysis
namespace {

struct NdBuild {
  const double* q0;
  const std::vector<int32_t>& pa;
  const std::vector<int32_t>& pb;
  std::vector<int8_t> mark;
  std::vector<std::vector<int32_t>> nodes;  // point sets, in postorder

  NdBuild(const double* q, int64_t n, const std::vector<int32_t>& a, const std::vector<int32_t>& b)
      : q0(q), pa(a), pb(b), mark(n, 0) {}

  double coord(int32_t b, int ax) const { return q0[12 * (int64_t)b + 9 + ax]; }

  void build(std::vector<int32_t>& bodies, std::vector<int32_t>& pts, int depth) {
    if (pts.empty()) return;
    if ((int)pts.size() <= MF_LEAF_PTS || bodies.size() <= 1 || depth > 64) {
      nodes.push_back(pts);
      return;
    }
    double lo[3] = {1e300, 1e300, 1e300}, hi[3] = {-1e300, -1e300, -1e300};
    for (int32_t b : bodies)
      for (int ax = 0; ax < 3; ++ax) {
        lo[ax] = std::min(lo[ax], coord(b, ax));
        hi[ax] = std::max(hi[ax], coord(b, ax));
      }
    int ax = 0;
    for (int i = 1; i < 3; ++i)
      if (hi[i] - lo[i] > hi[ax] - lo[ax]) ax = i;
    const size_t half = bodies.size() / 2;
    if (hi[ax] > lo[ax]) {
      std::nth_element(bodies.begin(), bodies.begin() + half, bodies.end(), [&](int32_t x, int32_t y) {
        const double cx = coord(x, ax), cy = coord(y, ax);
        return cx < cy || (cx == cy && x < y);
      });
    } else {
      std::nth_element(bodies.begin(), bodies.begin() + half, bodies.end());
    }
    std::vector<int32_t> BL(bodies.begin(), bodies.begin() + half), BR(bodies.begin() + half, bodies.end());
    for (int32_t b : BL) mark[b] = 0;
    for (int32_t b : BR) mark[b] = 1;
    std::vector<int32_t> PL, PR, PS;
    for (int32_t p : pts) {
      const int sa = mark[pa[p]];
      const int sb = pb[p] >= 0 ? mark[pb[p]] : sa;
      (sa != sb ? PS : sa == 0 ? PL : PR).push_back(p);
    }
    if (PL.empty() && PR.empty()) {  // no separation possible: one dense node
      nodes.push_back(pts);
      return;
    }
    std::vector<int32_t>().swap(pts);
    build(BL, PL, depth + 1);
    build(BR, PR, depth + 1);
    if (!PS.empty()) nodes.push_back(PS);
  }
};

}  // namespace

static bool mf_symbolic(const mabd_bodies* B, Plan* plan, std::string* msg) {
  SparsePlan& s = plan->sparse;
  const int64_t P = s.np, n = plan->n;
  if (P == 0) {
    s.nnode = 0;
    return true;
  }
  // ---- nested dissection on the bodies' initial positions
  NdBuild nd(B->q0, n, s.pa, s.pb);
  {
    std::vector<char> used(n, 0);
    for (int64_t p = 0; p < P; ++p) {
      used[s.pa[p]] = 1;
      if (s.pb[p] >= 0) used[s.pb[p]] = 1;
    }
    std::vector<int32_t> bodies, pts(P);
    for (int64_t b = 0; b < n; ++b)
      if (used[b]) bodies.push_back((int32_t)b);
    std::iota(pts.begin(), pts.end(), 0);
    nd.build(bodies, pts, 0);
  }
  const int NN = (int)nd.nodes.size();
  s.nnode = NN;
  s.epos.assign(P, -1);
  s.ipos.assign(P, -1);
  s.own_first.assign(NN, 0);
  s.nown.assign(NN, 0);
  std::vector<int32_t> owner(P), last(NN);
  {
    int32_t c = 0;
    for (int i = 0; i < NN; ++i) {
      s.own_first[i] = c;
      for (int32_t p : nd.nodes[i]) {
        s.epos[p] = c;
        s.ipos[c] = p;
        owner[c] = i;
        ++c;
      }
      s.nown[i] = 3 * (int32_t)nd.nodes[i].size();
      last[i] = c;
    }
    if (c != P) return *msg = "sparse symbolic: ordering lost points", false;
  }
  // ---- point adjacency (points sharing a body)
  auto for_neighbors = [&](int32_t p, const std::function<void(int32_t)>& fn) {
    for (int side = 0; side < 2; ++side) {
      const int32_t b = side == 0 ? s.pa[p] : s.pb[p];
      if (b < 0) continue;
      for (int i = s.inc_off[b]; i < s.inc_off[b + 1]; ++i) fn(s.inc[i] >> 1);
    }
  };
  // ---- boundary sets and the assembly tree (parent = owner of the smallest boundary position)
  std::vector<std::vector<int32_t>> bnd(NN), kids(NN);
  s.parent.assign(NN, -1);
  std::vector<int32_t> tmp;
  for (int i = 0; i < NN; ++i) {
    tmp.clear();
    for (int32_t p : nd.nodes[i])
      for_neighbors(p, [&](int32_t q) {
        if (s.epos[q] >= last[i]) tmp.push_back(s.epos[q]);
      });
    for (int c : kids[i])
      for (int32_t e : bnd[c])
        if (e >= last[i]) tmp.push_back(e);
    std::sort(tmp.begin(), tmp.end());
    tmp.erase(std::unique(tmp.begin(), tmp.end()), tmp.end());
    bnd[i] = tmp;
    if (!tmp.empty()) {
      const int par = owner[tmp[0]];
      s.parent[i] = par;
      kids[par].push_back(i);
    }
  }
  // ---- fronts, extend-add maps, heights
  s.fdim.assign(NN, 0);
  s.foff.assign(NN, 0);
  s.woff.assign(NN, 0);
  s.height.assign(NN, 0);
  s.bnd_off.assign(NN, 0);
  s.ea_off.assign(NN, 0);
  s.ch_off.assign(NN + 1, 0);
  s.bnd.clear();
  s.ea_map.clear();
  s.ch.clear();
  int64_t fo = 0, wo = 0;
  double flops = 0.0;
  s.max_f = 0;
  for (int i = 0; i < NN; ++i) {
    const int64_t nn = s.nown[i], mm = 3 * (int64_t)bnd[i].size();
    const int64_t f = nn + mm;
    if (f > 20000) return *msg = "sparse symbolic: front larger than 20000 rows (dense coupling too wide)", false;
    s.fdim[i] = (int32_t)f;
    s.max_f = std::max<int32_t>(s.max_f, (int32_t)f);
    s.foff[i] = fo;
    fo += (f * f + 31) & ~int64_t(31);
    s.woff[i] = wo;
    wo += (f + 3) & ~int64_t(3);
    // algorithmic multiply-adds of the front: POTRF nn³/6, TRSM nn²mm/2, SYRK (lower) nn·mm²/2
    flops += (double)nn * nn * nn / 6.0 + 0.5 * (double)nn * nn * mm + 0.5 * (double)nn * mm * mm;
    s.bnd_off[i] = (int32_t)s.bnd.size();
    s.bnd.insert(s.bnd.end(), bnd[i].begin(), bnd[i].end());
    for (int c : kids[i]) s.height[i] = std::max(s.height[i], s.height[c] + 1);
    s.ch_off[i + 1] = s.ch_off[i] + (int32_t)kids[i].size();
    s.ch.insert(s.ch.end(), kids[i].begin(), kids[i].end());
  }
  s.front_doubles = fo;
  s.w_doubles = wo;
  s.flops = 2.0 * flops;
  for (int i = 0; i < NN; ++i) {
    s.ea_off[i] = (int32_t)s.ea_map.size();
    const int par = s.parent[i];
    if (par < 0) continue;
    const int32_t pf = s.own_first[par], pl = last[par];
    const std::vector<int32_t>& pb = bnd[par];
    for (int32_t e : bnd[i]) {
      int32_t pos;
      if (e >= pf && e < pl) {
        pos = e - pf;
      } else {
        auto it = std::lower_bound(pb.begin(), pb.end(), e);
        if (it == pb.end() || *it != e) return *msg = "sparse symbolic: boundary not inherited by the parent", false;
        pos = s.nown[par] / 3 + (int32_t)(it - pb.begin());
      }
      s.ea_map.push_back(pos);
    }
  }
  // ---- assembly blocks: (row point q, column point p) with epos(q) ≥ epos(p), in the front of p's node
  s.ablk.clear();
  s.acoff.assign(1, 0);
  s.acon.clear();
  std::vector<int32_t> nb;
  for (int i = 0; i < NN; ++i) {
    const std::vector<int32_t>& bi = bnd[i];
    for (int32_t p : nd.nodes[i]) {
      nb.clear();
      for_neighbors(p, [&](int32_t q) {
        if (s.epos[q] >= s.epos[p]) nb.push_back(q);
      });
      std::sort(nb.begin(), nb.end(), [&](int32_t x, int32_t y) { return s.epos[x] < s.epos[y]; });
      nb.erase(std::unique(nb.begin(), nb.end()), nb.end());
      const int32_t cpos = s.epos[p] - s.own_first[i];
      for (int32_t q : nb) {
        const int32_t e = s.epos[q];
        int32_t rpos;
        if (e < last[i]) {
          rpos = e - s.own_first[i];
        } else {
          auto it = std::lower_bound(bi.begin(), bi.end(), e);
          if (it == bi.end() || *it != e) return *msg = "sparse symbolic: neighbour missing from the front", false;
          rpos = s.nown[i] / 3 + (int32_t)(it - bi.begin());
        }
        s.ablk.push_back(i);
        s.ablk.push_back(rpos);
        s.ablk.push_back(cpos);
        // shared bodies: (row side, column side)
        for (int sq = 0; sq < 2; ++sq) {
          const int32_t bq = sq == 0 ? s.pa[q] : s.pb[q];
          if (bq < 0) continue;
          for (int spp = 0; spp < 2; ++spp) {
            const int32_t bp = spp == 0 ? s.pa[p] : s.pb[p];
            if (bp != bq) continue;
            s.acon.push_back(2 * q + sq);
            s.acon.push_back(2 * p + spp);
          }
        }
        s.acoff.push_back((int32_t)(s.acon.size() / 2));
      }
    }
  }
  // ---- schedule by height: small fronts in shared memory, large ones by panels
  int H = 0;
  for (int i = 0; i < NN; ++i) H = std::max(H, s.height[i] + 1);
  std::vector<std::vector<int32_t>> byh(H);
  for (int i = 0; i < NN; ++i) byh[s.height[i]].push_back(i);
  s.levels.assign(H, SparsePlan::Level());
  s.lev_nodes.clear();
  s.tasks.clear();
  s.loff.assign(NN, 0);
  s.linv_doubles = 0;
  const int64_t small_cap = MF_SMALL;
  for (int h = 0; h < H; ++h) {
    SparsePlan::Level& L = s.levels[h];
    const std::vector<int32_t>& nodes = byh[h];
    L.nodes = (int64_t)s.lev_nodes.size();
    L.n_nodes = (int64_t)nodes.size();
    s.lev_nodes.insert(s.lev_nodes.end(), nodes.begin(), nodes.end());
    std::vector<int32_t> small, big;
    for (int32_t i : nodes) {
      L.max_f = std::max(L.max_f, s.fdim[i]);
      (s.fdim[i] <= small_cap ? small : big).push_back(i);
    }
    L.small = (int64_t)s.lev_nodes.size();
    L.n_small = (int64_t)small.size();
    s.lev_nodes.insert(s.lev_nodes.end(), small.begin(), small.end());
    L.big = (int64_t)s.lev_nodes.size();
    L.n_big = (int64_t)big.size();
    s.lev_nodes.insert(s.lev_nodes.end(), big.begin(), big.end());
    for (int32_t i : big) {
      s.loff[i] = s.linv_doubles;
      s.linv_doubles += (int64_t)((s.nown[i] + MF_NB - 1) / MF_NB) * MF_NB * MF_NB;
    }
    for (int32_t i : small) L.max_f_small = std::max(L.max_f_small, s.fdim[i]);
    int maxc = 0, maxpan = 0;
    for (int32_t i : big) {
      maxc = std::max(maxc, (int)kids[i].size());
      maxpan = std::max(maxpan, (s.nown[i] + MF_NB - 1) / MF_NB);
    }
    L.max_children = maxc;
    L.ea.assign(maxc, 0);
    L.n_ea.assign(maxc, 0);
    for (int sl = 0; sl < maxc; ++sl) {
      L.ea[sl] = (int64_t)s.tasks.size();
      for (int32_t i : big) {
        if ((int)kids[i].size() <= sl) continue;
        const int c = kids[i][sl];
        const int mc = s.fdim[c] - s.nown[c];
        for (int j = 0; j < mc; ++j) {
          s.tasks.push_back(i);
          s.tasks.push_back(j);
        }
      }
      L.n_ea[sl] = ((int64_t)s.tasks.size() - L.ea[sl]) / 2;
    }
    L.panels.assign(maxpan, SparsePlan::Panel());
    for (int pi = 0; pi < maxpan; ++pi) {
      SparsePlan::Panel& Pn = L.panels[pi];
      const int k0 = pi * MF_NB;
      std::vector<int32_t> act;
      for (int32_t i : big)
        if (s.nown[i] > k0) act.push_back(i);
      Pn.potrf = (int64_t)s.tasks.size();
      for (int32_t i : act) s.tasks.push_back(i);
      Pn.n_potrf = (int64_t)act.size();
      Pn.trsm = (int64_t)s.tasks.size();
      for (size_t sl = 0; sl < act.size(); ++sl) {
        const int i = act[sl];
        const int t0 = k0 + std::min(MF_NB, s.nown[i] - k0);
        for (int r0 = t0; r0 < s.fdim[i]; r0 += MF_NB) {
          s.tasks.push_back(i);
          s.tasks.push_back(r0);
          s.tasks.push_back((int32_t)sl);
        }
      }
      Pn.n_trsm = ((int64_t)s.tasks.size() - Pn.trsm) / 3;
      // Trailing updates by pairs of panels (look-ahead by one): when panels pi (even) and pi+1 are both full, the
      // even step updates only the next panel's column block (rank 64) and the odd step the rest of the trailing
      // matrix with both panels at once (rank 128: each trailing tile is read and written once per pair);
      // otherwise each panel updates its whole trailing matrix. Task = (node, r0, c0, first column, columns).
      Pn.syrk = (int64_t)s.tasks.size();
      auto tiles = [&](int32_t i, int t0, int cmax, int kbeg, int kcnt) {
        for (int r0 = t0; r0 < s.fdim[i]; r0 += MF_NB)
          for (int c0 = t0; c0 <= r0 && c0 < cmax; c0 += MF_NB)
            for (int32_t v : {i, (int32_t)r0, (int32_t)c0, (int32_t)kbeg, (int32_t)kcnt}) s.tasks.push_back(v);
      };
      for (int32_t i : act) {
        const int kb = std::min(MF_NB, s.nown[i] - k0);
        const bool even = pi % 2 == 0;
        const bool paired = even ? s.nown[i] >= k0 + 2 * MF_NB : s.nown[i] >= k0 + MF_NB;
        if (even && paired)
          tiles(i, k0 + MF_NB, k0 + 2 * MF_NB, k0, MF_NB);           // the next panel's block column
        else if (!even && paired)
          tiles(i, k0 + MF_NB, INT32_MAX, k0 - MF_NB, 2 * MF_NB);    // the rest, both panels
        else
          tiles(i, k0 + kb, INT32_MAX, k0, kb);
      }
      Pn.n_syrk = ((int64_t)s.tasks.size() - Pn.syrk) / 5;
    }
    // triangular-solve tasks of the big fronts, per group of MF_SG chunks
    const int ngrp = (maxpan + MF_SG - 1) / MF_SG;
    L.fwd.assign(ngrp, 0);
    L.n_fwd.assign(ngrp, 0);
    L.bwd.assign(ngrp, 0);
    L.n_bwd.assign(ngrp, 0);
    for (int c = 0; c < ngrp; ++c) {
      const int k0 = c * MF_SG * MF_NB;
      L.fwd[c] = (int64_t)s.tasks.size();
      for (int32_t i : big) {
        if (s.nown[i] <= k0) continue;
        int wr = 1;
        for (int r0 = k0 + std::min(MF_SG * MF_NB, s.nown[i] - k0); r0 < s.fdim[i]; r0 += MF_NB, wr = 0) {
          s.tasks.push_back(i);
          s.tasks.push_back(r0);
          s.tasks.push_back(wr);
        }
        if (wr) {
          s.tasks.push_back(i);
          s.tasks.push_back(-1);
          s.tasks.push_back(1);
        }
      }
      L.n_fwd[c] = ((int64_t)s.tasks.size() - L.fwd[c]) / 3;
      L.bwd[c] = (int64_t)s.tasks.size();
      for (int32_t i : big) {
        if (s.nown[i] <= k0) continue;
        int wr = 1;
        for (int t0 = 0; t0 < k0; t0 += MF_NB, wr = 0) {
          s.tasks.push_back(i);
          s.tasks.push_back(t0);
          s.tasks.push_back(wr);
        }
        if (wr) {
          s.tasks.push_back(i);
          s.tasks.push_back(-1);
          s.tasks.push_back(1);
        }
      }
      L.n_bwd[c] = ((int64_t)s.tasks.size() - L.bwd[c]) / 3;
    }
    L.bwdb = (int64_t)s.tasks.size();
    for (int32_t i : big)
      if (s.fdim[i] > s.nown[i])
        for (int t0 = 0; t0 < s.nown[i]; t0 += MF_NB) {
          s.tasks.push_back(i);
          s.tasks.push_back(t0);
        }
    L.n_bwdb = ((int64_t)s.tasks.size() - L.bwdb) / 2;
  }
#ifndef MF_ZERO_FULL
  s.zero = (int64_t)s.tasks.size();  // lower-triangle zeroing: MF_ZC columns per task
  for (int i = 0; i < s.nnode; ++i)
    for (int c0 = 0; c0 < s.fdim[i]; c0 += s.fdim[i] <= MF_SMALL ? s.fdim[i] : MF_ZC) {
      s.tasks.push_back(i);
      s.tasks.push_back(c0);
    }
  s.n_zero = ((int64_t)s.tasks.size() - s.zero) / 2;
#endif
  if (s.tasks.size() > (size_t)INT32_MAX || s.ablk.size() / 3 > (size_t)INT32_MAX)
    return *msg = "sparse symbolic: too many tasks", false;
  return true;
}

// ΔR_H of the five-row hinge: I + [v]× + [v]×²/(1 + a_y), v = a × e_y, turning the unit axis a onto e_y
// (a = −e_y, where the formula is singular: diag(1, −1, −1)).
static void hinge_frame(const double* a, double R[3][3]) {
  if (a[1] <= -1.0 + 1e-12) {
    const double D[3][3] = {{1, 0, 0}, {0, -1, 0}, {0, 0, -1}};
    std::memcpy(R, D, sizeof(D));
    return;
  }
  const double v[3] = {-a[2], 0.0, a[0]};  // a × e_y
  const double V[3][3] = {{0, -v[2], v[1]}, {v[2], 0, -v[0]}, {-v[1], v[0], 0}};
  for (int r = 0; r < 3; ++r)
    for (int c = 0; c < 3; ++c) {
      double vv = 0;
      for (int m = 0; m < 3; ++m) vv += V[r][m] * V[m][c];
      R[r][c] = (r == c ? 1.0 : 0.0) + V[r][c] + vv / (1.0 + a[1]);
    }
}

bool sparse_build(const mabd_bodies* B, const mabd_joints* J, Plan* p, std::vector<int64_t>* pos_of_body,
                  std::string* msg, bool symbolic) {
  const int64_t K = J->n_joints, n = B->n;
  SparsePlan& s = p->sparse;
  s = SparsePlan();
  int64_t P = 0;
  for (int64_t k = 0; k < K; ++k) P += J->npts[k];
  if (2 * P > (int64_t)INT32_MAX) return *msg = "too many joint points", false;
  s.np = P;
  s.pa.resize(P);
  s.pb.resize(P);
  s.py.resize(6 * P);
  std::vector<int32_t> cnt(n + 1, 0);
  int64_t pt = 0;
  for (int64_t k = 0; k < K; ++k)
    for (int q = 0; q < J->npts[k]; ++q, ++pt) {
      s.pa[pt] = J->body_a[k];
      s.pb[pt] = J->body_b[k];
      for (int e = 0; e < 3; ++e) {
        s.py[6 * pt + e] = J->ybar_a[3 * pt + e];
        s.py[6 * pt + 3 + e] = J->ybar_b[3 * pt + e];
      }
      cnt[J->body_a[k] + 1]++;
      if (J->body_b[k] >= 0) cnt[J->body_b[k] + 1]++;
    }
  s.inc_off.assign(n + 1, 0);
  for (int64_t i = 0; i < n; ++i) s.inc_off[i + 1] = s.inc_off[i] + cnt[i + 1];
  s.inc.assign(s.inc_off[n], 0);
  std::vector<int32_t> fill(n, 0);
  for (int64_t q = 0; q < P; ++q) {
    const int64_t a = s.pa[q], b = s.pb[q];
    s.inc[s.inc_off[a] + fill[a]++] = (int32_t)(2 * q);
    if (b >= 0) s.inc[s.inc_off[b] + fill[b]++] = (int32_t)(2 * q + 1);
  }
  // five-row hinges: the second point of each is projected (rows w0, w1 from ΔR_H of the axis in body a's frame);
  // a limited one also gets an extra point, the limit row (R14), appended after the joints' points
  s.pslot.clear();
  s.pdr.clear();
  s.pplist.clear();
  s.plim.clear();
  s.pgc.clear();
  if (J->kind) {
    s.pslot.assign(P, -1);
    int64_t p0 = 0;
    std::vector<int64_t> lim_joint;
    bool any_general = false;
    // a general slot (universal / prismatic rows, R17) at point `pt` with rows {type, d, e}
    auto general = [&](int64_t pt, std::initializer_list<std::array<double, 7>> rows) {
      s.pslot[pt] = (int32_t)s.pplist.size();
      s.pplist.push_back((int32_t)pt);
      for (int e = 0; e < 6; ++e) s.pdr.push_back(0.0);
      for (int e = 0; e < LIM_DOUBLES; ++e) s.plim.push_back(0.0);
      std::vector<double> rec(PGC_DOUBLES, 0.0);
      int i = 0;
      for (const auto& r : rows) {
        for (int e = 0; e < 7; ++e) rec[PGC_ROW * i + e] = r[e];
        ++i;
      }
      s.pgc.insert(s.pgc.end(), rec.begin(), rec.end());
      any_general = true;
    };
    auto sub = [](const double* x, const double* y, double* o) {
      for (int e = 0; e < 3; ++e) o[e] = x[e] - y[e];
    };
    for (int64_t k = 0; k < K; ++k) {
      if (J->kind[k] == 2 || J->kind[k] == 3) {
        const double *ya = J->ybar_a + 3 * p0, *yb = J->ybar_b + 3 * p0;
        double ax[3], e1[3];
        sub(ya + 3, ya, ax);
        sub(yb + 3, yb, e1);
        const double nrm = std::sqrt(ax[0] * ax[0] + ax[1] * ax[1] + ax[2] * ax[2]);
        if (!(nrm > 0) || !(e1[0] * e1[0] + e1[1] * e1[1] + e1[2] * e1[2] > 0))
          return *msg = "universal / prismatic joint with coincident axis points", false;
        for (double& v : ax) v /= nrm;
        if (J->kind[k] == 2) {  // the centre stays a ball; the second point: (A_a â₁)·(A_b e₂)
          general(p0 + 1, {{2.0, ax[0], ax[1], ax[2], e1[0], e1[1], e1[2]}});
        } else {                // prismatic: x̂, ẑ point rows; parallel axes; no twist
          double dR[3][3], ua[3], u[3];
          hinge_frame(ax, dR);
          sub(ya + 6, ya, ua);
          sub(yb + 6, yb, u);
          const double nu = std::sqrt(ua[0] * ua[0] + ua[1] * ua[1] + ua[2] * ua[2]);
          if (!(nu > 0)) return *msg = "prismatic joint with a coincident third point", false;
          for (double& v : ua) v /= nu;
          const double n[3] = {ax[1] * ua[2] - ax[2] * ua[1], ax[2] * ua[0] - ax[0] * ua[2],
                               ax[0] * ua[1] - ax[1] * ua[0]};
          general(p0, {{1.0, dR[0][0], dR[0][1], dR[0][2], 0, 0, 0}, {1.0, dR[2][0], dR[2][1], dR[2][2], 0, 0, 0}});
          general(p0 + 1, {{2.0, dR[0][0], dR[0][1], dR[0][2], e1[0], e1[1], e1[2]},
                           {2.0, dR[2][0], dR[2][1], dR[2][2], e1[0], e1[1], e1[2]}});
          general(p0 + 2, {{2.0, n[0], n[1], n[2], u[0], u[1], u[2]}});
        }
      }
      if (J->kind[k] == 1) {
        const double* y0 = J->ybar_a + 3 * p0;
        double ax[3] = {y0[3] - y0[0], y0[4] - y0[1], y0[5] - y0[2]};
        const double nrm = std::sqrt(ax[0] * ax[0] + ax[1] * ax[1] + ax[2] * ax[2]);
        if (!(nrm > 0)) return *msg = "five-row hinge with coincident axis points", false;
        for (double& v : ax) v /= nrm;
        double dR[3][3];
        hinge_frame(ax, dR);
        s.pslot[p0 + 1] = (int32_t)s.pplist.size();
        s.pplist.push_back((int32_t)(p0 + 1));
        for (int i : {0, 2})
          for (int c = 0; c < 3; ++c) s.pdr.push_back(dR[i][c]);
        for (int e = 0; e < LIM_DOUBLES; ++e) s.plim.push_back(0.0);
        s.pgc.insert(s.pgc.end(), PGC_DOUBLES, 0.0);
        const double* L = J->limits ? J->limits + 8 * k : nullptr;
        if (L && (std::isfinite(L[0]) || std::isfinite(L[1]))) {
          if (!(L[0] < L[1])) return *msg = "joint limits need lo < hi", false;
          std::vector<double> rec(LIM_DOUBLES, 0.0);
          rec[0] = std::isfinite(L[0]) ? L[0] : -1e300;
          rec[1] = std::isfinite(L[1]) ? L[1] : 1e300;
          for (int e = 0; e < 6; ++e) rec[2 + e] = L[2 + e];
          for (int e = 0; e < 3; ++e) {
            rec[8 + e] = y0[e];
            rec[11 + e] = ax[e];
          }
          rec[14] = nrm;
          // the limit point: body a's point is written per iteration; body b's is ȳ_b0 + ρ u_b
          const double* yb0 = J->ybar_b + 3 * p0;
          s.pa.push_back(J->body_a[k]);
          s.pb.push_back(J->body_b[k]);
          for (int e = 0; e < 3; ++e) s.py.push_back(y0[e] + nrm * L[2 + e]);
          for (int e = 0; e < 3; ++e) s.py.push_back(yb0[e] + nrm * L[5 + e]);
          s.pslot.push_back((int32_t)s.pplist.size());
          s.pplist.push_back((int32_t)(s.pa.size() - 1));
          for (int e = 0; e < 6; ++e) s.pdr.push_back(0.0);
          s.plim.insert(s.plim.end(), rec.begin(), rec.end());
          s.pgc.insert(s.pgc.end(), PGC_DOUBLES, 0.0);
          lim_joint.push_back(k);
        }
      }
      p0 += J->npts[k];
    }
    if (s.pplist.empty()) s.pslot.clear();
    if (!any_general) s.pgc.clear();
    if (!lim_joint.empty()) {  // the incidence with the limit points
      const int64_t P2 = (int64_t)s.pa.size();
      std::vector<int32_t> c2(n + 1, 0);
      for (int64_t q = 0; q < P2; ++q) {
        c2[s.pa[q] + 1]++;
        if (s.pb[q] >= 0) c2[s.pb[q] + 1]++;
      }
      s.inc_off.assign(n + 1, 0);
      for (int64_t i = 0; i < n; ++i) s.inc_off[i + 1] = s.inc_off[i] + c2[i + 1];
      s.inc.assign(s.inc_off[n], 0);
      std::vector<int32_t> f2(n, 0);
      for (int64_t q = 0; q < P2; ++q) {
        const int64_t a = s.pa[q], b = s.pb[q];
        s.inc[s.inc_off[a] + f2[a]++] = (int32_t)(2 * q);
        if (b >= 0) s.inc[s.inc_off[b] + f2[b]++] = (int32_t)(2 * q + 1);
      }
      s.np = P2;
    }
  }
  pos_of_body->resize(n);
  for (int64_t i = 0; i < n; ++i) (*pos_of_body)[i] = i;  // caller order
  p->ld = n;
  p->n = n;
  p->n_dual_rows = 3 * P;
  if (!symbolic) return true;  // line Gauss-Seidel (gs_build) needs the points and the incidence only
  if (!mf_symbolic(B, p, msg)) return false;
  s.refine = MF_REFINE;
  if (const char* ev = getenv("MABD_SPARSE_REFINE")) s.refine = std::max(0, std::min(8, atoi(ev)));  // developer knob
  s.refine_tol = MF_REFINE_TOL;
  s.syrk_dfma = getenv("MABD_SPARSE_SYRK_DFMA") != nullptr;  // developer knob: the DFMA trailing update
  if (const char* ev = getenv("MABD_SPARSE_REFINE_TOL")) s.refine_tol = atof(ev);                   // developer knob
  int64_t launches = 4 + (P ? 2 : 0) + (s.n_zero ? 1 : 0);
  for (const auto& L : s.levels) {
    int64_t per = (L.n_small ? 1 : 0);
    for (int64_t c : L.n_ea) per += c ? 1 : 0;
    for (const auto& Pn : L.panels) per += (Pn.n_potrf ? 1 : 0) + (Pn.n_trsm ? 1 : 0) + (Pn.n_syrk ? 1 : 0);
    int64_t sol = 2 * (L.n_small ? 1 : 0);
    if (L.n_big) sol += 2 + (L.n_bwdb ? 1 : 0) + (int64_t)L.fwd.size() + (int64_t)L.bwd.size();
    launches += per + sol * (1 + s.refine);
  }
  launches += 4 * s.refine;
  p->launches_per_step = (int32_t)std::min<int64_t>(launches, INT32_MAX);
  return true;
}

// ============================================================================ host side: line Gauss-Seidel plan
// Chain cover (R10): greedy paths in the body graph, each point (joint row block) on exactly one chain.
// A chain grows from its last point through that point's other body to an unused point of that body whose bodies are
// all new to the chain, taking the straightest continuation within ~26° of the direction of travel (the joint
// positions at create), so a grid net is covered by its rows and columns, as the paper's "multi-directional"
// relaxation along pre-defined chains.
// Chains are capped at GS_MAX_CHAIN points (parallelism); chains sharing a body get different colours (greedy).
constexpr int GS_MAX_CHAIN = 64;
constexpr double GS_MIN_COS = 0.9;

bool gs_build(const mabd_bodies* B, Plan* p, int32_t sweeps, double tol, std::string* msg) {
  SparsePlan& s = p->sparse;
  if (!s.pplist.empty()) return *msg = "five-row hinges need the direct sparse solver", false;
  const int64_t n = p->n, np = s.np;
  s.gs_sweeps = sweeps > 0 ? sweeps : 200;
  s.gs_tol = tol > 0 ? tol : 1e-12;
  if (s.gs_sweeps > 100000) return *msg = "gs_sweeps > 100000", false;
  // joint positions at create (side a)
  std::vector<double> xp(3 * np);
  for (int64_t q = 0; q < np; ++q) {
    const double* qa = B->q0 + 12 * (int64_t)s.pa[q];
    const double* y = s.py.data() + 6 * q;
    for (int r = 0; r < 3; ++r) xp[3 * q + r] = qa[r] * y[0] + qa[3 + r] * y[1] + qa[6 + r] * y[2] + qa[9 + r];
  }
  std::vector<char> used(np, 0);
  std::vector<int32_t> mark(n, -1);  // chain id that owns a body (body-path property)
  std::vector<int32_t> pts, off{0};
  auto other = [&](int32_t q, int32_t b) { return s.pa[q] == b ? s.pb[q] : s.pa[q]; };
  auto twin = [&](int64_t q, int64_t r) {  // two points of one multi-point joint (the same two bodies)
    return r >= 0 && r < np && s.pa[q] == s.pa[r] && s.pb[q] == s.pb[r];
  };
  for (int64_t q0 = 0; q0 < np; ++q0) {
    if (used[q0]) continue;
    const int32_t cid = (int32_t)off.size() - 1;
    std::vector<int32_t> ch{(int32_t)q0};
    used[q0] = 1;
    mark[s.pa[q0]] = cid;
    if (s.pb[q0] >= 0) mark[s.pb[q0]] = cid;
    // the points of a linear hinge share both bodies and are strongly coupled: they form a chain of their own
    // (relaxing them in different colours stalls the iteration); such a chain cannot continue through either body
    bool hinge = false;
    for (int64_t r = q0 + 1; r < np && twin(q0, r) && !used[r]; ++r) {
      ch.push_back((int32_t)r);
      used[r] = 1;
      hinge = true;
    }
    for (int dir = 0; dir < 2 && !hinge && (int)ch.size() < GS_MAX_CHAIN; ++dir) {
      // grow from the end (dir 0: through body b of the first point, then onwards; dir 1: the other way)
      int32_t last = dir == 0 ? ch.back() : ch.front();
      int32_t via = dir == 0 ? s.pb[q0] : s.pa[q0];
      if (ch.size() > 1 && dir == 0) via = -1;  // (only the seed point chooses the direction)
      while (via >= 0 && (int)ch.size() < GS_MAX_CHAIN) {
        int32_t best = -1;
        double best_score = GS_MIN_COS;  // continue only within ~26° of straight ahead
        const double* xl = xp.data() + 3 * last;
        double dprev[3] = {0, 0, 0};
        {  // direction of travel: previous point → last point (or body → last point at the start)
          const int32_t prev = ch.size() > 1 ? (dir == 0 ? ch[ch.size() - 2] : ch[1]) : -1;
          for (int r = 0; r < 3; ++r)
            dprev[r] = prev >= 0 ? xl[r] - xp[3 * prev + r] : B->q0[12 * (int64_t)via + 9 + r] - xl[r];
        }
        for (int i = s.inc_off[via]; i < s.inc_off[via + 1]; ++i) {
          const int32_t q = s.inc[i] >> 1;
          if (used[q] || twin(q, q + 1) || twin(q, q - 1)) continue;
          const int32_t o = other(q, via);
          if (o >= 0 && mark[o] == cid) continue;  // would revisit a body of this chain
          double dq[3], nd = 0, nq = 0, dot = 0;
          for (int r = 0; r < 3; ++r) {
            dq[r] = xp[3 * q + r] - xl[r];
            nd += dprev[r] * dprev[r];
            nq += dq[r] * dq[r];
            dot += dprev[r] * dq[r];
          }
          const double score = (nd > 0 && nq > 0) ? dot / std::sqrt(nd * nq) : 0.0;
          if (score > best_score) {
            best_score = score;
            best = q;
          }
        }
        if (best < 0) break;
        used[best] = 1;
        const int32_t o = other(best, via);
        if (o >= 0) mark[o] = cid;
        if (dir == 0)
          ch.push_back(best);
        else
          ch.insert(ch.begin(), best);
        last = best;
        via = o;
      }
    }
    pts.insert(pts.end(), ch.begin(), ch.end());
    off.push_back((int32_t)pts.size());
  }
  const int32_t nch = (int32_t)off.size() - 1;
  // colouring: chains that share a body conflict
  std::vector<std::vector<int32_t>> body_chains(n);
  for (int32_t c = 0; c < nch; ++c)
    for (int32_t k = off[c]; k < off[c + 1]; ++k) {
      const int32_t q = pts[k];
      for (int32_t b : {s.pa[q], s.pb[q]})
        if (b >= 0 && (body_chains[b].empty() || body_chains[b].back() != c)) body_chains[b].push_back(c);
    }
  std::vector<int32_t> color(nch, -1), order(nch);
  for (int32_t c = 0; c < nch; ++c) order[c] = c;
  std::stable_sort(order.begin(), order.end(),
                   [&](int32_t x, int32_t y) { return off[x + 1] - off[x] > off[y + 1] - off[y]; });
  int32_t ncolor = 0;
  std::vector<int32_t> seen;
  for (int32_t c : order) {
    seen.clear();
    for (int32_t k = off[c]; k < off[c + 1]; ++k) {
      const int32_t q = pts[k];
      for (int32_t b : {s.pa[q], s.pb[q]})
        if (b >= 0)
          for (int32_t d : body_chains[b])
            if (d != c && color[d] >= 0) seen.push_back(color[d]);
    }
    std::sort(seen.begin(), seen.end());
    int32_t col = 0;
    for (int32_t v : seen) {
      if (v == col) ++col;
      else if (v > col) break;
    }
    color[c] = col;
    ncolor = std::max(ncolor, col + 1);
  }
  // chains sorted by colour (stable), points in chain order
  std::vector<int32_t> by_color(nch);
  for (int32_t c = 0; c < nch; ++c) by_color[c] = c;
  std::stable_sort(by_color.begin(), by_color.end(), [&](int32_t x, int32_t y) { return color[x] < color[y]; });
  s.gs_chain_pts.clear();
  s.gs_chain_off.assign(1, 0);
  s.gs_color_off.assign(ncolor + 1, 0);
  for (int32_t c : by_color) {
    s.gs_chain_pts.insert(s.gs_chain_pts.end(), pts.begin() + off[c], pts.begin() + off[c + 1]);
    s.gs_chain_off.push_back((int32_t)s.gs_chain_pts.size());
    s.gs_color_off[color[c] + 1]++;
  }
  for (int32_t c = 0; c < ncolor; ++c) s.gs_color_off[c + 1] += s.gs_color_off[c];
  s.gs_ncolor = ncolor;
  p->launches_per_step = 5 + (np ? 4 + s.gs_sweeps * ncolor : 0);
  return true;
}

// ============================================================================ host side: layout and upload
void sparse_layout(Plan* p, const std::function<size_t(size_t)>& take) {
  SparsePlan& s = p->sparse;
  const int64_t np = std::max<int64_t>(1, s.np), n = p->n;
  auto nz = [](size_t x) { return std::max<size_t>(x, 1); };
  s.o_pa = take(sizeof(int32_t) * np);
  s.o_pb = take(sizeof(int32_t) * np);
  s.o_py = take(sizeof(double) * 6 * np);
  s.o_incoff = take(sizeof(int32_t) * (n + 1));
  s.o_inc = take(sizeof(int32_t) * nz(s.inc.size()));
  s.o_vec = take(sizeof(double) * 15 * np);  // rhs, λ, res, δλ, y: [3][np] each
  s.o_vv = take(sizeof(double) * 12 * n);
  s.o_dqt = take(sizeof(double) * 12 * n);
  s.o_iters = take(sizeof(int32_t) * 4 + sizeof(unsigned long long) * 3);  // iters[4], the gate's rmax[3]
  const size_t NN = nz(s.nnode);
  s.o_F = take(sizeof(double) * nz(s.front_doubles));
  s.o_foff = take(sizeof(int64_t) * NN);
  s.o_fdim = take(sizeof(int32_t) * NN);
  s.o_nown = take(sizeof(int32_t) * NN);
  s.o_ownf = take(sizeof(int32_t) * NN);
  s.o_choff = take(sizeof(int32_t) * (NN + 1));
  s.o_ch = take(sizeof(int32_t) * nz(s.ch.size()));
  s.o_eaoff = take(sizeof(int32_t) * NN);
  s.o_eamap = take(sizeof(int32_t) * nz(s.ea_map.size()));
  s.o_bndoff = take(sizeof(int32_t) * NN);
  s.o_bnd = take(sizeof(int32_t) * nz(s.bnd.size()));
  s.o_ipos = take(sizeof(int32_t) * np);
  s.o_ablk = take(sizeof(int32_t) * nz(s.ablk.size()));
  s.o_acoff = take(sizeof(int32_t) * nz(s.acoff.size()));
  s.o_acon = take(sizeof(int32_t) * nz(s.acon.size()));
  s.o_linv = take(sizeof(double) * nz(s.linv_doubles));
  s.o_loff = take(sizeof(int64_t) * NN);
  s.o_w = take(sizeof(double) * nz(s.w_doubles));
  s.o_woff = take(sizeof(int64_t) * NN);
  s.o_lev = take(sizeof(int32_t) * nz(s.lev_nodes.size()));
  s.o_tasks = take(sizeof(int32_t) * nz(s.tasks.size()));
  s.o_pslot = take(sizeof(int32_t) * nz(s.pslot.size()));
  s.o_pdr = take(sizeof(double) * nz(s.pdr.size()));
  s.o_pw = take(sizeof(double) * nz(s.pdr.size()));
  s.o_pnr = take(sizeof(int32_t) * nz(s.pplist.size()));
  s.o_plim = take(sizeof(double) * nz(s.plim.size()));
  s.o_pplist = take(sizeof(int32_t) * nz(s.pplist.size()));
  s.o_pgc = take(sizeof(double) * nz(s.pgc.size()));
  s.o_pg = take(sizeof(double) * nz(s.pgc.empty() ? 0 : PG_DOUBLES * s.pplist.size()));
  s.o_gs_pts = take(sizeof(int32_t) * nz(s.gs_chain_pts.size()));
  s.o_gs_off = take(sizeof(int32_t) * nz(s.gs_chain_off.size()));
  s.o_gs_col = take(sizeof(int32_t) * nz(s.gs_color_off.size()));
  s.o_gs_fac = s.gs_ncolor ? take(sizeof(double) * 24 * np) : 0;
  s.o_gs_res = take(sizeof(unsigned long long) * (1 + 2 * std::max(0, s.gs_sweeps)));
}

template <class T>
static cudaError_t upv(char* ws, size_t off, const std::vector<T>& v, cudaStream_t st) {
  if (v.empty()) return cudaSuccess;
  return cudaMemcpyAsync(ws + off, v.data(), sizeof(T) * v.size(), cudaMemcpyHostToDevice, st);
}

cudaError_t sparse_upload(const Plan& p, char* ws, cudaStream_t st, DevPtrs* d) {
  const SparsePlan& s = p.sparse;
  SparseArgs& A = d->sparse;
  const int64_t np = std::max<int64_t>(1, s.np);
  A.b = d->b;
  A.hinv_tab = p.mscale.empty() ? d->hinv : nullptr;
  A.n = p.n;
  A.np = s.np;
  A.pa = (const int32_t*)(ws + s.o_pa);
  A.pb = (const int32_t*)(ws + s.o_pb);
  A.py = (const double*)(ws + s.o_py);
  A.inc_off = (const int32_t*)(ws + s.o_incoff);
  A.inc = (const int32_t*)(ws + s.o_inc);
  double* v = (double*)(ws + s.o_vec);
  A.rhs = v;
  A.lam = v + 3 * np;
  A.res = v + 6 * np;
  A.dl = v + 9 * np;
  A.yy = v + 12 * np;
  A.vv = (double*)(ws + s.o_vv);
  A.dqt = (double*)(ws + s.o_dqt);
  A.iters = (int32_t*)(ws + s.o_iters);
  A.rmax = (unsigned long long*)(ws + s.o_iters + sizeof(int32_t) * 4);
  A.gate = nullptr;
  A.refine_tol = s.refine_tol;
  MfArgs& m = A.mf;
  m.F = (double*)(ws + s.o_F);
  m.foff = (const int64_t*)(ws + s.o_foff);
  m.fdim = (const int32_t*)(ws + s.o_fdim);
  m.nown = (const int32_t*)(ws + s.o_nown);
  m.own_first = (const int32_t*)(ws + s.o_ownf);
  m.ch_off = (const int32_t*)(ws + s.o_choff);
  m.ch = (const int32_t*)(ws + s.o_ch);
  m.ea_off = (const int32_t*)(ws + s.o_eaoff);
  m.ea_map = (const int32_t*)(ws + s.o_eamap);
  m.bnd_off = (const int32_t*)(ws + s.o_bndoff);
  m.bnd = (const int32_t*)(ws + s.o_bnd);
  m.ipos = (const int32_t*)(ws + s.o_ipos);
  m.ablk = (const int32_t*)(ws + s.o_ablk);
  m.acoff = (const int32_t*)(ws + s.o_acoff);
  m.acon = (const int32_t*)(ws + s.o_acon);
  m.nblk = (int64_t)s.ablk.size() / 3;
  m.linv = (double*)(ws + s.o_linv);
  m.loff = (const int64_t*)(ws + s.o_loff);
  m.wvec = (double*)(ws + s.o_w);
  m.woff = (const int64_t*)(ws + s.o_woff);
  A.nproj = (int64_t)s.pplist.size();
  A.pslot = A.nproj ? (const int32_t*)(ws + s.o_pslot) : nullptr;
  A.pdr = (const double*)(ws + s.o_pdr);
  A.pw = (double*)(ws + s.o_pw);
  A.pplist = (const int32_t*)(ws + s.o_pplist);
  A.pnr = (int32_t*)(ws + s.o_pnr);
  A.plim = (const double*)(ws + s.o_plim);
  A.pgc = s.pgc.empty() ? nullptr : (const double*)(ws + s.o_pgc);
  A.pg = (double*)(ws + s.o_pg);
  A.gs.chain_pts = (const int32_t*)(ws + s.o_gs_pts);
  A.gs.chain_off = (const int32_t*)(ws + s.o_gs_off);
  A.gs.color_off = (const int32_t*)(ws + s.o_gs_col);
  A.gs.fac = s.gs_ncolor ? (double*)(ws + s.o_gs_fac) : nullptr;
  A.gs.resmax = (unsigned long long*)(ws + s.o_gs_res);
  A.gs.ncolor = s.gs_ncolor;
  A.gs.max_sweeps = s.gs_sweeps;
  A.gs.tol = s.gs_tol;
  d->sparse_lev = (const int32_t*)(ws + s.o_lev);
  d->sparse_tasks = (const int32_t*)(ws + s.o_tasks);
  cudaError_t e;
  if ((e = upv(ws, s.o_pa, s.pa, st))) return e;
  if ((e = upv(ws, s.o_pb, s.pb, st))) return e;
  if ((e = upv(ws, s.o_py, s.py, st))) return e;
  if ((e = upv(ws, s.o_incoff, s.inc_off, st))) return e;
  if ((e = upv(ws, s.o_inc, s.inc, st))) return e;
  if ((e = upv(ws, s.o_foff, s.foff, st))) return e;
  if ((e = upv(ws, s.o_fdim, s.fdim, st))) return e;
  if ((e = upv(ws, s.o_nown, s.nown, st))) return e;
  if ((e = upv(ws, s.o_ownf, s.own_first, st))) return e;
  if ((e = upv(ws, s.o_choff, s.ch_off, st))) return e;
  if ((e = upv(ws, s.o_ch, s.ch, st))) return e;
  if ((e = upv(ws, s.o_eaoff, s.ea_off, st))) return e;
  if ((e = upv(ws, s.o_eamap, s.ea_map, st))) return e;
  if ((e = upv(ws, s.o_bndoff, s.bnd_off, st))) return e;
  if ((e = upv(ws, s.o_bnd, s.bnd, st))) return e;
  if ((e = upv(ws, s.o_ipos, s.ipos, st))) return e;
  if ((e = upv(ws, s.o_ablk, s.ablk, st))) return e;
  if ((e = upv(ws, s.o_acoff, s.acoff, st))) return e;
  if ((e = upv(ws, s.o_acon, s.acon, st))) return e;
  if ((e = upv(ws, s.o_woff, s.woff, st))) return e;
  if ((e = upv(ws, s.o_loff, s.loff, st))) return e;
  if ((e = upv(ws, s.o_lev, s.lev_nodes, st))) return e;
  if ((e = upv(ws, s.o_tasks, s.tasks, st))) return e;
  if ((e = upv(ws, s.o_pslot, s.pslot, st))) return e;
  if ((e = upv(ws, s.o_pdr, s.pdr, st))) return e;
  if ((e = upv(ws, s.o_pplist, s.pplist, st))) return e;
  if ((e = upv(ws, s.o_plim, s.plim, st))) return e;
  if ((e = upv(ws, s.o_pgc, s.pgc, st))) return e;
  if ((e = upv(ws, s.o_gs_pts, s.gs_chain_pts, st))) return e;
  if ((e = upv(ws, s.o_gs_off, s.gs_chain_off, st))) return e;
  if ((e = upv(ws, s.o_gs_col, s.gs_color_off, st))) return e;
  if ((e = cudaMemsetAsync(A.lam, 0, sizeof(double) * 3 * np, st))) return e;
  if ((e = cudaMemsetAsync(A.mf.F, 0, sizeof(double) * s.front_doubles, st))) return e;  // upper parts stay 0
  int32_t it[10] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0};  // iters[4] and rmax[3] = 0
  if ((e = cudaMemcpyAsync(A.iters, it, sizeof(it), cudaMemcpyHostToDevice, st))) return e;
  return cudaStreamSynchronize(st);  // the host vectors above are pageable; keep them alive until copied
}

}  // namespace mabd

// Developer introspection (not part of include/mabd.h): symbolic statistics of the sparse plan of a scene.
// See include/mabd.h (mabd_sparse_plan_stats).
extern "C" mabd_status mabd_sparse_plan_stats(const mabd_bodies* B, const mabd_joints* J, double* out) {
  mabd::Plan p;
  std::string msg;
  mabd_options o{};
  o.newton_iters = 1;
  o.residual_rhs = 1;
  o.solver = MABD_SOLVER_SPARSE;
  o.world = 1;
  const mabd_status st = mabd::build_plan(B, J, &o, &p, &msg);
  if (st != MABD_OK) return st;
  const mabd::SparsePlan& s = p.sparse;
  out[0] = s.nnode;
  out[1] = (double)s.levels.size();
  out[2] = s.max_f;
  out[3] = (double)s.front_doubles;
  out[4] = s.flops;
  out[5] = (double)s.tasks.size();
  out[6] = p.launches_per_step;
  out[7] = (double)p.n_dual_rows;
  return MABD_OK;
}

// See include/mabd.h (mabd_line_gs_plan).
extern "C" mabd_status mabd_line_gs_plan(const mabd_bodies* B, const mabd_joints* J, int32_t* chain_pts,
                                         int32_t* chain_off, int32_t* color_off, int64_t* counts) {
  if (!counts) return MABD_EINVAL;
  mabd::Plan p;
  std::string msg;
  mabd_options o{};
  o.solver = MABD_SOLVER_LINE_GS;
  o.world = 1;
  const mabd_status st = mabd::build_plan(B, J, &o, &p, &msg);
  if (st != MABD_OK) return st;
  const mabd::SparsePlan& s = p.sparse;
  counts[0] = (int64_t)s.gs_chain_pts.size();
  counts[1] = (int64_t)s.gs_chain_off.size() - 1;
  counts[2] = s.gs_ncolor;
  if (chain_pts) std::copy(s.gs_chain_pts.begin(), s.gs_chain_pts.end(), chain_pts);
  if (chain_off) std::copy(s.gs_chain_off.begin(), s.gs_chain_off.end(), chain_off);
  if (color_off) std::copy(s.gs_color_off.begin(), s.gs_color_off.end(), color_off);
  return MABD_OK;
}
