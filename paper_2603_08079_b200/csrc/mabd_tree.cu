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
// Parallel schedule: a predict kernel for all bodies; bodies are grouped into CTA-local subtrees (≤ 256 bodies;
// levels separated by __syncthreads; upward one warp per body, downward one thread per body) plus a top group
// (bodies whose subtree is larger), whose levels run as one launch each over the whole GPU.
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

// triangular index t → (row, column), column ≤ row, row-major over the lower triangle (lane-divergent indices:
// computed, not looked up in constant memory, which would serialise the lanes)
__device__ __forceinline__ void tri_rc(int t, int& r, int& c) {
  r = (int)((sqrtf(8.0f * (float)t + 1.0f) - 1.0f) * 0.5f);
  if ((r + 1) * (r + 2) / 2 <= t) ++r;
  if (r * (r + 1) / 2 > t) --r;
  c = t - r * (r + 1) / 2;
}

__device__ __forceinline__ void treport(const StepConsts& k, int32_t flag) {
  atomicOr(k.err, flag);
  atomicMin(k.err + 1, k.step_index);
}

// Stages 1-2 for every body at once (no tree dependency): R and δq̃ → bscr.
__global__ void tree_predict_kernel(TreeArgs a, int64_t b0, int64_t b1) {
  const StepConsts& k = a.k;
  const int64_t ld = a.b.ld;
  for (int64_t b = b0 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; b < b1; b += (int64_t)gridDim.x * blockDim.x) {
    double q[12], qd[12], R[9], dqt[12];
#pragma unroll
    for (int c = 0; c < 12; ++c) {
      q[c] = a.b.q[c * ld + b];
      qd[c] = a.b.qd[c * ld + b];
    }
    const int mid = a.b.mat_id ? a.b.mat_id[b] : 0;
    const double msc = a.b.mscale ? a.b.mscale[b] : 1.0;
    const Material M = a.b.mats[mid];
    HinvBlk H;
    if (a.hinv_tab)
      H = a.hinv_tab[mid];
    else
      hinv_blocks(M, msc, k.ih2, H);
    double W[6];
    if (!predict_body(q, qd, M, msc, H, k.ih, k.grav, R, dqt, load_wrench(a.b, b, W))) treport(k, ERR_NONFINITE);
    double* sc = a.bscr + 21 * b;
#pragma unroll
    for (int c = 0; c < 9; ++c) sc[c] = R[c];
#pragma unroll
    for (int c = 0; c < 12; ++c) sc[9 + c] = dqt[c];
  }
}

// Point i of body b's frontal matrix: the points of its child joints (sign +, b is their parent side), then the
// points of its up joint (sign −, b is its child side).
__device__ __forceinline__ void tree_point(const TreeArgs& a, int c0, int N, int u, int i, const double*& y, int& ji,
                                           int& pi, double& sg) {
  int row = 3 * i, jj = c0;
  if (row < N) {
    while (true) {
      const int n3 = 3 * a.jnpts[a.child_joint[jj]];
      if (row < n3) break;
      row -= n3;
      ++jj;
    }
    ji = a.child_joint[jj];
    pi = row / 3;
    sg = 1.0;
    y = a.jy + 12 * (int64_t)ji + 3 * pi;
  } else {
    ji = u;
    pi = (row - N) / 3;
    sg = -1.0;
    y = a.jy + 12 * (int64_t)ji + 6 + 3 * pi;
  }
}

// Upward elimination at body b by one warp. The frontal matrix F (M×M, lower part) with the right-hand side as
// column M lives in shared memory (row stride MS). A partial Cholesky over the N child-joint columns leaves
//   F[N:,N:] = Ŝ_u = F_uu − F_uX F_XX⁻¹ F_Xu,  F[N:,M] = r̂_u = r_u − F_uX F_XX⁻¹ r_X,
//   F[:N,:N] = L (F_XX = LLᵀ),  F[N:,:N] = F_uX L⁻ᵀ,  F[:N,M] = L⁻¹ r_X,
// then Lᵀ back substitutions give y = F_XX⁻¹ r_X and W = F_XX⁻¹ F_Xu for the downward pass.
__device__ void tree_up_warp(const TreeArgs& a, int b, int lane, double* F, int MS) {
  const StepConsts& k = a.k;
  const int64_t ld = a.b.ld;
  const int c0 = a.child_off[b], c1 = a.child_off[b + 1];
  const int u = a.up_joint[b];
  const int nn = a.body_nn[b], N = nn & 255, nu = nn >> 8;
  const int M = N + nu, npt = M / 3;
  const int32_t* pcode = a.pt_code + a.pt_off[b];
  double R[9], qt[12];
  {
    const double* sc = a.bscr + 21 * (int64_t)b;
#pragma unroll
    for (int c = 0; c < 9; ++c) R[c] = sc[c];
#pragma unroll
    for (int c = 0; c < 12; ++c) qt[c] = a.b.q[c * ld + b] + sc[9 + c];  // q̃
  }
  HinvBlk H;
  {
    const int mid = a.b.mat_id ? a.b.mat_id[b] : 0;
    if (a.hinv_tab)
      H = a.hinv_tab[mid];
    else
      hinv_blocks(a.b.mats[mid], a.b.mscale ? a.b.mscale[b] : 1.0, k.ih2, H);
  }
  // right-hand side: this body's side of C(q̃) plus the condensed child side
  for (int i = lane; i < npt; i += 32) {
    const int code = pcode[i];
    const int ji = code >> 2, pi = (code >> 1) & 1;
    const double si = (code & 1) ? -1.0 : 1.0;
    const double* yi = a.jy + 12 * (int64_t)ji + 6 * (code & 1) + 3 * pi;
    double x[3];
    point_pos(qt, yi, x);
#pragma unroll
    for (int e = 0; e < 3; ++e) {
      double v;
      if (si < 0)
        v = -x[e];
      else if (a.jchd[ji] < 0)  // anchor: C = x_b(ȳ) − p_world
        v = x[e] - a.jy[12 * (int64_t)ji + 6 + 3 * pi + e];
      else
        v = x[e] + a.rhat[6 * (int64_t)ji + 3 * pi + e];
      F[(3 * i + e) * MS + M] = v;
    }
  }
  // blocks (i, j), j ≤ i: s_i s_j R P(ȳ_i, ȳ_j) Rᵀ (+ Ŝ_k on a child joint's own block)
  const int npair = npt * (npt + 1) / 2;
  for (int t = lane; t < npair; t += 32) {
    int i, j;
    tri_rc(t, i, j);
    const int ci = pcode[i], cj = pcode[j];
    const int ji = ci >> 2, pi = (ci >> 1) & 1, jj = cj >> 2, pj = (cj >> 1) & 1;
    const double si = (ci & 1) ? -1.0 : 1.0, sj = (cj & 1) ? -1.0 : 1.0;
    const double* yi = a.jy + 12 * (int64_t)ji + 6 * (ci & 1) + 3 * pi;
    const double* yj = a.jy + 12 * (int64_t)jj + 6 * (cj & 1) + 3 * pj;
    double P[9], Bk[9];
    pblock(H, yi, yj, P);
    rot_conj(R, P, Bk);
    const double sg = si * sj;
    const bool add_s = si > 0 && sj > 0 && ji == jj && a.jchd[ji] >= 0;
#pragma unroll
    for (int r = 0; r < 3; ++r)
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        double v = sg * Bk[3 * r + c];
        if (add_s) v += a.Shat[36 * (int64_t)ji + 6 * (3 * pi + r) + 3 * pj + c];
        if (3 * i + r >= 3 * j + c) F[(3 * i + r) * MS + 3 * j + c] = v;
      }
  }
  __syncwarp();
  // partial Cholesky of the augmented lower matrix over the N child-joint columns, by 3×3 point blocks:
  // factor the diagonal block (lane 0, closed form, its inverse Li kept in shared memory), scale the block
  // column and the right-hand side, rank-3 update of the trailing lower part
  double* Li = F + (size_t)M * MS;  // [N/3][9] inverses of the diagonal blocks (after the front rows)
  const int NB = N / 3;
  for (int kb = 0; kb < NB; ++kb) {
    const int c = 3 * kb;
    if (lane == 0) {
      const double d00 = F[c * MS + c], d10 = F[(c + 1) * MS + c], d20 = F[(c + 2) * MS + c];
      const double d11 = F[(c + 1) * MS + c + 1], d21 = F[(c + 2) * MS + c + 1], d22 = F[(c + 2) * MS + c + 2];
      // pivots by refined hardware reciprocal square roots (fast_rsqrt, ≤ 1 ulp): l = p·p^{-1/2}
      double p0 = d00;
      bool ok = p0 > 0.0;
      const double i00 = fast_rsqrt(ok ? p0 : 1.0), l00 = (ok ? p0 : 1.0) * i00;
      const double l10 = d10 * i00, l20 = d20 * i00;
      const double p1 = d11 - l10 * l10;
      ok = ok && p1 > 0.0;
      const double i11 = fast_rsqrt(p1 > 0.0 ? p1 : 1.0), l11 = (p1 > 0.0 ? p1 : 1.0) * i11;
      const double l21 = (d21 - l20 * l10) * i11;
      const double p2 = d22 - l20 * l20 - l21 * l21;
      ok = ok && p2 > 0.0;
      const double i22 = fast_rsqrt(p2 > 0.0 ? p2 : 1.0), l22 = (p2 > 0.0 ? p2 : 1.0) * i22;
      if (!ok) treport(k, ERR_SINGULAR);
      F[c * MS + c] = l00;
      F[(c + 1) * MS + c] = l10;
      F[(c + 2) * MS + c] = l20;
      F[(c + 1) * MS + c + 1] = l11;
      F[(c + 2) * MS + c + 1] = l21;
      F[(c + 2) * MS + c + 2] = l22;
      // Li = L⁻¹ (lower): row-major 3×3
      double* li = Li + 9 * kb;
      li[0] = i00;
      li[1] = 0.0;
      li[2] = 0.0;
      li[3] = -l10 * i00 * i11;
      li[4] = i11;
      li[5] = 0.0;
      li[6] = (l10 * l21 - l20 * l11) * i00 * i11 * i22;
      li[7] = -l21 * i11 * i22;
      li[8] = i22;
      // right-hand side of the block: y_k = Li r_k
      const double r0 = F[c * MS + M], r1 = F[(c + 1) * MS + M], r2 = F[(c + 2) * MS + M];
      F[c * MS + M] = li[0] * r0;
      F[(c + 1) * MS + M] = li[3] * r0 + li[4] * r1;
      F[(c + 2) * MS + M] = li[6] * r0 + li[7] * r1 + li[8] * r2;
    }
    __syncwarp();
    const double* li = Li + 9 * kb;
    for (int r = c + 3 + lane; r < M; r += 32) {  // block column below: F[r, c:c+3] ← F[r, c:c+3] Liᵀ
      const double f0 = F[r * MS + c], f1 = F[r * MS + c + 1], f2 = F[r * MS + c + 2];
      F[r * MS + c] = li[0] * f0;
      F[r * MS + c + 1] = li[3] * f0 + li[4] * f1;
      F[r * MS + c + 2] = li[6] * f0 + li[7] * f1 + li[8] * f2;
    }
    __syncwarp();
    // trailing: F[r][cc] −= Σ_e L[r][c+e] L[cc][c+e] (c+3 ≤ cc ≤ r < M); rhs[r] −= Σ_e L[r][c+e] y[c+e]
    // lanes as a fixed 4 × 8 tile over (row, column): no runtime index division
    for (int r = c + 3 + (lane >> 3); r < M; r += 4) {
      const double l0 = F[r * MS + c], l1 = F[r * MS + c + 1], l2 = F[r * MS + c + 2];
      for (int cc = c + 3 + (lane & 7); cc <= r; cc += 8)
        F[r * MS + cc] -= l0 * F[cc * MS + c] + l1 * F[cc * MS + c + 1] + l2 * F[cc * MS + c + 2];
    }
    for (int r = c + 3 + lane; r < M; r += 32)
      F[r * MS + M] -= F[r * MS + c] * F[c * MS + M] + F[r * MS + c + 1] * F[(c + 1) * MS + M] +
                       F[r * MS + c + 2] * F[(c + 2) * MS + M];
    __syncwarp();
  }
  // back substitutions Lᵀ Z = V by 3×3 blocks (last block first): V column 0 = L⁻¹r_X (F column M), columns
  // 1..nu = the rows N..M−1 of F_uX L⁻ᵀ (F[N+col−1][0:N]); Z overwrites V: y = F_XX⁻¹ r_X, W = F_XX⁻¹ F_Xu
  auto vref = [&](int r, int col) -> double& { return col == 0 ? F[r * MS + M] : F[(N + col - 1) * MS + r]; };
  const int ncol = nu + 1;
  // lane → (row offset, column) of the (rows × ncol) updates, computed once (ncol ≤ 7, rstep = ⌊32/ncol⌋ rows)
  const int rstep = 32 / ncol, lcol = lane % ncol, lrow = lane / ncol;
  const bool lact = lrow < rstep;
  for (int kb = NB - 1; kb >= 0; --kb) {
    const int c = 3 * kb;
    const double* li = Li + 9 * kb;
    double z = 0.0;
    const int e = lane / ncol, col = lane % ncol;
    if (lane < 3 * ncol) {  // z_k = Liᵀ v_k (row e, column col)
      z = li[e] * vref(c, col) + li[3 + e] * vref(c + 1, col) + li[6 + e] * vref(c + 2, col);
    }
    __syncwarp();
    if (lane < 3 * ncol) vref(c + e, col) = z;
    __syncwarp();
    if (lact)
      for (int r = lrow; r < c; r += rstep)  // earlier rows: v_j −= L[c:c+3, j]ᵀ z_k
        vref(r, lcol) -= F[c * MS + r] * vref(c, lcol) + F[(c + 1) * MS + r] * vref(c + 1, lcol) +
                         F[(c + 2) * MS + r] * vref(c + 2, lcol);
    __syncwarp();
  }
  double* ws = a.ws + a.ws_off[b];  // y [N], W [N][nu]
  if (lact)
    for (int r = lrow; r < N; r += rstep) {
      if (lcol == 0)
        ws[r] = vref(r, 0);
      else
        ws[N + r * nu + lcol - 1] = vref(r, lcol);
    }
  if (u >= 0) {  // condensed child side of the up joint (Ŝ_u symmetric: lower part mirrored)
    for (int t = lane; t < nu * nu; t += 32) {
      const int r = t / nu, c = t % nu;
      const int rr = r > c ? r : c, cc = r > c ? c : r;
      a.Shat[36 * (int64_t)u + 6 * r + c] = F[(N + rr) * MS + N + cc];
    }
    if (lane < nu) a.rhat[6 * (int64_t)u + lane] = F[(N + lane) * MS + M];
  } else {  // root: λ_X = y
    __syncwarp();
    int off = 0;
    for (int j = c0; j < c1; ++j) {
      const int kj = a.child_joint[j];
      const int n3 = 3 * a.jnpts[kj];
      for (int r = lane; r < n3; r += 32) a.lam[6 * (int64_t)kj + r] = F[(off + r) * MS + M];
      off += n3;
    }
  }
  __syncwarp();
}

// Downward pass at body b: λ_X = y − W λ_u for its child-joint points, then the update (stage 4). Every input
// except λ_u (written by the parent's level) is fetched up front from the per-body tables (body_nn, pt_code,
// bscr, ws), so one thread waits on about three dependent memory round trips instead of walking the child
// lists.
__device__ void tree_down(const TreeArgs& a, int b) {
  const StepConsts& k = a.k;
  const int64_t ld = a.b.ld;
  const int nn = a.body_nn[b], N = nn & 255, nu = nn >> 8;
  const int u = a.up_joint[b];
  const int32_t* pcode = a.pt_code + a.pt_off[b];
  const double* ws = a.ws + a.ws_off[b];
  const double* sc = a.bscr + 21 * (int64_t)b;
  double R[9];
#pragma unroll
  for (int c = 0; c < 9; ++c) R[c] = sc[c];
  HinvBlk H;
  {
    const int mid = a.b.mat_id ? a.b.mat_id[b] : 0;
    if (a.hinv_tab)
      H = a.hinv_tab[mid];
    else
      hinv_blocks(a.b.mats[mid], a.b.mscale ? a.b.mscale[b] : 1.0, k.ih2, H);
  }
  double lu[6];  // fixed-size, fully unrolled accesses only (no local memory)
#pragma unroll
  for (int r = 0; r < 6; ++r) lu[r] = r < nu ? a.lam[6 * (int64_t)u + r] : 0.0;
  double gq[12];
#pragma unroll
  for (int c = 0; c < 12; ++c) gq[c] = 0.0;
#pragma unroll 2
  for (int i = 0; i < N / 3; ++i) {  // child-joint points (this body is their parent side, sign +)
    const int code = pcode[i];
    const int kj = code >> 2, pp = (code >> 1) & 1;
    double lam[3], w[3];
#pragma unroll
    for (int r = 0; r < 3; ++r) {
      double v = ws[3 * i + r];
      const double* wr = ws + N + (3 * i + r) * nu;
#pragma unroll
      for (int c = 0; c < 6; ++c)
        if (c < nu) v -= wr[c] * lu[c];
      lam[r] = v;
      a.lam[6 * (int64_t)kj + 3 * pp + r] = v;
    }
    mat3t_vec(R, lam, w);
    add_point_force(gq, a.jy + 12 * (int64_t)kj + 3 * pp, w, 1.0);
  }
#pragma unroll
  for (int pp = 0; pp < 2; ++pp) {  // up-joint points (this body is their child side, sign −)
    if (3 * pp >= nu) break;
    double w[3];
    mat3t_vec(R, lu + 3 * pp, w);
    add_point_force(gq, a.jy + 12 * (int64_t)u + 6 + 3 * pp, w, -1.0);
  }
  double uu[12];
  hinv_apply(H, gq, uu);
#pragma unroll
  for (int kb = 0; kb < 4; ++kb) {
    double c3[3];
    mat3_vec(R, uu + 3 * kb, c3);
#pragma unroll
    for (int e = 0; e < 3; ++e) {
      const int c = 3 * kb + e;
      const double dq = sc[9 + c] - c3[e];
      a.b.q[c * ld + b] += dq;
      if (k.niter == 1)
        a.b.qd[c * ld + b] = dq * k.ih;
      else  // K > 1: v ← v − δq/h + h·grav (launch_step in mabd_plan.cu)
        a.b.qd[c * ld + b] += -dq * k.ih + (c >= 9 ? k.h * k.grav[c - 9] : 0.0);
    }
  }
}

__global__ void __launch_bounds__(512) tree_kernel(TreeArgs a, int mode, int MS) {
  extern __shared__ double tsm[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  double* F = tsm + (size_t)warp * (a.front_rows * MS + 9 * (TREE_MAXN / 3));
  if (mode == TREE_UP_LEVEL || mode == TREE_DOWN_LEVEL) {  // one level of the top group over the whole grid
    const int l = a.group0;
    const int b = a.glev_off[l] + (mode == TREE_UP_LEVEL ? blockIdx.x * nw + warp : blockIdx.x * blockDim.x + threadIdx.x);
    if (b >= a.glev_off[l + 1]) return;
    if (mode == TREE_UP_LEVEL)
      tree_up_warp(a, b, lane, F, MS);
    else
      tree_down(a, b);
    return;
  }
  const int g = a.group0 + blockIdx.x;
  const int l0 = a.glev_ptr[g], l1 = a.glev_ptr[g + 1] - 1;  // levels l ∈ [l0, l1): [glev_off[l], glev_off[l+1])
  if (mode == TREE_UP || mode == TREE_BOTH) {
    for (int l = l0; l < l1; ++l) {  // deepest first; one warp per body
      for (int b = a.glev_off[l] + warp; b < a.glev_off[l + 1]; b += nw) tree_up_warp(a, b, lane, F, MS);
      __syncthreads();
    }
  }
  if (mode == TREE_DOWN || mode == TREE_BOTH) {
    for (int l = l1 - 1; l >= l0; --l) {  // shallowest first; one thread per body
      for (int b = a.glev_off[l] + threadIdx.x; b < a.glev_off[l + 1]; b += blockDim.x) tree_down(a, b);
      __syncthreads();
    }
  }
}

// Multi-part split: the condensed child side (Ŝ_u 36, r̂_u 6) of every joint from a top body into a bottom group,
// packed by the part owning the group into its block of the all-gather buffer, then unpacked by every part into
// Shat / rhat for the top levels. Root entries [r0, r1) are those of a part's groups.
__global__ void tree_pack_kernel(TreeArgs a, int r0, int r1) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const int r = r0 + i / 42, e = i % 42;
  if (r >= r1) return;
  const int u = a.root_joint[r];
  a.xbuf[(size_t)a.root_slot[r] * 42 + e] = e < 36 ? a.Shat[36 * (int64_t)u + e] : a.rhat[6 * (int64_t)u + e - 36];
}
__global__ void tree_unpack_kernel(TreeArgs a, int nroot) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const int r = i / 42, e = i % 42;
  if (r >= nroot) return;
  const int u = a.root_joint[r];
  const double v = a.xbuf[(size_t)a.root_slot[r] * 42 + e];
  if (e < 36)
    a.Shat[36 * (int64_t)u + e] = v;
  else
    a.rhat[6 * (int64_t)u + e - 36] = v;
}

static int tree_ms(int max_m) { return max_m + 2 + ((max_m & 1) ? 0 : 1); }  // row stride (odd)

cudaError_t launch_tree(const TreeArgs& a, int ngroups, int mode, int threads, cudaStream_t st) {
  if (ngroups <= 0) return cudaSuccess;
  const int MS = tree_ms(a.front_rows);
  const size_t sm = sizeof(double) * (size_t)(threads / 32) * (a.front_rows * MS + 9 * (TREE_MAXN / 3));
  tree_kernel<<<ngroups, threads, sm, st>>>(a, mode, MS);
  return cudaGetLastError();
}

static unsigned grid_for_bodies(int64_t nb) {
  return (unsigned)std::max<int64_t>(1, std::min<int64_t>((nb + 255) / 256, 148 * 8));
}

cudaError_t tree_step(const Plan& p, const DevPtrs& d, const StepConsts& k, cudaStream_t st) {
  TreeArgs a = d.tree;
  a.k = k;
  const TreePlan& t = p.tree;
  cudaError_t e;
  // warps per CTA of the CTA-local subtrees: up to 8 within the shared memory
  const size_t per_warp = sizeof(double) * ((size_t)t.max_m * tree_ms(t.max_m) + 9 * (TREE_MAXN / 3));
  const int bot_threads = 32 * (int)std::max<size_t>(1, std::min<size_t>(8, (200 * 1024) / std::max<size_t>(per_warp, 1)));
  // bottom groups of this process: all of them, or this rank's block when the tree is split across ranks
  const bool split = t.parts > 1 && !t.emulate;
  const int g_lo = split ? std::min(t.n_bottom, t.part * t.gpr) : 0;
  const int g_hi = split ? std::min(t.n_bottom, (t.part + 1) * t.gpr) : t.n_bottom;
  const int64_t top0 = t.group_off[t.n_bottom];
  if (split) {  // stages 1-2 for this rank's bottom bodies and the (replicated) top bodies
    const int64_t b0 = t.group_off[g_lo], b1 = t.group_off[g_hi];
    if (b1 > b0) tree_predict_kernel<<<grid_for_bodies(b1 - b0), 256, 0, st>>>(a, b0, b1);
    if (a.n > top0) tree_predict_kernel<<<grid_for_bodies(a.n - top0), 256, 0, st>>>(a, top0, a.n);
  } else {
    tree_predict_kernel<<<grid_for_bodies(a.n), 256, 0, st>>>(a, 0, a.n);
  }
  if (!t.has_top) {
    a.group0 = g_lo;
    return launch_tree(a, g_hi - g_lo, TREE_BOTH, bot_threads, st);
  }
  a.group0 = g_lo;
  if ((e = launch_tree(a, g_hi - g_lo, TREE_UP, bot_threads, st))) return e;
  if (t.parts > 1) {  // exchange of the group roots' condensed blocks (one all-gather; emulated: every part local)
    const int q0 = split ? t.part : 0, q1 = split ? t.part + 1 : t.parts;
    for (int q = q0; q < q1; ++q) {
      const int lo = std::min(t.n_bottom, q * t.gpr), hi = std::min(t.n_bottom, (q + 1) * t.gpr);
      const int r0 = t.root_off[lo], r1 = t.root_off[hi];
      if (r1 > r0) tree_pack_kernel<<<(unsigned)(((r1 - r0) * 42 + 255) / 256), 256, 0, st>>>(a, r0, r1);
    }
    if (split && t.rpp > 0) {
      const int rc = nccl_allgather_doubles(d.nccl_comm, a.xbuf, (size_t)t.rpp * 42, t.part, st);
      if (rc != 0) return cudaErrorUnknown;
    }
    const int nroot = t.root_off[t.n_bottom];
    if (nroot > 0) tree_unpack_kernel<<<(unsigned)((nroot * 42 + 255) / 256), 256, 0, st>>>(a, nroot);
  }
  // the top group: one launch per level over the whole GPU (a body per warp up, per thread down), deepest first
  const int g = t.n_bottom;
  const int l0 = t.glev_ptr[g], l1 = t.glev_ptr[g + 1] - 1;
  const int MS = tree_ms(a.front_rows);
  const int wpc = 4;  // warps per CTA of the level launches
  const size_t sm = sizeof(double) * (size_t)wpc * (a.front_rows * MS + 9 * (TREE_MAXN / 3));
  for (int l = l0; l < l1; ++l) {
    const int nb = t.glev_off[l + 1] - t.glev_off[l];
    a.group0 = l;
    tree_kernel<<<(nb + wpc - 1) / wpc, 32 * wpc, sm, st>>>(a, TREE_UP_LEVEL, MS);
  }
  for (int l = l1 - 1; l >= l0; --l) {
    const int nb = t.glev_off[l + 1] - t.glev_off[l];
    a.group0 = l;
    tree_kernel<<<(nb + 127) / 128, 128, 0, st>>>(a, TREE_DOWN_LEVEL, MS);
  }
  if ((e = cudaGetLastError())) return e;
  a.group0 = g_lo;
  return launch_tree(a, g_hi - g_lo, TREE_DOWN, bot_threads, st);
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

cudaError_t tree_init() {
  return cudaFuncSetAttribute(tree_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 210 * 1024);
}

// ============================================================================ host: topology and ordering
bool tree_build(const mabd_joints* J, int64_t n, Plan* p, std::vector<int64_t>* pos_of_body, std::string* msg) {
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
  std::vector<int64_t> local_roots;
  for (int64_t v : bfs)
    if (size[v] <= TREE_CAP && (parent[v] < 0 || size[parent[v]] > TREE_CAP)) local_roots.push_back(v);
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
    if (cur.size() + sub.size() > (size_t)TREE_CAP) {
      groups.push_back(cur);
      cur.clear();
    }
    cur.insert(cur.end(), sub.begin(), sub.end());
  }
  if (!cur.empty()) groups.push_back(cur);
  TreePlan& t = p->tree;
  t = TreePlan();
  t.n_bottom = (int32_t)groups.size();
  std::vector<int64_t> top;
  for (int64_t v : bfs)
    if (size[v] > TREE_CAP) top.push_back(v);
  if (!top.empty()) {
    groups.push_back(top);
    t.has_top = true;
  }
  // internal order: groups in sequence, each sorted by depth (deepest first). Level ranges: group g owns
  // levels l ∈ [glev_ptr[g], glev_ptr[g+1]−1), level l spans bodies [glev_off[l], glev_off[l+1]).
  pos_of_body->assign(n, -1);
  std::vector<int64_t> body_of(n);
  int64_t pos = 0;
  t.group_off.push_back(0);
  for (auto& gvec : groups) {
    std::stable_sort(gvec.begin(), gvec.end(), [&](int64_t x, int64_t y) { return depth[x] > depth[y]; });
    t.glev_ptr.push_back((int32_t)t.glev_off.size());
    for (size_t i = 0; i < gvec.size(); ++i) {
      if (i == 0 || depth[gvec[i]] != depth[gvec[i - 1]]) t.glev_off.push_back((int32_t)(pos + i));
      (*pos_of_body)[gvec[i]] = pos + (int64_t)i;
      body_of[pos + i] = gvec[i];
    }
    pos += (int64_t)gvec.size();
    t.glev_off.push_back((int32_t)pos);  // terminator of the group's last level
    t.group_off.push_back((int32_t)pos);
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
    t.max_m = std::max(t.max_m, N + nu);
    // frontal point list: child joints' points (parent side, +), then the up joint's (child side, −);
    // code = 4·joint + 2·point + (1 for the child side)
    t.pt_off.push_back((int32_t)t.pt_code.size());
    for (int32_t kk : cj[i])
      for (int q = 0; q < t.jnpts[kk]; ++q) t.pt_code.push_back(4 * kk + 2 * q);
    if (upj[v] >= 0)
      for (int q = 0; q < t.jnpts[upj[v]]; ++q) t.pt_code.push_back(4 * (int32_t)upj[v] + 2 * q + 1);
    t.body_nn.push_back((int32_t)(N | (nu << 8)));
  }
  t.pt_off.push_back((int32_t)t.pt_code.size());
  t.ws_total = t.ws_off[n];
  p->ld = n;
  {
    int top_levels = 0;
    if (t.has_top) top_levels = t.glev_ptr[t.n_bottom + 1] - 1 - t.glev_ptr[t.n_bottom];
    p->launches_per_step = 1 + (t.has_top ? 2 + 2 * top_levels : 1);
  }
  return true;
}

}  // namespace mabd
