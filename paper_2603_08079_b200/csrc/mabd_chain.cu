// Chain solver of the M-ABD step on sm_100a: fused per-segment kernel (stages 1-4) and the hierarchical
// block-tridiagonal reduced-system kernels for chains longer than one segment.
//
// Paper: the chain dual is block tridiagonal (Eq. chain-btd); the paper solves it with block
// Thomas in O(K) on one thread. Here each CTA owns a 256-slot segment of a chain and solves its
// 257-equation block-tridiagonal system by block cyclic reduction in shared memory (log₂ 256 = 8 levels),
// so the per-body stages and the solve are fused into one pass over HBM:
//   per body:  load qⁿ, q̇ⁿ → polar R → f_A → δq̃ (stages 1-2)
//   per joint: D, B, r = C(q̃) from the constant 3×3 kernels P(ȳ,ȳ') rotated by R
//   per segment: cyclic reduction → λ
//   per body:  qⁿ⁺¹ = q̃ − diag₄(R)H̄⁻¹ Σ ±(ȳ_aug ⊗ Rᵀλ), q̇ⁿ⁺¹ = (qⁿ⁺¹ − qⁿ)/h
// Chains that span several segments are partitioned (SPIKE-style): each segment reduces its interior to a
// 2-equation "top" system on its end slots (REDUCE), the tops form a smaller block-tridiagonal system
// solved recursively by btd_kernel, and each segment then recomputes and back-substitutes (FINISH).
#include <cuda_runtime.h>

#include "mabd_device.cuh"
#include "mabd_kernels.h"

namespace mabd {

// ------------------------------------------------------------------ shared-memory cyclic reduction
// Equations i = 0..256:  Bl_i λ_{i-s} + D_i λ_i + Br_i λ_{i+s} = r_i at stride s, with Bl_i = Br_{i-s}ᵀ.
// sD [NEQ][6] (sym; replaced by its inverse once eliminated), sB [NEQ][9] (Br), sBl [NEQ][9] (saved Br_{i-s}
// of eliminated i), sR [NEQ][3] (rhs, then λ).
struct CRS {
  double* D;
  double* B;
  double* Bl;
  double* r;
};

__device__ __forceinline__ void report(const StepConsts& k, int32_t flag) {
  atomicOr(k.err, flag);
  atomicMin(k.err + 1, k.step_index);
}

__device__ void cr_forward(const CRS& s, int t, const StepConsts& k) {
  for (int st = 1; st < SEG; st <<= 1) {
    const int two = st << 1;
    if ((t & (two - 1)) == st) {  // eliminated at this level: invert its D
      double Di[6];
      if (!sym_inv_spd(s.D + 6 * t, Di)) report(k, ERR_SINGULAR);
#pragma unroll
      for (int e = 0; e < 6; ++e) s.D[6 * t + e] = Di[e];
    }
    __syncthreads();
    const int kq = (t == SEG - 1) ? SEG : t;  // thread 255 (never even) carries equation 256
    if ((kq & (two - 1)) == 0) {
      double D[9], Br[9], r[3];
      full_from_sym(s.D + 6 * kq, D);
#pragma unroll
      for (int e = 0; e < 9; ++e) Br[e] = s.B[9 * kq + e];
#pragma unroll
      for (int e = 0; e < 3; ++e) r[e] = s.r[3 * kq + e];
      double nBr[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
      if (kq >= st) {  // left neighbour i = kq - st:  α = Br_iᵀ D_i⁻¹
        const int i = kq - st;
        double Di[9], Bi[9], al[9], tmp[9];
        full_from_sym(s.D + 6 * i, Di);
#pragma unroll
        for (int e = 0; e < 9; ++e) Bi[e] = s.B[9 * i + e];
        mat3_mul_at(Bi, Di, al);          // α = Biᵀ Di⁻¹
        mat3_mul(al, Bi, tmp);            // α Br_i
#pragma unroll
        for (int e = 0; e < 9; ++e) D[e] -= tmp[e];
        double ri[3], ar[3];
#pragma unroll
        for (int e = 0; e < 3; ++e) ri[e] = s.r[3 * i + e];
        mat3_vec(al, ri, ar);
#pragma unroll
        for (int e = 0; e < 3; ++e) r[e] -= ar[e];
      }
      if (kq < SEG) {  // right neighbour j = kq + st:  γ = Br_k D_j⁻¹
        const int j = kq + st;
        double Dj[9], ga[9], tmp[9], Bj[9];
        full_from_sym(s.D + 6 * j, Dj);
        mat3_mul(Br, Dj, ga);             // γ
        mat3_mul_bt(ga, Br, tmp);         // γ Br_kᵀ  (= γ Bl_j)
#pragma unroll
        for (int e = 0; e < 9; ++e) D[e] -= tmp[e];
        double rj[3], gr[3];
#pragma unroll
        for (int e = 0; e < 3; ++e) rj[e] = s.r[3 * j + e];
        mat3_vec(ga, rj, gr);
#pragma unroll
        for (int e = 0; e < 3; ++e) r[e] -= gr[e];
#pragma unroll
        for (int e = 0; e < 9; ++e) Bj[e] = s.B[9 * j + e];
        mat3_mul(ga, Bj, tmp);            // new Br_k = −γ Br_j
#pragma unroll
        for (int e = 0; e < 9; ++e) nBr[e] = -tmp[e];
#pragma unroll
        for (int e = 0; e < 9; ++e) s.Bl[9 * j + e] = Br[e];  // j's left coupling at this level
      }
      double Ds[6];
      sym_from_full(D, Ds);
      // symmetrise (the two updates are symmetric in exact arithmetic)
      Ds[1] = 0.5 * (D[1] + D[3]);
      Ds[2] = 0.5 * (D[2] + D[6]);
      Ds[4] = 0.5 * (D[5] + D[7]);
#pragma unroll
      for (int e = 0; e < 6; ++e) s.D[6 * kq + e] = Ds[e];
#pragma unroll
      for (int e = 0; e < 9; ++e) s.B[9 * kq + e] = nBr[e];
#pragma unroll
      for (int e = 0; e < 3; ++e) s.r[3 * kq + e] = r[e];
    }
    __syncthreads();
  }
}

// Solve the remaining 2-equation system [D0 B; Bᵀ D1][λ0; λ1] = [r0; r1] (one thread).
__device__ void cr_solve_top(const CRS& s, const StepConsts& k) {
  double D0i[6], D0[9], B[9], D1s[6], D1[9], r0[3], r1[3];
#pragma unroll
  for (int e = 0; e < 9; ++e) B[e] = s.B[e];
#pragma unroll
  for (int e = 0; e < 3; ++e) { r0[e] = s.r[e]; r1[e] = s.r[3 * SEG + e]; }
  if (!sym_inv_spd(s.D, D0i)) report(k, ERR_SINGULAR);
  full_from_sym(D0i, D0);
  full_from_sym(s.D + 6 * SEG, D1);
  double W[9], T[9];
  mat3_mul(D0, B, W);          // D0⁻¹ B
  mat3_mul_at(B, W, T);        // Bᵀ D0⁻¹ B
#pragma unroll
  for (int e = 0; e < 9; ++e) D1[e] -= T[e];
  double y[3], z[3];
  mat3_vec(D0, r0, y);         // D0⁻¹ r0
  mat3t_vec(B, y, z);          // Bᵀ D0⁻¹ r0
#pragma unroll
  for (int e = 0; e < 3; ++e) r1[e] -= z[e];
  sym_from_full(D1, D1s);
  D1s[1] = 0.5 * (D1[1] + D1[3]);
  D1s[2] = 0.5 * (D1[2] + D1[6]);
  D1s[4] = 0.5 * (D1[5] + D1[7]);
  double S1i[6], l1[3], l0[3], Bl1[3];
  if (!sym_inv_spd(D1s, S1i)) report(k, ERR_SINGULAR);
  sym_vec(S1i, r1, l1);
  mat3_vec(B, l1, Bl1);
#pragma unroll
  for (int e = 0; e < 3; ++e) r0[e] -= Bl1[e];
  mat3_vec(D0, r0, l0);
#pragma unroll
  for (int e = 0; e < 3; ++e) { s.r[e] = l0[e]; s.r[3 * SEG + e] = l1[e]; }
}

// Back substitution; sR[0] and sR[256] hold λ of the end equations on entry, all λ on exit.
__device__ void cr_backward(const CRS& s, int t) {
  for (int st = SEG / 2; st >= 1; st >>= 1) {
    const int two = st << 1;
    if ((t & (two - 1)) == st) {
      const int i = t;
      double Bl[9], Br[9], Di[6], ll[3], lr[3], v[3], w[3];
#pragma unroll
      for (int e = 0; e < 9; ++e) { Bl[e] = s.Bl[9 * i + e]; Br[e] = s.B[9 * i + e]; }
#pragma unroll
      for (int e = 0; e < 6; ++e) Di[e] = s.D[6 * i + e];
#pragma unroll
      for (int e = 0; e < 3; ++e) { ll[e] = s.r[3 * (i - st) + e]; lr[e] = s.r[3 * (i + st) + e]; v[e] = s.r[3 * i + e]; }
      mat3t_vec(Bl, ll, w);  // Bl_i λ_{i-s} = Br_{i-s}ᵀ λ_{i-s}
#pragma unroll
      for (int e = 0; e < 3; ++e) v[e] -= w[e];
      mat3_vec(Br, lr, w);
#pragma unroll
      for (int e = 0; e < 3; ++e) v[e] -= w[e];
      sym_vec(Di, v, w);
#pragma unroll
      for (int e = 0; e < 3; ++e) s.r[3 * i + e] = w[e];
    }
    __syncthreads();
  }
}

__device__ __forceinline__ CRS cr_smem(double* smem) {
  CRS s;
  s.D = smem;
  s.B = s.D + NEQ * 6;
  s.Bl = s.B + NEQ * 9;
  s.r = s.Bl + NEQ * 9;
  return s;
}

// ------------------------------------------------------------------ the fused chain segment kernel
template <bool FINISH>
__global__ void __launch_bounds__(SEG) chain_kernel(ChainArgs a) {
  extern __shared__ double smem[];
  const CRS s = cr_smem(smem);
  const int t = threadIdx.x;
  const int g = a.seg_list ? a.seg_list[blockIdx.x] : (int)blockIdx.x;
  const int flags = a.seg_flags[g];
  const bool is_long = (flags & SEG_LONG) != 0;
  const int64_t slot = (int64_t)g * SEG + t;
  const uint32_t info = a.slot_info[slot];
  const uint32_t infoN = a.slot_info[slot + 1];
  const bool has_body = slot_right(info) == SIDE_BODY;
  const bool eq_real = slot_real(info);
  const bool right_real = slot_real(infoN) && slot_left(infoN) == SIDE_BODY;
  const StepConsts& k = a.k;

  double q[12], dqt[12], R[9];
  HinvBlk H;
  double yR[3] = {0, 0, 0}, yL[3] = {0, 0, 0};
  double DR[6] = {0, 0, 0, 0, 0, 0}, DL[6] = {0, 0, 0, 0, 0, 0}, Bt[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
  double xR[3] = {0, 0, 0}, xL[3] = {0, 0, 0};
  if (eq_real) {
    const double* gp = a.geo + 6 * (size_t)slot_geo(info);
    if (slot_right(info) == SIDE_BODY) {
#pragma unroll
      for (int e = 0; e < 3; ++e) yR[e] = gp[3 + e];
    } else {  // end anchor: the right side is a world point
#pragma unroll
      for (int e = 0; e < 3; ++e) xR[e] = gp[3 + e];
    }
  }
  if (has_body) {
    double qd[12];
    const double* qb = a.b.q + slot;
    const double* qdb = a.b.qd + slot;
#pragma unroll
    for (int c = 0; c < 12; ++c) q[c] = __ldcs(qb + c * a.b.ld);
#pragma unroll
    for (int c = 0; c < 12; ++c) qd[c] = __ldcs(qdb + c * a.b.ld);
    const int mid = a.b.mat_id ? a.b.mat_id[slot] : 0;
    const double msc = a.b.mscale ? a.b.mscale[slot] : 1.0;
    const Material M = a.b.mats[mid];
    if (a.hinv_tab)
      H = a.hinv_tab[mid];
    else
      hinv_blocks(M, msc, k.ih2, H);
    if (!predict_body(q, qd, M, msc, H, k.ih, k.grav, R, dqt)) report(k, ERR_NONFINITE);
    double qt[12];
#pragma unroll
    for (int c = 0; c < 12; ++c) qt[c] = q[c] + dqt[c];
    double P[9], F[9];
    if (eq_real) {  // joint to the left: body is its right side (sign −)
      pblock(H, yR, yR, P);
      rot_conj(R, P, F);
      sym_from_full(F, DR);
      point_pos(qt, yR, xR);
    }
    if (right_real) {  // joint to the right: body is its left side (sign +)
      const double* gp = a.geo + 6 * (size_t)slot_geo(infoN);
#pragma unroll
      for (int e = 0; e < 3; ++e) yL[e] = gp[e];
      pblock(H, yL, yL, P);
      rot_conj(R, P, F);
      sym_from_full(F, DL);
      point_pos(qt, yL, xL);
      if (eq_real) {  // B_t = −R P(ȳ_R, ȳ_L') Rᵀ  (sign −·+)
        pblock(H, yR, yL, P);
        rot_conj(R, P, F);
#pragma unroll
        for (int e = 0; e < 9; ++e) Bt[e] = -F[e];
      }
    }
  }
  // exchange the right-joint contributions through shared memory (sBl reused as [NEQ][9] scratch)
  {
    double* x = s.Bl + 9 * (t + 1);
#pragma unroll
    for (int e = 0; e < 6; ++e) x[e] = DL[e];
#pragma unroll
    for (int e = 0; e < 3; ++e) x[6 + e] = xL[e];
    if (t == 0) {
#pragma unroll
      for (int e = 0; e < 9; ++e) s.Bl[e] = 0.0;
    }
  }
  __syncthreads();
  {
    double D[6], r[3];
    if (eq_real) {
      const double* x = s.Bl + 9 * t;
      const uint32_t ls = slot_left(info);
      double left[3] = {0, 0, 0};
      if (ls == SIDE_BODY) {
#pragma unroll
        for (int e = 0; e < 3; ++e) left[e] = x[6 + e];
#pragma unroll
        for (int e = 0; e < 6; ++e) D[e] = DR[e] + x[e];
      } else {  // world on the left (start anchor): fixed world point
        const double* gp = a.geo + 6 * (size_t)slot_geo(info);
#pragma unroll
        for (int e = 0; e < 3; ++e) left[e] = gp[e];
#pragma unroll
        for (int e = 0; e < 6; ++e) D[e] = DR[e];
      }
#pragma unroll
      for (int e = 0; e < 3; ++e) r[e] = left[e] - xR[e];  // r = C(q̃) (footnote P:459)
    } else {  // padding / absent slot: decoupled identity equation, λ = 0
      D[0] = 1; D[1] = 0; D[2] = 0; D[3] = 1; D[4] = 0; D[5] = 1;
      r[0] = r[1] = r[2] = 0;
    }
    double D256[6], r256[3];
    if (t == SEG - 1) {
      if (flags & SEG_RIGHT_IFACE) {
        const double* x = s.Bl + 9 * SEG;
#pragma unroll
        for (int e = 0; e < 6; ++e) D256[e] = x[e];
#pragma unroll
        for (int e = 0; e < 3; ++e) r256[e] = x[6 + e];
      } else {
        D256[0] = 1; D256[1] = 0; D256[2] = 0; D256[3] = 1; D256[4] = 0; D256[5] = 1;
        r256[0] = r256[1] = r256[2] = 0;
      }
    }
    __syncthreads();  // all reads of the scratch done before the CR arrays are written
#pragma unroll
    for (int e = 0; e < 6; ++e) s.D[6 * t + e] = D[e];
#pragma unroll
    for (int e = 0; e < 9; ++e) s.B[9 * t + e] = Bt[e];
#pragma unroll
    for (int e = 0; e < 3; ++e) s.r[3 * t + e] = r[e];
    if (t == SEG - 1) {
#pragma unroll
      for (int e = 0; e < 6; ++e) s.D[6 * SEG + e] = D256[e];
#pragma unroll
      for (int e = 0; e < 9; ++e) s.B[9 * SEG + e] = 0.0;
#pragma unroll
      for (int e = 0; e < 3; ++e) s.r[3 * SEG + e] = r256[e];
    }
  }
  __syncthreads();
  cr_forward(s, t, k);

  if (!is_long) {
    if (t == 0) cr_solve_top(s, k);
  } else if (!FINISH) {
    if (t == 0) {
      Top* o = a.top_out + a.seg_red[g];
#pragma unroll
      for (int e = 0; e < 6; ++e) { o->D0[e] = s.D[e]; o->D1[e] = s.D[6 * SEG + e]; }
#pragma unroll
      for (int e = 0; e < 9; ++e) o->B[e] = s.B[e];
#pragma unroll
      for (int e = 0; e < 3; ++e) { o->r0[e] = s.r[e]; o->r1[e] = s.r[3 * SEG + e]; }
    }
    return;
  } else {
    if (t == 0) {
      const int u = a.seg_red[g];
#pragma unroll
      for (int e = 0; e < 3; ++e) {
        s.r[e] = a.lam_in[3 * u + e];
        s.r[3 * SEG + e] = (flags & SEG_RIGHT_IFACE) ? a.lam_in[3 * (u + 1) + e] : 0.0;
      }
    }
  }
  __syncthreads();
  cr_backward(s, t);

  if (has_body) {  // stage 4: qⁿ⁺¹ = q̃ − diag₄(R) H̄⁻¹ Σ ±Γ(ȳ)ᵀ Rᵀλ
    double gq[12];
#pragma unroll
    for (int c = 0; c < 12; ++c) gq[c] = 0.0;
    double w[3], lam[3];
    if (eq_real) {
#pragma unroll
      for (int e = 0; e < 3; ++e) lam[e] = s.r[3 * t + e];
      mat3t_vec(R, lam, w);
      add_point_force(gq, yR, w, -1.0);
    }
    if (right_real) {
#pragma unroll
      for (int e = 0; e < 3; ++e) lam[e] = s.r[3 * (t + 1) + e];
      mat3t_vec(R, lam, w);
      add_point_force(gq, yL, w, 1.0);
    }
    double u[12];
    hinv_apply(H, gq, u);
    double* qb = a.b.q + slot;
    double* qdb = a.b.qd + slot;
#pragma unroll
    for (int kb = 0; kb < 4; ++kb) {
      double c3[3];
      mat3_vec(R, u + 3 * kb, c3);
#pragma unroll
      for (int e = 0; e < 3; ++e) {
        const int c = 3 * kb + e;
        const double dq = dqt[c] - c3[e];
        __stcs(qb + c * a.b.ld, q[c] + dq);
        __stcs(qdb + c * a.b.ld, dq * k.ih);
      }
    }
  }
}

// ------------------------------------------------------------------ reduced block-tridiagonal levels
// Unknown u of level L owns the equation built from the level-(L−1) tops:
//   D_u = top[u].D0 + (left(u) ? top[u−1].D1 : 0),  B_u = top[u].B,  r_u likewise.
// A window w of 256 unknowns is one CTA; its equation 256 is the first unknown of window w+1 (partial:
// D = 0, r = 0; its coupling from unknown 256w+255 is B_{256w+255}), or padding.
__global__ void __launch_bounds__(SEG) btd_kernel(BtdArgs a) {
  extern __shared__ double smem[];
  const CRS s = cr_smem(smem);
  const int t = threadIdx.x;
  const int64_t w = blockIdx.x;
  const int64_t u = w * SEG + t;
  const int64_t nu = a.n_u;
  {
    double D[6] = {1, 0, 0, 1, 0, 1}, B[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0}, r[3] = {0, 0, 0};
    if (u < nu) {
      const Top& T = a.top_in[u];
      const bool left = a.left_iface ? (a.left_iface[u] != 0) : (u > 0);
#pragma unroll
      for (int e = 0; e < 6; ++e) D[e] = T.D0[e] + (left ? a.top_in[u - 1].D1[e] : 0.0);
#pragma unroll
      for (int e = 0; e < 3; ++e) r[e] = T.r0[e] + (left ? a.top_in[u - 1].r1[e] : 0.0);
#pragma unroll
      for (int e = 0; e < 9; ++e) B[e] = T.B[e];
    }
#pragma unroll
    for (int e = 0; e < 6; ++e) s.D[6 * t + e] = D[e];
#pragma unroll
    for (int e = 0; e < 9; ++e) s.B[9 * t + e] = B[e];
#pragma unroll
    for (int e = 0; e < 3; ++e) s.r[3 * t + e] = r[e];
    if (t == SEG - 1) {
      const bool real_next = (w + 1) * SEG < nu;
      const double Dn[6] = {real_next ? 0.0 : 1.0, 0, 0, real_next ? 0.0 : 1.0, 0, real_next ? 0.0 : 1.0};
#pragma unroll
      for (int e = 0; e < 6; ++e) s.D[6 * SEG + e] = Dn[e];
#pragma unroll
      for (int e = 0; e < 9; ++e) s.B[9 * SEG + e] = 0.0;
#pragma unroll
      for (int e = 0; e < 3; ++e) s.r[3 * SEG + e] = 0.0;
    }
  }
  __syncthreads();
  cr_forward(s, t, a.k);
  if (a.mode == BTD_REDUCE) {
    if (t == 0) {
      Top* o = a.top_out + w;
#pragma unroll
      for (int e = 0; e < 6; ++e) { o->D0[e] = s.D[e]; o->D1[e] = s.D[6 * SEG + e]; }
#pragma unroll
      for (int e = 0; e < 9; ++e) o->B[e] = s.B[e];
#pragma unroll
      for (int e = 0; e < 3; ++e) { o->r0[e] = s.r[e]; o->r1[e] = s.r[3 * SEG + e]; }
    }
    return;
  }
  if (a.mode == BTD_FUSED) {
    if (t == 0) cr_solve_top(s, a.k);
  } else {
    if (t == 0) {
      const bool real_next = (w + 1) * SEG < nu;
#pragma unroll
      for (int e = 0; e < 3; ++e) {
        s.r[e] = a.lam_in[3 * w + e];
        s.r[3 * SEG + e] = real_next ? a.lam_in[3 * (w + 1) + e] : 0.0;
      }
    }
  }
  __syncthreads();
  cr_backward(s, t);
  if (u < nu) {
#pragma unroll
    for (int e = 0; e < 3; ++e) a.lam_out[3 * u + e] = s.r[3 * t + e];
  }
}

size_t cr_smem_bytes() { return sizeof(double) * NEQ * (6 + 9 + 9 + 3); }

cudaError_t launch_chain(const ChainArgs& a, int nblocks, bool finish, cudaStream_t st) {
  if (nblocks <= 0) return cudaSuccess;
  const size_t sm = cr_smem_bytes();
  if (finish)
    chain_kernel<true><<<nblocks, SEG, sm, st>>>(a);
  else
    chain_kernel<false><<<nblocks, SEG, sm, st>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_btd(const BtdArgs& a, int nblocks, cudaStream_t st) {
  if (nblocks <= 0) return cudaSuccess;
  btd_kernel<<<nblocks, SEG, cr_smem_bytes(), st>>>(a);
  return cudaGetLastError();
}

cudaError_t chain_kernels_init() {
  const int sm = (int)cr_smem_bytes();
  cudaError_t e = cudaFuncSetAttribute(chain_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
  if (e != cudaSuccess) return e;
  e = cudaFuncSetAttribute(chain_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
  if (e != cudaSuccess) return e;
  return cudaFuncSetAttribute(btd_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
}

// prefactor: per-material closed-form H̄⁻¹ ("pre-factorized")
__global__ void hinv_table_kernel(const Material* mats, int nm, double ih2, HinvBlk* out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < nm) hinv_blocks(mats[i], 1.0, ih2, out[i]);
}

cudaError_t launch_hinv_table(const Material* mats, int nm, double ih2, HinvBlk* out, cudaStream_t st) {
  if (nm <= 0) return cudaSuccess;
  hinv_table_kernel<<<(nm + 127) / 128, 128, 0, st>>>(mats, nm, ih2, out);
  return cudaGetLastError();
}

// state gather / scatter between the caller's AoS order and the internal SoA slots
__global__ void gather_state_kernel(const double* q, const double* qd, int64_t ld, const int64_t* perm, int64_t n,
                                    double* qo, double* qdo) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n * 12) return;
  const int64_t b = i / 12, c = i % 12;
  const int64_t sidx = perm[b];
  if (qo) qo[i] = q[c * ld + sidx];
  if (qdo) qdo[i] = qd[c * ld + sidx];
}
__global__ void scatter_state_kernel(double* q, double* qd, int64_t ld, const int64_t* perm, int64_t n,
                                     const double* qi, const double* qdi) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n * 12) return;
  const int64_t b = i / 12, c = i % 12;
  const int64_t sidx = perm[b];
  if (qi) q[c * ld + sidx] = qi[i];
  if (qdi) qd[c * ld + sidx] = qdi[i];
}

cudaError_t launch_gather(const double* q, const double* qd, int64_t ld, const int64_t* perm, int64_t n, double* qo,
                          double* qdo, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  const int64_t tot = n * 12;
  gather_state_kernel<<<(unsigned)((tot + 255) / 256), 256, 0, st>>>(q, qd, ld, perm, n, qo, qdo);
  return cudaGetLastError();
}
cudaError_t launch_scatter(double* q, double* qd, int64_t ld, const int64_t* perm, int64_t n, const double* qi,
                           const double* qdi, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  const int64_t tot = n * 12;
  scatter_state_kernel<<<(unsigned)((tot + 255) / 256), 256, 0, st>>>(q, qd, ld, perm, n, qi, qdi);
  return cudaGetLastError();
}

}  // namespace mabd
