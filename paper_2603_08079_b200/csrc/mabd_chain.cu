// Chain solver of the M-ABD step on sm_100a: fused per-segment kernel (stages 1-4) and the hierarchical
// block-tridiagonal reduced-system kernels for chains longer than one segment.
//
// Paper: the chain dual is block tridiagonal (Eq. chain-btd); the paper solves it with block
// Thomas in O(K) on one thread. Here one 128-thread CTA owns a 256-slot segment of a chain and
// solves its 257-equation block-tridiagonal system by block cyclic reduction in shared memory
// (log₂ 256 = 8 levels), fused with the per-body stages in one pass over HBM (details: chain_kernel below):
//   staging, by TMA: the segment's qⁿ, q̇ⁿ rows (cp.async.bulk, mbarrier) into the shared-memory CR rows;
//   phase 1, per body:  qⁿ, q̇ⁿ → tensor memory (TMEM, per-thread storage); polar R → f_A → δq̃ (stages 1-2,
//                       P:260-281); δq̃ and rows 0-1 of R stay in TMEM; per joint D, B, r = C(q̃) from the 3×3
//                       kernels P(ȳ,ȳ') rotated by R into the CR rows
//   phase 2, per segment: cyclic reduction → λ
//   phase 3, per body:  qⁿ, δq̃, R from TMEM, qⁿ⁺¹ = q̃ − diag₄(R)H̄⁻¹Σ±(ȳ_aug ⊗ Rᵀλ), q̇ⁿ⁺¹ = (qⁿ⁺¹ − qⁿ)/h
//                        → HBM
// Shared memory holds only the CR arrays (4 CTAs × 56.8 KB per SM); TMEM holds the per-body state across the solve.
// Chains spanning several segments are partitioned (SPIKE-style): each segment reduces its interior to a
// 2-equation "top" system on its end slots (REDUCE), the tops form a smaller block-tridiagonal system
// solved recursively by btd_kernel, and each segment then recomputes and back-substitutes (FINISH).
#include <cuda_runtime.h>

#include <algorithm>
#include <climits>

#include "mabd_device.cuh"
#include "mabd_kernels.h"

namespace mabd {

// ------------------------------------------------------------------ shared-memory cyclic reduction
// Equations k = 0..256:  Bl_k λ_{k−s} + D_k λ_k + Br_k λ_{k+s} = r_k at stride s, with Bl_k = Br_{k−s}ᵀ.
// Component-major arrays D[6][NEQ] (sym; replaced by D⁻¹ once eliminated), B[9][NEQ] (Br), Bl[9][NEQ]
// (saved Br_{k−s} of an eliminated k), r[3][NEQ] (rhs, then λ). Equation k lives at position cr_pos(k):
// the equations eliminated at stride 2^l are stored contiguously (level-major order), so every CR level
// reads and writes contiguous positions (no shared-memory bank conflicts).
struct CRS {
  double* D;
  double* B;
  double* Bl;
  double* r;
};

__device__ __forceinline__ int cr_pos(int k) {
  if (k == 0) return SEG - 1;
  if (k >= SEG) return SEG;
  const int l = __ffs(k) - 1;
  return (SEG - (SEG >> l)) + (k >> (l + 1));
}

// View of one equation's N components. Components are stored in pairs: components 2j, 2j+1 of the equation at
// position p form one 16-byte word of row-pair j (a row of 2·LDS doubles), an odd last component sits in a row of
// its own; so ldv/stv move a 3×3 block with 5 shared-memory accesses (LDS.128) instead of 9, and lanes that read
// consecutive positions stay conflict-free.
template <int N>
struct SV {
  double* p;  // group base + 2·pos (pairs)
  double* s;  // group base + (N/2)·2·LDS + pos (odd last component)
  __device__ __forceinline__ double& operator[](int e) const {
    return (N % 2 == 1 && e == N - 1) ? *s : p[(e >> 1) * 2 * LDS + (e & 1)];
  }
};
template <int N>
__device__ __forceinline__ SV<N> sview(double* g, int pos) {
  return SV<N>{g + 2 * pos, g + (N / 2) * 2 * LDS + pos};
}
__device__ __forceinline__ SV<6> eqD(const CRS& s, int pos) { return sview<6>(s.D, pos); }
__device__ __forceinline__ SV<9> eqB(const CRS& s, int pos) { return sview<9>(s.B, pos); }
__device__ __forceinline__ SV<9> eqBl(const CRS& s, int pos) { return sview<9>(s.Bl, pos); }
__device__ __forceinline__ SV<3> eqR(const CRS& s, int pos) { return sview<3>(s.r, pos); }
template <int N>
__device__ __forceinline__ void ldv(SV<N> v, double* x) {
#pragma unroll
  for (int j = 0; j < N / 2; ++j) {
    const double2 t = *reinterpret_cast<const double2*>(v.p + j * 2 * LDS);
    x[2 * j] = t.x;
    x[2 * j + 1] = t.y;
  }
  if (N % 2 == 1) x[N - 1] = *v.s;
}
template <int N>
__device__ __forceinline__ void stv(SV<N> v, const double* x) {
#pragma unroll
  for (int j = 0; j < N / 2; ++j) *reinterpret_cast<double2*>(v.p + j * 2 * LDS) = make_double2(x[2 * j], x[2 * j + 1]);
  if (N % 2 == 1) *v.s = x[N - 1];
}

#ifdef MABD_EXP_CLOCK
__device__ unsigned long long g_phase_clk[16];
#define PH_MARK(i)                                                        \
  do {                                                                    \
    if (threadIdx.x == 0) {                                               \
      const long long now = clock64();                                    \
      atomicAdd(&g_phase_clk[i], (unsigned long long)(now - ph_last));    \
      ph_last = now;                                                      \
    }                                                                     \
  } while (0)
extern "C" int mabd_dbg_phases(unsigned long long* out) {
  return (int)cudaMemcpyFromSymbol(out, g_phase_clk, sizeof(g_phase_clk));
}
extern "C" int mabd_dbg_reset() {
  unsigned long long z[16] = {0};
  return (int)cudaMemcpyToSymbol(g_phase_clk, z, sizeof(z));
}
#else
#define PH_MARK(i) \
  do {             \
  } while (0)
#endif

__device__ __forceinline__ void report(const StepConsts& k, int32_t flag) {
  atomicOr(k.err, flag);
  atomicMin(k.err + 1, k.step_index);
}

// invalidate one 128-byte L2 line without write-back (PTX discard.global.L2, sm_80+)
__device__ __forceinline__ void l2_discard128(const void* p) {
  asm volatile("discard.global.L2 [%0], 128;" ::"l"(p) : "memory");
}
__device__ __forceinline__ void l2_prefetch(const void* p) { asm volatile("prefetch.global.L2 [%0];" ::"l"(p)); }

// Position of the equation eliminated at level L (stride 2^L) with index e (equation 2^L·(2e+1)).
template <int L>
__device__ __forceinline__ int elim_pos(int e) { return (SEG - (SEG >> L)) + e; }
__device__ __forceinline__ int elim_pos_rt(int L, int e) { return (SEG - (SEG >> L)) + e; }

// update of the surviving equation kq = 2^{L+1}·m at stride ST = 2^L (both neighbours already hold D⁻¹).
// The level is a runtime argument: one copy of this code serves every level (instruction-cache footprint).
// inv: kq is eliminated at the next level, so its new D is inverted here (in registers, no reload)
// add: kq's equation still lacks its left body's part, parked in its Bl row (chain phase 1): added first
__device__ __forceinline__ void cr_update_rt(const CRS& s, int L, int m, bool inv = false,
                                             const StepConsts* ks = nullptr, bool add = false) {
  const int ST = 1 << L;
  const int kq = 2 * ST * m;
  const int pk = cr_pos(kq);
  double Ds[6], D[9], Br[9], r[3];
  ldv<6>(eqD(s, pk), Ds);
  ldv<9>(eqB(s, pk), Br);
  ldv<3>(eqR(s, pk), r);
  if (add) {
    double x[9];
    ldv<9>(eqBl(s, pk), x);
#pragma unroll
    for (int e = 0; e < 6; ++e) Ds[e] += x[e];
#pragma unroll
    for (int e = 0; e < 3; ++e) r[e] += x[6 + e];
  }
  full_from_sym(Ds, D);
  double nBr[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
  if (m > 0) {  // left neighbour i = kq − st:  α = Br_iᵀ D_i⁻¹;  D −= α Br_i;  r −= α r_i
    const int pi = elim_pos_rt(L, m - 1);
    double Dis[6], Di[9], Bi[9], al[9], ri[3], ar[3];
    ldv<6>(eqD(s, pi), Dis);
    full_from_sym(Dis, Di);
    ldv<9>(eqB(s, pi), Bi);
    mat3_mul_at(Bi, Di, al);
#pragma unroll
    for (int r0 = 0; r0 < 3; ++r0)
#pragma unroll
      for (int c = r0; c < 3; ++c) {  // α Br_i is symmetric: lower part only
        const double v = al[3 * r0] * Bi[c] + al[3 * r0 + 1] * Bi[3 + c] + al[3 * r0 + 2] * Bi[6 + c];
        D[3 * r0 + c] -= v;
        if (c != r0) D[3 * c + r0] -= v;
      }
    ldv<3>(eqR(s, pi), ri);
    mat3_vec(al, ri, ar);
#pragma unroll
    for (int e = 0; e < 3; ++e) r[e] -= ar[e];
  }
  if (kq < SEG) {  // right neighbour j = kq + st:  γ = Br_k D_j⁻¹;  D −= γ Br_kᵀ;  r −= γ r_j;  Br_k ← −γ Br_j
    const int pj = elim_pos_rt(L, m);
    double Djs[6], Dj[9], ga[9], tmp[9], Bj[9], rj[3], gr[3];
    ldv<6>(eqD(s, pj), Djs);
    full_from_sym(Djs, Dj);
    mat3_mul(Br, Dj, ga);
#pragma unroll
    for (int r0 = 0; r0 < 3; ++r0)
#pragma unroll
      for (int c = r0; c < 3; ++c) {
        const double v = ga[3 * r0] * Br[3 * c] + ga[3 * r0 + 1] * Br[3 * c + 1] + ga[3 * r0 + 2] * Br[3 * c + 2];
        D[3 * r0 + c] -= v;
        if (c != r0) D[3 * c + r0] -= v;
      }
    ldv<3>(eqR(s, pj), rj);
    mat3_vec(ga, rj, gr);
#pragma unroll
    for (int e = 0; e < 3; ++e) r[e] -= gr[e];
    ldv<9>(eqB(s, pj), Bj);
    mat3_mul(ga, Bj, tmp);
#pragma unroll
    for (int e = 0; e < 9; ++e) nBr[e] = -tmp[e];
    stv<9>(eqBl(s, pj), Br);  // j's left coupling at this level (Bl_j = Br_kᵀ), kept for back substitution
  }
  const double Dn[6] = {D[0], D[1], D[2], D[4], D[5], D[8]};
  if (inv) {
    double Di[6];
    if (!sym_inv_spd(Dn, Di)) report(*ks, ERR_SINGULAR);
    stv<6>(eqD(s, pk), Di);
  } else {
    stv<6>(eqD(s, pk), Dn);
  }
  stv<9>(eqB(s, pk), nBr);
  stv<3>(eqR(s, pk), r);
}

template <int L>
__device__ __forceinline__ void cr_update(const CRS& s, int m) {
  cr_update_rt(s, L, m);
}

__device__ __forceinline__ void cr_invert_at(const CRS& s, int p, const StepConsts& ks) {
  double Ds[6], Di[6];
  ldv<6>(eqD(s, p), Ds);
  if (!sym_inv_spd(Ds, Di)) report(ks, ERR_SINGULAR);
  stv<6>(eqD(s, p), Di);
}
__device__ __forceinline__ void cr_invert(const CRS& s, int k, const StepConsts& ks) { cr_invert_at(s, cr_pos(k), ks); }

// One forward level at stride 2^L over survivors m = first, first+step, …; a survivor that is eliminated at the
// next level (m odd) inverts its own D right after its update (no one else reads it at this level).
// With end = false the last survivor (equation SEG) is skipped: in a segment without a right interface it is the
// decoupled padding equation (identity, zero couplings at every level), so its updates are no-ops — and they
// would be a second, serial update for one lane.
__device__ __forceinline__ void cr_level_fwd_rt(const CRS& s, int L, int first, int step, const StepConsts& k,
                                                bool end = true) {
  const int NE = SEG >> (L + 1);
  const int last = end ? NE : NE - 1;
  for (int m = first; m <= last; m += step) {
    cr_update_rt(s, L, m, (m & 1) && (2 << L) < SEG, &k);
  }
}
template <int L>
__device__ __forceinline__ void cr_level_fwd(const CRS& s, int first, int step, const StepConsts& k,
                                             bool end = true) {
  cr_level_fwd_rt(s, L, first, step, k, end);
}

// Forward reduction, lower levels (strides 1, 2) by the whole CTA. Precondition: every odd equation already
// holds D⁻¹. One barrier per level.
template <int NT>
__device__ __forceinline__ void cr_forward_lower(const CRS& s, int t, const StepConsts& k, bool end = true) {
#pragma unroll 1
  for (int L = 0; L < 2; ++L) {  // one copy of the level code (instruction-cache footprint)
    cr_level_fwd_rt(s, L, t, NT, k, end);
    __syncthreads();
  }
}
// Upper levels (strides 4 … 128, ≤ 33 survivors) by one warp, warp-synchronous.
__device__ __forceinline__ void cr_forward_upper(const CRS& s, int lane, const StepConsts& k, bool end = true) {
#pragma unroll 1
  for (int L = 2; L <= 7; ++L) {
    cr_level_fwd_rt(s, L, lane, 32, k, end);
    __syncwarp();
  }
}
__device__ __forceinline__ void cr_forward(const CRS& s, int t, const StepConsts& k) {
  cr_forward_lower<CT>(s, t, k);
  if (t < 32) cr_forward_upper(s, t, k);
  __syncthreads();
}

// Solve the remaining 2-equation system [D0 B; Bᵀ D1][λ0; λ1] = [r0; r1] (one thread).
__device__ void cr_solve_top(const CRS& s, const StepConsts& k) {
  const int p0 = cr_pos(0), p1 = cr_pos(SEG);
  double D0s[6], D0i[6], D0[9], B[9], D1s[6], D1[9], r0[3], r1[3];
  ldv<9>(eqB(s, p0), B);
  ldv<3>(eqR(s, p0), r0);
  ldv<3>(eqR(s, p1), r1);
  ldv<6>(eqD(s, p0), D0s);
  ldv<6>(eqD(s, p1), D1s);
  if (!sym_inv_spd(D0s, D0i)) report(k, ERR_SINGULAR);
  full_from_sym(D0i, D0);
  full_from_sym(D1s, D1);
  double W[9], T[9];
  mat3_mul(D0, B, W);     // D0⁻¹ B
  mat3_mul_at(B, W, T);   // Bᵀ D0⁻¹ B
#pragma unroll
  for (int e = 0; e < 9; ++e) D1[e] -= T[e];
  double y[3], z[3];
  mat3_vec(D0, r0, y);
  mat3t_vec(B, y, z);
#pragma unroll
  for (int e = 0; e < 3; ++e) r1[e] -= z[e];
  D1s[0] = D1[0];
  D1s[1] = 0.5 * (D1[1] + D1[3]);
  D1s[2] = 0.5 * (D1[2] + D1[6]);
  D1s[3] = D1[4];
  D1s[4] = 0.5 * (D1[5] + D1[7]);
  D1s[5] = D1[8];
  double S1i[6], l1[3], l0[3], Bl1[3];
  if (!sym_inv_spd(D1s, S1i)) report(k, ERR_SINGULAR);
  sym_vec(S1i, r1, l1);
  mat3_vec(B, l1, Bl1);
#pragma unroll
  for (int e = 0; e < 3; ++e) r0[e] -= Bl1[e];
  mat3_vec(D0, r0, l0);
  stv<3>(eqR(s, p0), l0);
  stv<3>(eqR(s, p1), l1);
}

// Back substitution at stride 2^L: eliminated i = 2^L·(2m+1), m = first, first+step, … < NE.
__device__ __forceinline__ void cr_bwd_one(const CRS& s, int L, int m) {
  const int ST = 1 << L;
  const int i = ST * (2 * m + 1);
  const int pi = elim_pos_rt(L, m);
  double Bl[9], Br[9], Di[6], ll[3], lr[3], v[3], w[3];
  ldv<9>(eqBl(s, pi), Bl);
  ldv<9>(eqB(s, pi), Br);
  ldv<6>(eqD(s, pi), Di);
  ldv<3>(eqR(s, cr_pos(i - ST)), ll);
  ldv<3>(eqR(s, cr_pos(i + ST)), lr);
  ldv<3>(eqR(s, pi), v);
  mat3t_vec(Bl, ll, w);  // Bl_i λ_{i−s} = Br_{i−s}ᵀ λ_{i−s}
#pragma unroll
  for (int e = 0; e < 3; ++e) v[e] -= w[e];
  mat3_vec(Br, lr, w);
#pragma unroll
  for (int e = 0; e < 3; ++e) v[e] -= w[e];
  sym_vec(Di, v, w);
  stv<3>(eqR(s, pi), w);
}
__device__ __forceinline__ void cr_level_bwd_rt(const CRS& s, int L, int first, int step) {
  const int NE = SEG >> (L + 1);
  for (int m = first; m < NE; m += step) cr_bwd_one(s, L, m);
}
template <int L>
__device__ __forceinline__ void cr_level_bwd(const CRS& s, int first, int step) {
  cr_level_bwd_rt(s, L, first, step);
}
// λ of equations 0 and 256 are in r on entry, all λ on exit. Upper levels by one warp, then the CTA.
__device__ __forceinline__ void cr_backward_upper(const CRS& s, int lane) {
#pragma unroll 1
  for (int L = 7; L >= 2; --L) {
    cr_level_bwd_rt(s, L, lane, 32);
    __syncwarp();
  }
}
template <int NT>
__device__ __forceinline__ void cr_backward_lower(const CRS& s, int t) {
#pragma unroll 1
  for (int L = 1; L >= 0; --L) {
    cr_level_bwd_rt(s, L, t, NT);
    __syncthreads();
  }
}
__device__ __forceinline__ void cr_backward(const CRS& s, int t) {
  if (t < 32) cr_backward_upper(s, t);
  __syncthreads();
  cr_backward_lower<CT>(s, t);
}

__device__ __forceinline__ CRS cr_smem(double* smem) {
  CRS s;
  s.D = smem;
  s.B = s.D + LDS * 6;
  s.Bl = s.B + LDS * 9;
  s.r = s.Bl + LDS * 9;
  return s;
}

__device__ __forceinline__ void write_top(const CRS& s, Top* o) {
  const int p0 = cr_pos(0), p1 = cr_pos(SEG);
  ldv<6>(eqD(s, p0), o->D0);
  ldv<6>(eqD(s, p1), o->D1);
  ldv<9>(eqB(s, p0), o->B);
  ldv<3>(eqR(s, p0), o->r0);
  ldv<3>(eqR(s, p1), o->r1);
}

// ------------------------------------------------------------------ the fused chain segment kernel
// Persistent: each 128-thread CTA (4 per SM) loops over segments it ← blockIdx.x, += gridDim.x; thread t owns
// slots t and t+128 (the bodies at those positions and the joints to their left).
//   staging:  the segment's qⁿ, q̇ⁿ rows (24 × 2 KB) arrive by TMA bulk copies (cp.async.bulk, completion on an
//             mbarrier) into the CR rows D/B/Bl, its slot-code / mass-scale / material rows into the CR rows r;
//             all of them are dead while the previous segment finishes phase 3. No L2 round trip of the state
//             is on the critical path.
//   phase 1:  each thread moves its two bodies' qⁿ, q̇ⁿ into tensor memory (TMEM, 120 of the CTA's 128 columns,
//             its own lane), barrier (the CR rows are free), then per body: predict (stages 1-2) with δq̃ kept
//             in TMEM over q̇ⁿ and R's first two rows beside it, and assemble the joint equations (stage 3). TMEM is used purely as per-thread
//             storage (12-cycle loads): it carries qⁿ, δq̃ and R across the solve without registers, shared or
//             global memory, so shared memory holds only the CR arrays and 4 CTAs fit per SM.
//   phase 2:  block cyclic reduction (stage 3 solve)
//   phase 3:  per body: R from TMEM (rows 0, 1 stored in phase 1; row 2 = row 0 × row 1), λ from the CR rows,
//             qⁿ⁺¹ = q̃ − diag₄(R)H̄⁻¹Σ±Γᵀ Rᵀλ, q̇ⁿ⁺¹ = δq/h → HBM; then a barrier and the next segment's staging.
// FINISH = false: first pass (fused segments solve completely; long segments REDUCE to their top);
// FINISH = true: second pass of long segments (recompute, read the ends' λ, back-substitute, update).
constexpr int SLOT_ROW = SEG + 4;    // staged slot codes per segment (257 used, padded to 16 B)
constexpr int TMEM_COLS = 128;       // per CTA: 2 bodies × (24 words qⁿ + 24 words q̇ⁿ/δq̃ + 12 words R rows 0-1)

__host__ __device__ constexpr size_t chain_smem_size() { return sizeof(double) * LDS * 27 + 16; }

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* bar) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(bar)));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// TMEM as per-thread storage: 8 doubles (16 columns) of this thread's lane per call, warp-collective.
__device__ __forceinline__ void tm_st8(uint32_t taddr, const double* v) {
  uint32_t w[16];
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const unsigned long long b = (unsigned long long)__double_as_longlong(v[i]);
    w[2 * i] = (uint32_t)b;
    w[2 * i + 1] = (uint32_t)(b >> 32);
  }
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
      "%15, %16};" ::"r"(taddr),
      "r"(w[0]), "r"(w[1]), "r"(w[2]), "r"(w[3]), "r"(w[4]), "r"(w[5]), "r"(w[6]), "r"(w[7]), "r"(w[8]), "r"(w[9]),
      "r"(w[10]), "r"(w[11]), "r"(w[12]), "r"(w[13]), "r"(w[14]), "r"(w[15])
      : "memory");
}
__device__ __forceinline__ void tm_ld8(uint32_t taddr, double* v) {
  uint32_t w[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
      "%15}, [%16];"
      : "=r"(w[0]), "=r"(w[1]), "=r"(w[2]), "=r"(w[3]), "=r"(w[4]), "=r"(w[5]), "=r"(w[6]), "=r"(w[7]), "=r"(w[8]),
        "=r"(w[9]), "=r"(w[10]), "=r"(w[11]), "=r"(w[12]), "=r"(w[13]), "=r"(w[14]), "=r"(w[15])
      : "r"(taddr)
      : "memory");
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 8; ++i)
    v[i] = __longlong_as_double((long long)(((unsigned long long)w[2 * i + 1] << 32) | w[2 * i]));
}
// 4 doubles (8 columns) and 2 doubles (4 columns)
__device__ __forceinline__ void tm_st4(uint32_t taddr, const double* v) {
  uint32_t w[8];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const unsigned long long b = (unsigned long long)__double_as_longlong(v[i]);
    w[2 * i] = (uint32_t)b;
    w[2 * i + 1] = (uint32_t)(b >> 32);
  }
  asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"r"(taddr),
               "r"(w[0]), "r"(w[1]), "r"(w[2]), "r"(w[3]), "r"(w[4]), "r"(w[5]), "r"(w[6]), "r"(w[7])
               : "memory");
}
__device__ __forceinline__ void tm_ld4(uint32_t taddr, double* v) {
  uint32_t w[8];
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
               : "=r"(w[0]), "=r"(w[1]), "=r"(w[2]), "=r"(w[3]), "=r"(w[4]), "=r"(w[5]), "=r"(w[6]), "=r"(w[7])
               : "r"(taddr)
               : "memory");
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 4; ++i)
    v[i] = __longlong_as_double((long long)(((unsigned long long)w[2 * i + 1] << 32) | w[2 * i]));
}
__device__ __forceinline__ void tm_st2(uint32_t taddr, const double* v) {
  uint32_t w[4];
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    const unsigned long long b = (unsigned long long)__double_as_longlong(v[i]);
    w[2 * i] = (uint32_t)b;
    w[2 * i + 1] = (uint32_t)(b >> 32);
  }
  asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1, %2, %3, %4};" ::"r"(taddr), "r"(w[0]), "r"(w[1]),
               "r"(w[2]), "r"(w[3])
               : "memory");
}
__device__ __forceinline__ void tm_ld2(uint32_t taddr, double* v) {
  uint32_t w[4];
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0, %1, %2, %3}, [%4];"
               : "=r"(w[0]), "=r"(w[1]), "=r"(w[2]), "=r"(w[3])
               : "r"(taddr)
               : "memory");
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 2; ++i)
    v[i] = __longlong_as_double((long long)(((unsigned long long)w[2 * i + 1] << 32) | w[2 * i]));
}
// 12 doubles = exactly columns c0 … c0+23
__device__ __forceinline__ void tm_st12(uint32_t taddr, const double* v) {
  tm_st8(taddr, v);
  tm_st4(taddr + 16, v + 8);
}
__device__ __forceinline__ void tm_ld12(uint32_t taddr, double* v) {
  tm_ld8(taddr, v);
  tm_ld4(taddr + 16, v + 8);
}
// 6 doubles = columns c0 … c0+11
__device__ __forceinline__ void tm_st6(uint32_t taddr, const double* v) {
  tm_st4(taddr, v);
  tm_st2(taddr + 8, v + 4);
}
__device__ __forceinline__ void tm_ld6(uint32_t taddr, double* v) {
  tm_ld4(taddr, v);
  tm_ld2(taddr + 8, v + 4);
}
__device__ __forceinline__ void tm_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

// Thread 0: stage segment `it` and arm the mbarrier; the caller has made every earlier read of the CR rows
// happen-before (barrier).
__device__ __forceinline__ void stage_segment(const ChainArgs& a, double* cr, uint64_t* bar, int it) {
  if (it >= a.n_items) return;
  const int g = a.seg_list ? a.seg_list[it] : it;
  const int64_t base = (int64_t)g * SEG;
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic-proxy accesses before async writes
  uint32_t bytes = 24 * SEG * sizeof(double) + SLOT_ROW * sizeof(uint32_t);
  if (a.b.mscale) bytes += SEG * sizeof(double);
  if (a.b.mat_id) bytes += SEG * sizeof(int32_t);
  mbar_expect_tx(bar, bytes);
  for (int r = 0; r < 12; ++r) {
    bulk_g2s(cr + r * LDS, a.b.q + r * a.b.ld + base, SEG * sizeof(double), bar);
    bulk_g2s(cr + (12 + r) * LDS, a.b.qd + r * a.b.ld + base, SEG * sizeof(double), bar);
  }
  bulk_g2s(cr + 24 * LDS, a.slot_info + base, SLOT_ROW * sizeof(uint32_t), bar);
  if (a.b.mscale) bulk_g2s(cr + 25 * LDS, a.b.mscale + base, SEG * sizeof(double), bar);
  if (a.b.mat_id) bulk_g2s(cr + 26 * LDS, a.b.mat_id + base, SEG * sizeof(int32_t), bar);
}

__device__ __forceinline__ void get_hinv(const ChainArgs& a, const Material& M, int mid, double msc, HinvBlk& H) {
  if (a.hinv_tab)
    H = a.hinv_tab[mid];
  else
    hinv_blocks(M, msc, a.k.ih2, H);
}

#ifndef MABD_CHAIN_CTAS
#define MABD_CHAIN_CTAS 4  // CTAs per SM (shared memory: 4 × 56.8 KB; TMEM: 4 × 128 columns)
#endif
// WRENCH: external wrenches are set (a.b.wr != nullptr); the common no-wrench instance carries no wrench code
// LP: polar-free variant (R9): R := A; phase 3 takes A from the qⁿ parked in TMEM
template <bool FINISH, bool WRENCH, bool LP>
__global__ void __launch_bounds__(CT, MABD_CHAIN_CTAS) chain_kernel(ChainArgs a) {
  extern __shared__ __align__(16) double smem[];
  const CRS s = cr_smem(smem);
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + LDS * 27);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bar + 1);
  const int tid = threadIdx.x, warp = tid >> 5;
  const StepConsts& k = a.k;
  if (warp == 0) {  // TMEM: 128 columns for this CTA
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "n"(TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    mbar_init(bar);
    stage_segment(a, smem, bar, blockIdx.x);
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tbase = *tmem_slot + ((uint32_t)(32 * warp) << 16);  // this warp's lane quarter
  uint32_t phase = 0;
#ifdef MABD_EXP_CLOCK
  long long ph_last = clock64();
#endif
  for (int it = blockIdx.x; it < a.n_items; it += gridDim.x) {
    PH_MARK(7);
    const int g = a.seg_list ? a.seg_list[it] : it;
    const int flags = a.seg_flags[g];
    const bool is_long = (flags & SEG_LONG) != 0;
    const bool update = !is_long || FINISH;  // this pass writes the new state
    const bool reduce_only = is_long && !FINISH;
    const int64_t base = (int64_t)g * SEG;
    while (!mbar_try_wait(bar, phase)) {
    }
    phase ^= 1;
    PH_MARK(12);

    // ---------------- phase 1a: staged rows → registers (slot codes, mass scale, material) and TMEM (qⁿ, q̇ⁿ)
    // per-slot scalars of the two bodies as separate registers (a runtime-indexed array would go to local memory)
    uint32_t info0, info1, infoN0, infoN1;
    double msc0, msc1;
    int mid0, mid1;
    {
      const uint32_t* sinfo = reinterpret_cast<const uint32_t*>(smem + 24 * LDS);
      const int32_t* smid = reinterpret_cast<const int32_t*>(smem + 26 * LDS);
      const int t0 = 2 * tid;  // this thread's slots t0, t0 + 1 (adjacent: one 16-byte word per staged row)
      info0 = sinfo[t0];
      infoN0 = sinfo[t0 + 1];
      info1 = infoN0;
      infoN1 = sinfo[t0 + 2];
      if (a.b.mscale) {
        const double2 m2 = *reinterpret_cast<const double2*>(smem + 25 * LDS + t0);
        msc0 = m2.x;
        msc1 = m2.y;
      } else {
        msc0 = msc1 = 1.0;
      }
      if (a.b.mat_id) {
        const int2 i2 = *reinterpret_cast<const int2*>(smid + t0);
        mid0 = i2.x;
        mid1 = i2.y;
      } else {
        mid0 = mid1 = 0;
      }
#pragma unroll
      for (int h = 0; h < 2; ++h) {  // qⁿ rows, then q̇ⁿ rows
        double v0[12], v1[12];
#pragma unroll
        for (int r = 0; r < 12; ++r) {
          const double2 w = *reinterpret_cast<const double2*>(smem + (12 * h + r) * LDS + t0);
          v0[r] = w.x;
          v1[r] = w.y;
        }
        tm_st12(tbase + 24 * h, v0);
        tm_st12(tbase + 48 + 24 * h, v1);
      }
    }
    tm_wait_st();
    __syncthreads();  // the staged rows are consumed: the CR rows take the equations
    PH_MARK(13);

    // ---------------- phase 1b: per body predict + joint contributions
    // Equation t is assembled in place: D part of body t, rhs part, B_t; body t's contribution to equation
    // t+1 goes to the scratch row Bl[t+1]. The odd equation t0 + 1 has both bodies in this thread: it is completed
    // and inverted here; the even one t0 takes the left neighbour's part after the barrier.
#pragma unroll 1
    for (int b = 0; b < 2; ++b) {
      const int t = 2 * tid + b;
      const uint32_t inf = b ? info1 : info0, infN = b ? infoN1 : infoN0;
      const double msb = b ? msc1 : msc0;
      const int mdb = b ? mid1 : mid0;
      const bool has_body = slot_right(inf) == SIDE_BODY;
      const bool eq_real = slot_real(inf);
      const bool right_real = slot_real(infN) && slot_left(infN) == SIDE_BODY;
      const int pt = cr_pos(t);
      const auto sd = eqD(s, pt);
      const auto sr = eqR(s, pt);
      const auto sb = eqB(s, pt);
      const auto sx = eqBl(s, cr_pos(t + 1));  // scratch row: body t's contribution to equation t+1
      {
        const double one = eq_real ? 0.0 : 1.0;  // not a constraint: decoupled identity equation, λ = 0
        sd[0] = one; sd[1] = 0; sd[2] = 0; sd[3] = one; sd[4] = 0; sd[5] = one;
        double rr[3] = {0, 0, 0};
        if (eq_real) {
          const double* gp = a.geo + 6 * (size_t)slot_geo(inf);
          if (slot_left(inf) == SIDE_WORLD)  // start anchor: +p_world
#pragma unroll
            for (int e = 0; e < 3; ++e) rr[e] = __ldg(gp + e);
          if (slot_right(inf) == SIDE_WORLD)  // end anchor: −p_world
#pragma unroll
            for (int e = 0; e < 3; ++e) rr[e] -= __ldg(gp + 3 + e);
        }
#pragma unroll
        for (int e = 0; e < 3; ++e) sr[e] = rr[e];
#pragma unroll
        for (int e = 0; e < 9; ++e) sb[e] = 0.0;
#pragma unroll
        for (int e = 0; e < 9; ++e) sx[e] = 0.0;
      }
      // every lane runs the predict (warp-collective TMEM loads inside); slots without a body use A = I
      double q[12], dqt[12], R[9];
      HinvBlk H;
      {
        tm_ld12(tbase + 48 * b, q);
        if (!has_body) {
#pragma unroll
          for (int r = 0; r < 12; ++r) q[r] = (r == 0 || r == 4 || r == 8) ? 1.0 : 0.0;
        }
        const Material M = a.b.mats[mdb];
        const double ms = msb;
        const int md = mdb;
        double W[9];
        const bool ok = predict_body_lazy<LP>(
            q, [&](double* o) { tm_ld12(tbase + 48 * b + 24, o); }, M, ms,
            [&](HinvBlk& o) { get_hinv(a, M, md, ms, o); }, H, k.ih, k.grav, R, dqt,
            WRENCH ? load_wrench(a.b, base + t, W) : nullptr);
        if (!ok && has_body) report(k, ERR_NONFINITE);
      }
      if (update) {
        tm_st12(tbase + 48 * b + 24, dqt);  // δq̃ over q̇ⁿ (warp-collective: every lane)
        tm_st6(tbase + 96 + 12 * b, R);     // rows 0, 1 of R (row 2 = row 0 × row 1 in phase 3)
      }
      if (has_body) {
#pragma unroll
        for (int r = 0; r < 12; ++r) q[r] += dqt[r];  // q̃
        double y[3], x[3];
        if (eq_real) {  // joint to the left: this body is its right side (sign −): r_t −= x(q̃; ȳ_R)
          const double* gp = a.geo + 6 * (size_t)slot_geo(inf);
#pragma unroll
          for (int e = 0; e < 3; ++e) y[e] = __ldg(gp + 3 + e);
          point_pos(q, y, x);
#pragma unroll
          for (int e = 0; e < 3; ++e) sr[e] -= x[e];
        }
        if (right_real) {  // joint to the right: this body is its left side (sign +): r_{t+1} += x(q̃; ȳ_L)
          const double* gp = a.geo + 6 * (size_t)slot_geo(infN);
#pragma unroll
          for (int e = 0; e < 3; ++e) y[e] = __ldg(gp + e);
          point_pos(q, y, x);
#pragma unroll
          for (int e = 0; e < 3; ++e) sx[6 + e] = x[e];
        }
        double P[9], F[6], yR[3] = {0, 0, 0}, yL[3] = {0, 0, 0};
        if (eq_real) {
          const double* gp = a.geo + 6 * (size_t)slot_geo(inf);
#pragma unroll
          for (int e = 0; e < 3; ++e) yR[e] = __ldg(gp + 3 + e);
        }
        if (right_real) {
          const double* gp = a.geo + 6 * (size_t)slot_geo(infN);
#pragma unroll
          for (int e = 0; e < 3; ++e) yL[e] = __ldg(gp + e);
        }
        const int ax = LP ? -1 : common_axis(point_axis(yR), point_axis(yL));
        if (ax >= 0) {  // both points on one principal axis (R18): every block is tinv I + s R Q_k Rᵀ
          double Mq[6];
          axis_kernel_rot(H, R, ax, Mq);
          const double yr = yR[0] + yR[1] + yR[2], yl = yL[0] + yL[1] + yL[2];  // the on-axis components
          const double ti = H.tinv;
          if (eq_real) {
            const double s2 = yr * yr;
            sd[0] = fma(s2, Mq[0], ti); sd[1] = s2 * Mq[1]; sd[2] = s2 * Mq[2];
            sd[3] = fma(s2, Mq[3], ti); sd[4] = s2 * Mq[4]; sd[5] = fma(s2, Mq[5], ti);
          }
          if (right_real) {
            const double s2 = yl * yl;
            sx[0] = fma(s2, Mq[0], ti); sx[1] = s2 * Mq[1]; sx[2] = s2 * Mq[2];
            sx[3] = fma(s2, Mq[3], ti); sx[4] = s2 * Mq[4]; sx[5] = fma(s2, Mq[5], ti);
            if (eq_real) {  // B_t = −R P(ȳ_R, ȳ_L') Rᵀ (symmetric here)
              const double s = -(yr * yl);
              const double b0 = fma(s, Mq[0], -ti), b1 = s * Mq[1], b2 = s * Mq[2];
              const double b3 = fma(s, Mq[3], -ti), b4 = s * Mq[4], b5 = fma(s, Mq[5], -ti);
              sb[0] = b0; sb[1] = b1; sb[2] = b2;
              sb[3] = b1; sb[4] = b3; sb[5] = b4;
              sb[6] = b2; sb[7] = b4; sb[8] = b5;
            }
          }
        } else {
          if (eq_real) {  // D_t += R P(ȳ_R, ȳ_R) Rᵀ
            pblock(H, yR, yR, P);
            rot_conj_sym(R, P, F);
#pragma unroll
            for (int e = 0; e < 6; ++e) sd[e] = F[e];
          }
          if (right_real) {  // D_{t+1} += R P(ȳ_L, ȳ_L) Rᵀ
            pblock(H, yL, yL, P);
            rot_conj_sym(R, P, F);
#pragma unroll
            for (int e = 0; e < 6; ++e) sx[e] = F[e];
            if (eq_real) {  // B_t = −R P(ȳ_R, ȳ_L') Rᵀ  (signs −·+)
              double Fb[9];
              pblock(H, yR, yL, P);
              rot_conj(R, P, Fb);
#pragma unroll
              for (int e = 0; e < 9; ++e) sb[e] = -Fb[e];
            }
          }
        }
      }
    }
    {  // equation t0 + 1 (odd: eliminated at stride 1): + body t0's part, then D⁻¹
      const int pt = cr_pos(2 * tid + 1);
      if (slot_real(info1) && slot_left(info1) == SIDE_BODY) {
        double x[9], D[6], r[3], Di[6];
        ldv<9>(eqBl(s, pt), x);
        ldv<6>(eqD(s, pt), D);
        ldv<3>(eqR(s, pt), r);
#pragma unroll
        for (int e = 0; e < 6; ++e) D[e] += x[e];
#pragma unroll
        for (int e = 0; e < 3; ++e) r[e] += x[6 + e];
        stv<3>(eqR(s, pt), r);
        if (!sym_inv_spd(D, Di)) report(k, ERR_SINGULAR);
        stv<6>(eqD(s, pt), Di);
      } else {
        cr_invert_at(s, pt, k);
      }
    }
    if (tid == CT - 1) {  // equation 256 (this thread's scratch): next segment's first slot (partial) or padding
      const bool real = (flags & SEG_RIGHT_IFACE) != 0;
      const auto x = eqBl(s, SEG);
      double D[6], r[3];
#pragma unroll
      for (int e = 0; e < 6; ++e) D[e] = real ? x[e] : ((e == 0 || e == 3 || e == 5) ? 1.0 : 0.0);
#pragma unroll
      for (int e = 0; e < 3; ++e) r[e] = real ? x[6 + e] : 0.0;
      const double Z[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
      stv<6>(eqD(s, SEG), D);
      stv<9>(eqB(s, SEG), Z);
      stv<3>(eqR(s, SEG), r);
    }
    tm_wait_st();
    PH_MARK(0);
    __syncthreads();
    PH_MARK(1);

    // ---------------- phase 2: block cyclic reduction
    PH_MARK(2);
#ifndef MABD_EXP_SKIP_CR
    const bool right_iface = (flags & SEG_RIGHT_IFACE) != 0;
    // stride 1: survivor 2·tid is this thread's even equation t0, completed here with its left neighbour's part
    // (equation 0's left body lies in the previous segment: its part of the interface equation is added by that
    // segment's REDUCE output); equation 256 (built above) is updated by thread 0 when it is an interface
    cr_update_rt(s, 0, tid, (tid & 1) != 0, &k, tid > 0 && slot_real(info0) && slot_left(info0) == SIDE_BODY);
    if (tid == 0 && right_iface) cr_update_rt(s, 0, SEG >> 1, false, &k);
    __syncthreads();
    cr_level_fwd_rt(s, 1, tid, CT, k, right_iface);
    __syncthreads();
    PH_MARK(8);
    if (tid < 32) {  // upper levels, the 2-equation top and the upper back substitution: warp 0 alone
      cr_forward_upper(s, tid, k, right_iface);
      PH_MARK(9);
      if (tid == 0) {
        if (!is_long) {
          cr_solve_top(s, k);
        } else if (!FINISH) {
          write_top(s, a.top_out + a.seg_red[g]);
        } else {
          const int u = a.seg_red[g];
#pragma unroll
          for (int e = 0; e < 3; ++e) {
            eqR(s, cr_pos(0))[e] = a.lam_in[3 * u + e];
            eqR(s, SEG)[e] = (flags & SEG_RIGHT_IFACE) ? a.lam_in[3 * (u + 1) + e] : 0.0;
          }
        }
      }
      __syncwarp();
      PH_MARK(10);
      if (!reduce_only) cr_backward_upper(s, tid);
      PH_MARK(11);
    }
    __syncthreads();
    PH_MARK(3);
    if (reduce_only) {  // REDUCE pass of a long segment: its top is written, nothing else to do
      if (tid == 0) stage_segment(a, smem, bar, it + gridDim.x);
      continue;
    }
    PH_MARK(4);
    // strides 2, 1 back; no barrier after stride 1: phase 3 of this thread reads λ of its own equations t0, t0 + 1
    // (the odd one solved just now by this thread) and of t0 + 2 (solved at a higher level)
    cr_level_bwd_rt(s, 1, tid, CT);
    __syncthreads();
    cr_level_bwd_rt(s, 0, tid, CT);
#else
    __syncthreads();
    if (reduce_only) {
      if (tid == 0) stage_segment(a, smem, bar, it + gridDim.x);
      continue;
    }
#endif
    PH_MARK(5);
    // ---------------- phase 3: qⁿ⁺¹ = q̃ − diag₄(R) H̄⁻¹ Σ ±Γ(ȳ)ᵀ Rᵀλ
#pragma unroll 1
    for (int b = 0; b < 2; ++b) {
      const int t = 2 * tid + b;
      const int64_t slot = base + t;
      const uint32_t inf = b ? info1 : info0, infN = b ? infoN1 : infoN0;
      const double msb = b ? msc1 : msc0;
      const int mdb = b ? mid1 : mid0;
      double lam[6];
#pragma unroll
      for (int e = 0; e < 3; ++e) {
        lam[e] = eqR(s, cr_pos(t))[e];
        lam[3 + e] = eqR(s, cr_pos(t + 1))[e];
      }
      const bool has_body = slot_right(inf) == SIDE_BODY;
      const bool eq_real = slot_real(inf);
      const bool right_real = slot_real(infN) && slot_left(infN) == SIDE_BODY;
      double R[9], u[12];
      if (LP) {  // R := A = mat(qⁿ[0:9])
        double qa[12];
        tm_ld12(tbase + 48 * b, qa);
#pragma unroll
        for (int r = 0; r < 3; ++r)
#pragma unroll
          for (int c = 0; c < 3; ++c) R[3 * r + c] = qa[3 * c + r];
      } else {
        tm_ld6(tbase + 96 + 12 * b, R);  // rows 0, 1 of phase 1's R; row 2 = row 0 × row 1 (det R = +1)
        R[6] = R[1] * R[5] - R[2] * R[4];
        R[7] = R[2] * R[3] - R[0] * R[5];
        R[8] = R[0] * R[4] - R[1] * R[3];
      }
      {
        double gq[12];
#pragma unroll
        for (int r = 0; r < 12; ++r) gq[r] = 0.0;
        double w[3], y[3];
        if (eq_real) {
          const double* gp = a.geo + 6 * (size_t)slot_geo(inf);
#pragma unroll
          for (int e = 0; e < 3; ++e) y[e] = __ldg(gp + 3 + e);
          mat3t_vec(R, lam, w);
          add_point_force(gq, y, w, -1.0);
        }
        if (right_real) {
          const double* gp = a.geo + 6 * (size_t)slot_geo(infN);
#pragma unroll
          for (int e = 0; e < 3; ++e) y[e] = __ldg(gp + e);
          mat3t_vec(R, lam + 3, w);
          add_point_force(gq, y, w, 1.0);
        }
        HinvBlk H;
        if (has_body) {
          const Material M = a.b.mats[mdb];
          get_hinv(a, M, mdb, msb, H);
          hinv_apply(H, gq, u);
        }
      }
      double q[12], dqt[12];
      tm_ld12(tbase + 48 * b, q);
      tm_ld12(tbase + 48 * b + 24, dqt);
      if (has_body) {
        double* qb = a.b.q + slot;
        double* qdb = a.b.qd + slot;
        double dq[12];  // δq = δq̃ − correction
#pragma unroll
        for (int kb = 0; kb < 4; ++kb) {
          double c3[3];
          mat3_vec(R, u + 3 * kb, c3);
#pragma unroll
          for (int e = 0; e < 3; ++e) dq[3 * kb + e] = dqt[3 * kb + e] - c3[e];
        }
        const bool pair = slot_right(info0) == SIDE_BODY && slot_right(info1) == SIDE_BODY;
        if (k.niter == 1 && pair && b == 0) {  // stash slot t0's results (dead CR rows, this thread's column)
#pragma unroll
          for (int r = 0; r < 12; ++r) {
            smem[r * LDS + t] = q[r] + dq[r];
            smem[(12 + r) * LDS + t] = dq[r] * k.ih;
          }
        } else if (k.niter == 1 && pair) {  // slots t0, t0 + 1 as one 16-byte store per row
#pragma unroll
          for (int r = 0; r < 12; ++r) {
            __stcs(reinterpret_cast<double2*>(qb - 1 + r * a.b.ld), make_double2(smem[r * LDS + t - 1], q[r] + dq[r]));
            __stcs(reinterpret_cast<double2*>(qdb - 1 + r * a.b.ld),
                   make_double2(smem[(12 + r) * LDS + t - 1], dq[r] * k.ih));
          }
        } else if (k.niter == 1) {  // uniform branch outside the store loops (no if-converted second path)
#pragma unroll
          for (int r = 0; r < 12; ++r) __stcs(qb + r * a.b.ld, q[r] + dq[r]);
#pragma unroll
          for (int r = 0; r < 12; ++r) __stcs(qdb + r * a.b.ld, dq[r] * k.ih);
        } else {
#pragma unroll
          for (int r = 0; r < 12; ++r) __stcs(qb + r * a.b.ld, q[r] + dq[r]);
          // K > 1: v ← v − δq/h + h·grav (launch_step in mabd_plan.cu)
#pragma unroll
          for (int r = 0; r < 12; ++r)
            qdb[r * a.b.ld] = qdb[r * a.b.ld] - dq[r] * k.ih + (r >= 9 ? k.h * k.grav[r - 9] : 0.0);
        }
      }
    }
    PH_MARK(6);
    __syncthreads();  // λ read: every CR row is dead, stage the next segment into them
    if (tid == 0) stage_segment(a, smem, bar, it + gridDim.x);
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(*tmem_slot), "n"(TMEM_COLS));
}

// ------------------------------------------------------------------ a small scene: one warp, block Thomas
// A scene whose chains fit the first 32 slots of one window (config 1: 8 bodies, 9 joints) is latency-bound in the
// 256-slot segment kernel (TMA staging, 8 CR levels and their barriers for 9 equations). Here one warp does it:
// lane t owns slot t (the body there and the joint to its left); the equations are assembled as in chain_kernel's
// phase 1 and solved by block Thomas over the real equations by lane 0; then phase 3 per lane.
__global__ void __launch_bounds__(32) small_chain_kernel(ChainArgs a) {
  __shared__ double sD[SMALL_SLOTS + 1][9], sB[SMALL_SLOTS + 1][9], sr[SMALL_SLOTS + 1][3], sx[SMALL_SLOTS + 1][9];
  const int t = threadIdx.x;
  const StepConsts& k = a.k;
  const uint32_t inf = a.slot_info[t], infN = a.slot_info[t + 1];
  const bool has_body = slot_right(inf) == SIDE_BODY;
  const bool eq_real = slot_real(inf);
  const bool right_real = slot_real(infN) && slot_left(infN) == SIDE_BODY;
  const int mid = a.b.mat_id ? a.b.mat_id[t] : 0;
  const double msc = a.b.mscale ? a.b.mscale[t] : 1.0;
  const Material M = a.b.mats[mid];
  double q[12], qd[12], R[9], dqt[12];
#pragma unroll
  for (int c = 0; c < 12; ++c) {  // unconditional loads (slot t < 32 ≤ ld), issued with the slot codes' loads
    q[c] = a.b.q[c * a.b.ld + t];
    qd[c] = a.b.qd[c * a.b.ld + t];
  }
  if (!has_body)
#pragma unroll
    for (int c = 0; c < 12; ++c) {
      q[c] = (c == 0 || c == 4 || c == 8) ? 1.0 : 0.0;
      qd[c] = 0.0;
    }
  HinvBlk H;
  if (a.hinv_tab)
    H = a.hinv_tab[mid];
  else
    hinv_blocks(M, msc, k.ih2, H);
  double W[9];
  const double* Wp = has_body ? load_wrench(a.b, t, W) : nullptr;
  // a.nsteps > 1 (step_end folded, one Newton iteration): the steps of one mabd_step call run here back to back, the
  // state staying in registers (config 1: one launch per call instead of one per step)
  const int nst = a.nsteps > 1 ? a.nsteps : 1;
#pragma unroll 1
  for (int st = 0; st < nst; ++st) {
  const bool ok = k.lp ? predict_body<true>(q, qd, M, msc, H, k.ih, k.grav, R, dqt, Wp)
                       : predict_body<false>(q, qd, M, msc, H, k.ih, k.grav, R, dqt, Wp);
  if (!ok && has_body) report(k, ERR_NONFINITE);
  // equation t (own part) and body t's part of equation t+1 (sx)
  double D[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0}, rr[3] = {0, 0, 0}, Bq[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
  double X[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
  if (!eq_real) D[0] = D[4] = D[8] = 1.0;
  if (eq_real) {
    const double* gp = a.geo + 6 * (size_t)slot_geo(inf);
    if (slot_left(inf) == SIDE_WORLD)
#pragma unroll
      for (int e = 0; e < 3; ++e) rr[e] = gp[e];
    if (slot_right(inf) == SIDE_WORLD)
#pragma unroll
      for (int e = 0; e < 3; ++e) rr[e] -= gp[3 + e];
  }
  if (has_body) {
    double qt[12], x[3], P[9], F[9];
#pragma unroll
    for (int c = 0; c < 12; ++c) qt[c] = q[c] + dqt[c];
    if (eq_real) {
      const double* yR = a.geo + 6 * (size_t)slot_geo(inf) + 3;
      point_pos(qt, yR, x);
#pragma unroll
      for (int e = 0; e < 3; ++e) rr[e] -= x[e];
      pblock(H, yR, yR, P);
      rot_conj(R, P, F);
#pragma unroll
      for (int e = 0; e < 9; ++e) D[e] += F[e];
    }
    if (right_real) {
      const double* yL = a.geo + 6 * (size_t)slot_geo(infN);
      point_pos(qt, yL, x);
#pragma unroll
      for (int e = 0; e < 3; ++e) X[6 + e] = x[e];
      pblock(H, yL, yL, P);
      rot_conj(R, P, F);
#pragma unroll
      for (int e = 0; e < 6; ++e) X[e] = 0.0;
      double Fs[6];
      sym_from_full(F, Fs);
#pragma unroll
      for (int e = 0; e < 6; ++e) X[e] = Fs[e];
      if (eq_real) {
        const double* yR = a.geo + 6 * (size_t)slot_geo(inf) + 3;
        pblock(H, yR, yL, P);
        rot_conj(R, P, F);
#pragma unroll
        for (int e = 0; e < 9; ++e) Bq[e] = -F[e];
      }
    }
  }
#pragma unroll
  for (int e = 0; e < 9; ++e) {
    sD[t][e] = D[e];
    sB[t][e] = Bq[e];
    sx[t + 1][e] = X[e];
  }
#pragma unroll
  for (int e = 0; e < 3; ++e) sr[t][e] = rr[e];
  const unsigned real = __ballot_sync(0xffffffffu, eq_real);
  __syncwarp();
  if (t > 0 && eq_real && slot_left(inf) == SIDE_BODY) {  // the left body's part of this equation
    double Xs[9];
    full_from_sym(&sx[t][0], Xs);
#pragma unroll
    for (int e = 0; e < 9; ++e) sD[t][e] += Xs[e];
#pragma unroll
    for (int e = 0; e < 3; ++e) sr[t][e] += sx[t][6 + e];
  }
  __syncwarp();
  const int ne = real ? 32 - __clz((int)real) : 0;  // equations 0 .. ne−1 (beyond: decoupled padding, λ = 0)
  if (t == 0) {  // block Thomas: D'_0 = D_0, L_k = B_{k−1}ᵀ D'_{k−1}⁻¹, D'_k = D_k − L_k B_{k−1}, y_k = r_k − L_k y_{k−1}
    double Dpi[9], y[3];
    for (int kq = 0; kq < ne; ++kq) {
      double Dk[9], Ds[6], Di[6];
#pragma unroll
      for (int e = 0; e < 9; ++e) Dk[e] = sD[kq][e];
      double yk[3] = {sr[kq][0], sr[kq][1], sr[kq][2]};
      if (kq > 0) {
        double Bp[9], L[9], T[9], v[3];
#pragma unroll
        for (int e = 0; e < 9; ++e) Bp[e] = sB[kq - 1][e];
        mat3_mul_at(Bp, Dpi, L);
        mat3_mul(L, Bp, T);
        mat3_vec(L, y, v);
#pragma unroll
        for (int e = 0; e < 9; ++e) Dk[e] -= T[e];
#pragma unroll
        for (int e = 0; e < 3; ++e) yk[e] -= v[e];
      }
      Ds[0] = Dk[0]; Ds[1] = 0.5 * (Dk[1] + Dk[3]); Ds[2] = 0.5 * (Dk[2] + Dk[6]);
      Ds[3] = Dk[4]; Ds[4] = 0.5 * (Dk[5] + Dk[7]); Ds[5] = Dk[8];
      if (!sym_inv_spd(Ds, Di)) report(k, ERR_SINGULAR);
      full_from_sym(Di, Dpi);
#pragma unroll
      for (int e = 0; e < 9; ++e) sD[kq][e] = Dpi[e];
#pragma unroll
      for (int e = 0; e < 3; ++e) sr[kq][e] = y[e] = yk[e];
    }
    double lam[3] = {0, 0, 0};
    for (int kq = ne - 1; kq >= 0; --kq) {  // λ_k = D'_k⁻¹ (y_k − B_k λ_{k+1})
      double Bk[9], Dk[9], v[3], w[3];
#pragma unroll
      for (int e = 0; e < 9; ++e) {
        Bk[e] = sB[kq][e];
        Dk[e] = sD[kq][e];
      }
      mat3_vec(Bk, lam, w);
#pragma unroll
      for (int e = 0; e < 3; ++e) v[e] = sr[kq][e] - (kq + 1 < ne ? w[e] : 0.0);
      mat3_vec(Dk, v, lam);
#pragma unroll
      for (int e = 0; e < 3; ++e) sr[kq][e] = lam[e];
    }
  }
  __syncwarp();
  if (a.step_end && t == 0) {  // the step_end node folded in (one CTA: every report of this step is above)
    __threadfence();
    int32_t* e = k.err;
    if (e[0] != 0 && e[2] == INT_MAX) e[2] = e[3];
    e[3] += 1;
  }
  if (has_body) {
  // phase 3: qⁿ⁺¹ = q̃ − diag₄(R) H̄⁻¹ Σ ±Γ(ȳ)ᵀ Rᵀλ
  double gq[12] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0}, w[3], lam[3], u[12];
  if (eq_real) {
#pragma unroll
    for (int e = 0; e < 3; ++e) lam[e] = t < ne ? sr[t][e] : 0.0;
    mat3t_vec(R, lam, w);
    add_point_force(gq, a.geo + 6 * (size_t)slot_geo(inf) + 3, w, -1.0);
  }
  if (right_real) {
#pragma unroll
    for (int e = 0; e < 3; ++e) lam[e] = t + 1 < ne ? sr[t + 1][e] : 0.0;
    mat3t_vec(R, lam, w);
    add_point_force(gq, a.geo + 6 * (size_t)slot_geo(infN), w, 1.0);
  }
  hinv_apply(H, gq, u);
  double dq[12];
#pragma unroll
  for (int kb = 0; kb < 4; ++kb) {
    double c3[3];
    mat3_vec(R, u + 3 * kb, c3);
#pragma unroll
    for (int e = 0; e < 3; ++e) dq[3 * kb + e] = dqt[3 * kb + e] - c3[e];
  }
#pragma unroll
  for (int c = 0; c < 12; ++c) {
    q[c] += dq[c];
    qd[c] = k.niter == 1 ? dq[c] * k.ih : qd[c] - dq[c] * k.ih + (c >= 9 ? k.h * k.grav[c - 9] : 0.0);
  }
  }
  __syncwarp();  // every lane has read this step's λ before the next step's equations overwrite them
  }
  if (!has_body) return;
#pragma unroll
  for (int c = 0; c < 12; ++c) {
    a.b.q[c * a.b.ld + t] = q[c];
    a.b.qd[c * a.b.ld + t] = qd[c];
  }
}

cudaError_t launch_small_chain(const ChainArgs& a, cudaStream_t st) {
  small_chain_kernel<<<1, 32, 0, st>>>(a);
  return cudaGetLastError();
}

// ------------------------------------------------------------------ reduced block-tridiagonal levels
// Unknown u of level L owns the equation built from the level-(L−1) tops:
//   D_u = top[u].D0 + (left(u) ? top[u−1].D1 : 0),  B_u = top[u].B,  r_u likewise.
// A window w of 256 unknowns is one CTA; its equation 256 is the first unknown of window w+1 (partial:
// D = 0, r = 0; its coupling from unknown 256w+255 is B_{256w+255}), or padding.
__global__ void __launch_bounds__(CT) btd_kernel(BtdArgs a) {
  extern __shared__ double smem[];
  const CRS s = cr_smem(smem);
  const int tid = threadIdx.x;
  const int64_t w = blockIdx.x;
  const int64_t nu = a.n_u;
  for (int b = 0; b < 2; ++b) {
    const int t = tid + b * CT;
    const int64_t u = w * SEG + t;
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
    const int pt = cr_pos(t);
    stv<6>(eqD(s, pt), D);
    stv<9>(eqB(s, pt), B);
    stv<3>(eqR(s, pt), r);
    if (t & 1) cr_invert(s, t, a.k);  // eliminated at stride 1
  }
  if (tid == CT - 1) {
    // equation 256: the next window's first unknown (partial, completed by that window), the next part's
    // first unknown (partial from this part's last unknown: its top D1, r1), or padding
    const bool real_next = (w + 1) * SEG < nu;
    const double Z[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
    if (!real_next && a.right_open) {
      stv<6>(eqD(s, SEG), a.top_in[nu - 1].D1);
      stv<3>(eqR(s, SEG), a.top_in[nu - 1].r1);
    } else {
      const double dv = real_next ? 0.0 : 1.0;
      const double Dn[6] = {dv, 0, 0, dv, 0, dv};
      stv<6>(eqD(s, SEG), Dn);
      stv<3>(eqR(s, SEG), Z);
    }
    stv<9>(eqB(s, SEG), Z);
  }
  __syncthreads();
  cr_forward(s, tid, a.k);
  if (a.mode == BTD_REDUCE) {
    if (tid == 0) write_top(s, a.top_out + w);
    return;
  }
  if (a.mode == BTD_FUSED) {
    if (tid == 0) cr_solve_top(s, a.k);
  } else if (tid == 0) {
    const bool real_next = (w + 1) * SEG < nu;
#pragma unroll
    for (int e = 0; e < 3; ++e) {
      eqR(s, cr_pos(0))[e] = a.lam_in[3 * w + e];
      eqR(s, SEG)[e] = real_next ? a.lam_in[3 * (w + 1) + e] : (a.right_open ? a.lam_remote[e] : 0.0);
    }
  }
  __syncthreads();
  cr_backward(s, tid);
  for (int b = 0; b < 2; ++b) {
    const int t = tid + b * CT;
    const int64_t u = w * SEG + t;
    if (u < nu) {
#pragma unroll
      for (int e = 0; e < 3; ++e) a.lam_out[3 * u + e] = eqR(s, cr_pos(t))[e];
    }
  }
}

// ------------------------------------------------------------------ multi-part chains: sequential part top
// A part (one rank's share of a long chain, or an emulated rank) reduces its n level unknowns u = 0..n−1 and
// the next part's first unknown ρ (partial, from this side) onto {0, ρ}: eliminate u = 1..n−1 in order,
// carrying the coupling X of equation 0 to the current frontier (block Thomas with a spike).
// n is small (≤ 256 by construction, typically ≤ 17), so one thread does it.
__device__ __forceinline__ void seq_eq(const SeqArgs& a, int u, double* D, double* r) {
  // equation u from the tops of the level below: D_u = top[u].D0 + top[u−1].D1 (u > 0), same for r;
  // u = n is the remote unknown ρ (partial: top[n−1].D1, r1 if right-open; else padding)
  const int n = a.n;
  if (u == n) {
    if (a.right_open) {
#pragma unroll
      for (int e = 0; e < 6; ++e) D[e] = a.top_in[n - 1].D1[e];
#pragma unroll
      for (int e = 0; e < 3; ++e) r[e] = a.top_in[n - 1].r1[e];
    } else {
      D[0] = 1; D[1] = 0; D[2] = 0; D[3] = 1; D[4] = 0; D[5] = 1;
      r[0] = r[1] = r[2] = 0;
    }
    return;
  }
#pragma unroll
  for (int e = 0; e < 6; ++e) D[e] = a.top_in[u].D0[e] + (u > 0 ? a.top_in[u - 1].D1[e] : 0.0);
#pragma unroll
  for (int e = 0; e < 3; ++e) r[e] = a.top_in[u].r0[e] + (u > 0 ? a.top_in[u - 1].r1[e] : 0.0);
}

__global__ void seq_top_kernel(SeqArgs a) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  const int n = a.n;
  double D0s[6], r0[3], X[9], Dks[6], rk[3];
  seq_eq(a, 0, D0s, r0);
#pragma unroll
  for (int e = 0; e < 9; ++e) X[e] = a.top_in[0].B[e];  // coupling 0 → 1 (or → ρ when n = 1)
  seq_eq(a, n == 1 ? 1 : 1, Dks, rk);
  for (int k = 1; k < n; ++k) {
    double Di[6], Dif[9], Bk[9];
    if (!sym_inv_spd(Dks, Di)) report(a.k, ERR_SINGULAR);
    full_from_sym(Di, Dif);
#pragma unroll
    for (int e = 0; e < 9; ++e) Bk[e] = a.top_in[k].B[e];  // k → k+1 (ρ when k = n−1)
    double* sc = a.scratch + 27 * (size_t)k;
#pragma unroll
    for (int e = 0; e < 6; ++e) sc[e] = Di[e];
#pragma unroll
    for (int e = 0; e < 9; ++e) { sc[6 + e] = X[e]; sc[15 + e] = Bk[e]; }
#pragma unroll
    for (int e = 0; e < 3; ++e) sc[24 + e] = rk[e];
    // eq 0:  D0 −= X D⁻¹ Xᵀ,  r0 −= X D⁻¹ r_k,  X ← −X D⁻¹ B_k
    double XD[9], T[9], v[3];
    mat3_mul(X, Dif, XD);
    mat3_mul_bt(XD, X, T);
    double D0f[9];
    full_from_sym(D0s, D0f);
#pragma unroll
    for (int e = 0; e < 9; ++e) D0f[e] -= T[e];
    D0s[0] = D0f[0]; D0s[1] = 0.5 * (D0f[1] + D0f[3]); D0s[2] = 0.5 * (D0f[2] + D0f[6]);
    D0s[3] = D0f[4]; D0s[4] = 0.5 * (D0f[5] + D0f[7]); D0s[5] = D0f[8];
    mat3_vec(XD, rk, v);
#pragma unroll
    for (int e = 0; e < 3; ++e) r0[e] -= v[e];
    double nX[9];
    mat3_mul(XD, Bk, nX);
#pragma unroll
    for (int e = 0; e < 9; ++e) X[e] = -nX[e];
    // eq k+1:  D −= B_kᵀ D⁻¹ B_k,  r −= B_kᵀ D⁻¹ r_k
    double Dn[6], rn[3], DB[9], BDB[9], Dnf[9], w[3], bw[3];
    seq_eq(a, k + 1, Dn, rn);
    mat3_mul(Dif, Bk, DB);
    mat3_mul_at(Bk, DB, BDB);
    full_from_sym(Dn, Dnf);
#pragma unroll
    for (int e = 0; e < 9; ++e) Dnf[e] -= BDB[e];
    Dks[0] = Dnf[0]; Dks[1] = 0.5 * (Dnf[1] + Dnf[3]); Dks[2] = 0.5 * (Dnf[2] + Dnf[6]);
    Dks[3] = Dnf[4]; Dks[4] = 0.5 * (Dnf[5] + Dnf[7]); Dks[5] = Dnf[8];
    mat3_vec(Dif, rk, w);
    mat3t_vec(Bk, w, bw);
#pragma unroll
    for (int e = 0; e < 3; ++e) rk[e] = rn[e] - bw[e];
  }
  Top* o = a.top_out;
#pragma unroll
  for (int e = 0; e < 6; ++e) { o->D0[e] = D0s[e]; o->D1[e] = Dks[e]; }
#pragma unroll
  for (int e = 0; e < 9; ++e) o->B[e] = X[e];
#pragma unroll
  for (int e = 0; e < 3; ++e) { o->r0[e] = r0[e]; o->r1[e] = rk[e]; }
}

__global__ void seq_finish_kernel(SeqArgs a) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  const int n = a.n;
  double l0[3], lnext[3];
#pragma unroll
  for (int e = 0; e < 3; ++e) {
    l0[e] = a.lam_ends[e];
    lnext[e] = a.right_open ? a.lam_ends[3 + e] : 0.0;
    a.lam_out[e] = l0[e];
  }
  for (int k = n - 1; k >= 1; --k) {  // λ_k = D'_k⁻¹ (r'_k − X_kᵀ λ_0 − B_k λ_{k+1})
    const double* sc = a.scratch + 27 * (size_t)k;
    double v[3], w[3];
#pragma unroll
    for (int e = 0; e < 3; ++e) v[e] = sc[24 + e];
    mat3t_vec(sc + 6, l0, w);
#pragma unroll
    for (int e = 0; e < 3; ++e) v[e] -= w[e];
    mat3_vec(sc + 15, lnext, w);
#pragma unroll
    for (int e = 0; e < 3; ++e) v[e] -= w[e];
    sym_vec(sc, v, w);
#pragma unroll
    for (int e = 0; e < 3; ++e) {
      a.lam_out[3 * k + e] = w[e];
      lnext[e] = w[e];
    }
  }
}

cudaError_t launch_seq_top(const SeqArgs& a, cudaStream_t st) {
  seq_top_kernel<<<1, 32, 0, st>>>(a);
  return cudaGetLastError();
}
cudaError_t launch_seq_finish(const SeqArgs& a, cudaStream_t st) {
  seq_finish_kernel<<<1, 32, 0, st>>>(a);
  return cudaGetLastError();
}

size_t cr_smem_bytes() { return sizeof(double) * LDS * (6 + 9 + 9 + 3); }
static size_t chain_smem_bytes() { return chain_smem_size(); }

static int g_num_sms = 0;

cudaError_t launch_chain(const ChainArgs& a0, int nitems, bool finish, cudaStream_t st) {
  if (nitems <= 0) return cudaSuccess;
  ChainArgs a = a0;
  a.n_items = nitems;
  const size_t sm = chain_smem_bytes();
  const int grid = std::min(nitems, MABD_CHAIN_CTAS * std::max(g_num_sms, 1));
  const bool w = a.b.wr != nullptr;
  if (a.k.lp) {
    if (finish)
      (w ? chain_kernel<true, true, true> : chain_kernel<true, false, true>)<<<grid, CT, sm, st>>>(a);
    else
      (w ? chain_kernel<false, true, true> : chain_kernel<false, false, true>)<<<grid, CT, sm, st>>>(a);
  } else {
    if (finish)
      (w ? chain_kernel<true, true, false> : chain_kernel<true, false, false>)<<<grid, CT, sm, st>>>(a);
    else
      (w ? chain_kernel<false, true, false> : chain_kernel<false, false, false>)<<<grid, CT, sm, st>>>(a);
  }
  return cudaGetLastError();
}

cudaError_t launch_btd(const BtdArgs& a, int nblocks, cudaStream_t st) {
  if (nblocks <= 0) return cudaSuccess;
  btd_kernel<<<nblocks, CT, cr_smem_bytes(), st>>>(a);
  return cudaGetLastError();
}

cudaError_t chain_kernels_init() {
  const int sm = (int)cr_smem_bytes();
  cudaError_t e;
  int dev = 0;
  if ((e = cudaGetDevice(&dev))) return e;
  if ((e = cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev))) return e;
  const int smc = (int)chain_smem_bytes();
  void (*const kernels[8])(ChainArgs) = {
      chain_kernel<true, false, false>, chain_kernel<false, false, false>, chain_kernel<true, true, false>,
      chain_kernel<false, true, false>, chain_kernel<true, false, true>,  chain_kernel<false, false, true>,
      chain_kernel<true, true, true>,   chain_kernel<false, true, true>};
  for (auto kf : kernels) {
    if ((e = cudaFuncSetAttribute(kf, cudaFuncAttributeMaxDynamicSharedMemorySize, smc))) return e;
    // favour shared memory in the unified L1/shared carve-out so that 4 segment CTAs fit per SM
    cudaFuncSetAttribute(kf, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
  }
  if ((e = cudaFuncSetAttribute(btd_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, sm))) return e;
  return cudaSuccess;
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

// state gather / scatter between the caller's AoS order and the internal SoA positions
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

// caller frame ↔ canonical frame (R8): q = (A'Q, t' − A o) out, q' = (A Qᵀ, t + A o) in; velocities alike
__device__ __forceinline__ void frame_out(const double* F, double* v) {
  double A[9];
#pragma unroll
  for (int e = 0; e < 9; ++e) A[e] = v[e];  // column-major A'
#pragma unroll
  for (int c = 0; c < 3; ++c)
#pragma unroll
    for (int r = 0; r < 3; ++r) v[3 * c + r] = A[r] * F[c] + A[3 + r] * F[3 + c] + A[6 + r] * F[6 + c];  // (A'Q)[r][c]
#pragma unroll
  for (int r = 0; r < 3; ++r) v[9 + r] -= v[r] * F[9] + v[3 + r] * F[10] + v[6 + r] * F[11];
}
__device__ __forceinline__ void frame_in(const double* F, double* v) {
  double A[9];
#pragma unroll
  for (int e = 0; e < 9; ++e) A[e] = v[e];
#pragma unroll
  for (int r = 0; r < 3; ++r) v[9 + r] += A[r] * F[9] + A[3 + r] * F[10] + A[6 + r] * F[11];
#pragma unroll
  for (int c = 0; c < 3; ++c)
#pragma unroll
    for (int r = 0; r < 3; ++r)
      v[3 * c + r] = A[r] * F[3 * c] + A[3 + r] * F[3 * c + 1] + A[6 + r] * F[3 * c + 2];  // (A Qᵀ)[r][c]
}
__global__ void gather_frames_kernel(const double* q, const double* qd, int64_t ld, const int64_t* perm, int64_t n,
                                     const double* frame, double* qo, double* qdo) {
  const int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (b >= n) return;
  const int64_t s = perm[b];
  double F[12], v[12];
#pragma unroll
  for (int e = 0; e < 12; ++e) F[e] = frame[12 * b + e];
  if (qo) {
#pragma unroll
    for (int e = 0; e < 12; ++e) v[e] = q[e * ld + s];
    frame_out(F, v);
#pragma unroll
    for (int e = 0; e < 12; ++e) qo[12 * b + e] = v[e];
  }
  if (qdo) {
#pragma unroll
    for (int e = 0; e < 12; ++e) v[e] = qd[e * ld + s];
    frame_out(F, v);
#pragma unroll
    for (int e = 0; e < 12; ++e) qdo[12 * b + e] = v[e];
  }
}
__global__ void scatter_frames_kernel(double* q, double* qd, int64_t ld, const int64_t* perm, int64_t n,
                                      const double* frame, const double* qi, const double* qdi) {
  const int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (b >= n) return;
  const int64_t s = perm[b];
  double F[12], v[12];
#pragma unroll
  for (int e = 0; e < 12; ++e) F[e] = frame[12 * b + e];
  if (qi) {
#pragma unroll
    for (int e = 0; e < 12; ++e) v[e] = qi[12 * b + e];
    frame_in(F, v);
#pragma unroll
    for (int e = 0; e < 12; ++e) q[e * ld + s] = v[e];
  }
  if (qdi) {
#pragma unroll
    for (int e = 0; e < 12; ++e) v[e] = qdi[12 * b + e];
    frame_in(F, v);
#pragma unroll
    for (int e = 0; e < 12; ++e) qd[e * ld + s] = v[e];
  }
}
// the wrench's force point in the canonical frame: ȳ_f = −Q o (the caller's frame origin), rows 6-8 of wr
__global__ void wrench_point_kernel(double* wr, int64_t ld, const int64_t* perm, int64_t n, const double* frame) {
  const int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (b >= n) return;
  const double* F = frame + 12 * b;
#pragma unroll
  for (int r = 0; r < 3; ++r) wr[(6 + r) * ld + perm[b]] = -(F[3 * r] * F[9] + F[3 * r + 1] * F[10] + F[3 * r + 2] * F[11]);
}

cudaError_t launch_wrench_point(double* wr, int64_t ld, const int64_t* perm, int64_t n, const double* frame,
                                cudaStream_t st) {
  if (n <= 0 || !frame) return cudaSuccess;
  wrench_point_kernel<<<(unsigned)((n + 127) / 128), 128, 0, st>>>(wr, ld, perm, n, frame);
  return cudaGetLastError();
}

cudaError_t launch_gather(const double* q, const double* qd, int64_t ld, const int64_t* perm, int64_t n,
                          const double* frame, double* qo, double* qdo, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  if (frame) {
    gather_frames_kernel<<<(unsigned)((n + 127) / 128), 128, 0, st>>>(q, qd, ld, perm, n, frame, qo, qdo);
    return cudaGetLastError();
  }
  const int64_t tot = n * 12;
  gather_state_kernel<<<(unsigned)((tot + 255) / 256), 256, 0, st>>>(q, qd, ld, perm, n, qo, qdo);
  return cudaGetLastError();
}
__global__ void scatter_rows_kernel(double* dst, int64_t ld, const int64_t* perm, int64_t n, const double* src, int nc) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n * nc) return;
  const int64_t b = i / nc, c = i % nc;
  dst[c * ld + perm[b]] = src[i];
}
cudaError_t launch_scatter_rows(double* dst, int64_t ld, const int64_t* perm, int64_t n, const double* src, int nc,
                                cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  scatter_rows_kernel<<<(unsigned)((n * nc + 255) / 256), 256, 0, st>>>(dst, ld, perm, n, src, nc);
  return cudaGetLastError();
}
cudaError_t launch_scatter(double* q, double* qd, int64_t ld, const int64_t* perm, int64_t n, const double* frame,
                           const double* qi, const double* qdi, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  if (frame) {
    scatter_frames_kernel<<<(unsigned)((n + 127) / 128), 128, 0, st>>>(q, qd, ld, perm, n, frame, qi, qdi);
    return cudaGetLastError();
  }
  const int64_t tot = n * 12;
  scatter_state_kernel<<<(unsigned)((tot + 255) / 256), 256, 0, st>>>(q, qd, ld, perm, n, qi, qdi);
  return cudaGetLastError();
}

}  // namespace mabd
