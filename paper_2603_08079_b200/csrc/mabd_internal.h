// Internal data layout shared by the host runtime (mabd_host.cu) and the kernels. Not part of the ABI.
#pragma once
#include <cstdint>

namespace mabd {

// Per-material constants (central principal frame: M̄ = diag(a0, a1, a2, m); reading A8).
// Bodies that differ only by density share a material and carry a per-body mass scale.
struct Material {
  double a0, a1, a2, m;  // ∫ρx², ∫ρy², ∫ρz², ∫ρ  of the reference body
  double V, mu, lam;     // volume and Lamé parameters
  double pad;
};

// Closed-form H̄⁻¹ of one body (see hinv_blocks in mabd_device.cuh): G⁻¹ on (A00,A11,A22), three 2×2
// pair blocks on (A_rc, A_cr), r < c, and h²/m on t.
struct HinvBlk {
  double g[6];     // G⁻¹ packed sym
  double pr[3][3]; // pair k ∈ {(0,1),(0,2),(1,2)}: [p0 p1; p1 p2]
  double tinv;     // h²/m
};

// Slot encoding for the chain solver: a "slot" is the joint to the LEFT of a body position.
// bits 0-1: left side, bits 2-3: right side (SIDE_*), bits 4-31: geometry index.
enum : uint32_t { SIDE_NONE = 0, SIDE_BODY = 1, SIDE_WORLD = 2 };
__host__ __device__ inline uint32_t slot_left(uint32_t s) { return s & 3u; }
__host__ __device__ inline uint32_t slot_right(uint32_t s) { return (s >> 2) & 3u; }
__host__ __device__ inline uint32_t slot_geo(uint32_t s) { return s >> 4; }
__host__ __device__ inline bool slot_real(uint32_t s) { return slot_left(s) != SIDE_NONE && slot_right(s) != SIDE_NONE; }
__host__ __device__ inline uint32_t slot_pack(uint32_t l, uint32_t r, uint32_t g) { return l | (r << 2) | (g << 4); }

constexpr int SEG = 256;        // owned slots per segment
constexpr int CT = 128;         // threads per segment CTA (2 slots per thread)
constexpr int NEQ = SEG + 1;    // equations per segment CR (the 257th is the next segment's first slot)
constexpr int LDS = SEG + 2;    // shared-memory row stride of the CR arrays (even: 16-B aligned rows)
constexpr int SMALL_SLOTS = 32; // a one-window scene using at most this many slots takes the one-warp kernel

// Segment flags
enum : int32_t { SEG_LEFT_IFACE = 1, SEG_RIGHT_IFACE = 2, SEG_LONG = 4 };

// Reduced ("top") system of one segment after cyclic reduction of its interior: equations 0 and 256.
struct Top {
  double D0[6];   // sym
  double B[9];    // row-major coupling eq0 → eq256
  double D1[6];   // sym
  double r0[3];
  double r1[3];
};

// Device pointers for the body state and parameters (SoA, component stride ld).
struct BodyArrays {
  double* q;               // [12][ld]
  double* qd;              // [12][ld]
  double* rs;              // [9][ld] scratch: R between the phases of one launch (L2 only, discarded)
  double* z;               // [12][ld] K > 1 Newton iterations: q̇ⁿ + h[0;g] of this step
  const double* wr;        // [6][ld] external wrench (τ, f) per body, or null (mabd_set_wrench)
  int64_t ld;
  const int32_t* mat_id;   // [ld] or null (all material 0)
  const double* mscale;    // [ld] or null (all 1)
  const Material* mats;
};

struct StepConsts {
  double h, ih, ih2;
  double grav[3];          // gravity in the Newton r.h.s. (zero for iterations ≥ 1: q̂ carries it, see below)
  int32_t step_index;
  int32_t iter, niter;     // Newton iteration of this launch sequence, iterations per step
  int32_t lp;              // 1: polar-free variant (options.rotation = MABD_ROTATION_LENGTH_PRESERVING, DESIGN R9)
  int32_t phase;           // host side only: 0 whole step; host exchange: 1 up to the exchange, 2 after it
  int32_t* err;            // [0] flags (1 nonfinite, 2 singular), [1] first failing step
};

enum : int32_t { ERR_NONFINITE = 1, ERR_SINGULAR = 2 };

}  // namespace mabd
