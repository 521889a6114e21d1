// Host-side analysis of a scene: validation, materials, topology classification, chain ordering, the
// hierarchical reduced-system plan and the device memory layout. Also the per-step launch sequence.
#include <cuda_runtime.h>

#include <algorithm>
#include <climits>
#include <cmath>
#include <cstring>
#include <functional>
#include <string>
#include <unordered_map>
#include <vector>

#include "mabd_plan.h"

namespace mabd {

namespace {

struct Key48 {
  uint64_t w[6];
  bool operator==(const Key48& o) const { return std::memcmp(w, o.w, sizeof(w)) == 0; }
};
struct Key48Hash {
  size_t operator()(const Key48& k) const {
    uint64_t h = 1469598103934665603ull;
    for (int i = 0; i < 6; ++i) {
      h ^= k.w[i] + 0x9e3779b97f4a7c15ull + (h << 6) + (h >> 2);
    }
    return (size_t)h;
  }
};
Key48 key_of(const double* v) {
  Key48 k;
  std::memcpy(k.w, v, sizeof(k.w));
  for (int i = 0; i < 6; ++i)
    if (v[i] == 0.0) k.w[i] = 0;  // +0 / −0
  return k;
}

std::string fmt(const char* f, long long a = 0, long long b = 0) {
  char buf[512];
  snprintf(buf, sizeof(buf), f, a, b);
  return buf;
}

size_t align_up(size_t x) { return (x + 255) & ~size_t(255); }

}  // namespace

// ------------------------------------------------------------------------------------------ body frames
// Packed M̄ (00,01,02,03,11,12,13,22,23,33) → full 4×4.
static void unpack_mbar(const double* m, double M[4][4]) {
  static const int I[10] = {0, 0, 0, 0, 1, 1, 1, 2, 2, 3}, J[10] = {0, 1, 2, 3, 1, 2, 3, 2, 3, 3};
  for (int k = 0; k < 10; ++k) M[I[k]][J[k]] = M[J[k]][I[k]] = m[k];
}

// Cholesky test: every pivot positive and finite.
static bool spd4(const double M[4][4]) {
  double L[4][4] = {};
  for (int j = 0; j < 4; ++j) {
    double d = M[j][j];
    for (int k = 0; k < j; ++k) d -= L[j][k] * L[j][k];
    if (!(d > 0.0) || !std::isfinite(d)) return false;
    L[j][j] = std::sqrt(d);
    for (int i = j + 1; i < 4; ++i) {
      double v = M[i][j];
      for (int k = 0; k < j; ++k) v -= L[i][k] * L[j][k];
      L[i][j] = v / L[j][j];
    }
  }
  return true;
}

// Symmetric 3×3 eigen-decomposition by cyclic Jacobi rotations: S = Vᵀ diag(w) V with the eigenvectors as the ROWS
// of V, det V = +1.
static void sym3_eig(const double S0[3][3], double w[3], double V[3][3]) {
  double S[3][3], U[3][3] = {{1, 0, 0}, {0, 1, 0}, {0, 0, 1}};  // S = U diag Uᵀ, eigenvectors in U's columns
  std::memcpy(S, S0, sizeof(S));
  for (int sweep = 0; sweep < 64; ++sweep) {
    const double off = S[0][1] * S[0][1] + S[0][2] * S[0][2] + S[1][2] * S[1][2];
    const double dia = S[0][0] * S[0][0] + S[1][1] * S[1][1] + S[2][2] * S[2][2];
    if (off <= 1e-40 * dia) break;
    for (int p = 0; p < 2; ++p)
      for (int q = p + 1; q < 3; ++q) {
        if (S[p][q] == 0.0) continue;
        const double th = (S[q][q] - S[p][p]) / (2.0 * S[p][q]);
        const double t = (th >= 0 ? 1.0 : -1.0) / (std::fabs(th) + std::sqrt(th * th + 1.0));
        const double c = 1.0 / std::sqrt(t * t + 1.0), sn = t * c;
        for (int k = 0; k < 3; ++k) {  // S ← Jᵀ S J with the rotation J in the (p, q) plane
          const double skp = S[k][p], skq = S[k][q];
          S[k][p] = c * skp - sn * skq;
          S[k][q] = sn * skp + c * skq;
        }
        for (int k = 0; k < 3; ++k) {
          const double spk = S[p][k], sqk = S[q][k];
          S[p][k] = c * spk - sn * sqk;
          S[q][k] = sn * spk + c * sqk;
        }
        for (int k = 0; k < 3; ++k) {
          const double ukp = U[k][p], ukq = U[k][q];
          U[k][p] = c * ukp - sn * ukq;
          U[k][q] = sn * ukp + c * ukq;
        }
      }
  }
  for (int i = 0; i < 3; ++i) {
    w[i] = S[i][i];
    for (int k = 0; k < 3; ++k) V[i][k] = U[k][i];
  }
  const double det = V[0][0] * (V[1][1] * V[2][2] - V[1][2] * V[2][1]) - V[0][1] * (V[1][0] * V[2][2] - V[1][2] * V[2][0]) +
                     V[0][2] * (V[1][0] * V[2][1] - V[1][1] * V[2][0]);
  if (det < 0)
    for (int k = 0; k < 3; ++k) V[2][k] = -V[2][k];
}

// Canonical (central, principal) body frames: DESIGN.md reading R8. A body given with a general SPD M̄ =
// [[J, s], [sᵀ, m]] is re-expressed in the frame x̄' = Q(x̄ − o), o = s/m, Q the eigenvector rows of J − s sᵀ/m,
// where M̄' = diag(eig, m). The co-rotated step is covariant under this rigid change of material frame (the
// coordinates map by q' = (T̄ ⊗ I₃) q, T̄ = [[Q, 0], [oᵀ, 1]], which commutes with diag₄(R); K̄_A is invariant
// under δA ↦ Q δA Qᵀ; the elastic force depends on AᵀA only through rotation invariants), so the library steps the
// canonical copy with the closed-form H̄⁻¹ and maps states back on output. Bodies whose M̄ is already diagonal keep
// their frame (identity map, bitwise the same arithmetic).
struct Canon {
  bool any = false;
  std::vector<double> q0, qd0, mbar, ya, yb;  // canonical copies of the inputs
  std::vector<double> frame;                  // [n][12]: Q row-major (9), o (3); identity for diagonal bodies
  mabd_bodies B;
  mabd_joints J;
};

static bool canonical_frames(const mabd_bodies* B, const mabd_joints* J, Canon* c) {
  const int64_t n = B->n;
  c->any = false;
  for (int64_t i = 0; i < n && !c->any; ++i) {
    const double* m = B->mbar + 10 * i;
    c->any = m[1] != 0.0 || m[2] != 0.0 || m[3] != 0.0 || m[5] != 0.0 || m[6] != 0.0 || m[8] != 0.0;
  }
  if (!c->any) return false;
  c->frame.assign(12 * n, 0.0);
  c->q0.assign(B->q0, B->q0 + 12 * n);
  c->qd0.assign(B->qd0, B->qd0 + 12 * n);
  c->mbar.assign(B->mbar, B->mbar + 10 * n);
  for (int64_t i = 0; i < n; ++i) {
    double* F = c->frame.data() + 12 * i;
    double M[4][4];
    unpack_mbar(B->mbar + 10 * i, M);
    const bool diag = M[0][1] == 0.0 && M[0][2] == 0.0 && M[0][3] == 0.0 && M[1][2] == 0.0 && M[1][3] == 0.0 &&
                      M[2][3] == 0.0;
    if (diag) {
      F[0] = F[4] = F[8] = 1.0;
      continue;
    }
    const double m = M[3][3];
    const double o[3] = {M[0][3] / m, M[1][3] / m, M[2][3] / m};
    double Jc[3][3], w[3], Q[3][3];
    for (int r = 0; r < 3; ++r)
      for (int k = 0; k < 3; ++k) Jc[r][k] = M[r][k] - m * o[r] * o[k];
    sym3_eig(Jc, w, Q);
    for (int r = 0; r < 3; ++r)
      for (int k = 0; k < 3; ++k) F[3 * r + k] = Q[r][k];
    for (int r = 0; r < 3; ++r) F[9 + r] = o[r];
    double* mb = c->mbar.data() + 10 * i;
    for (int k = 0; k < 10; ++k) mb[k] = 0.0;
    mb[0] = w[0];
    mb[4] = w[1];
    mb[7] = w[2];
    mb[9] = m;
    // A' = A Qᵀ, t' = t + A o (and the same map of the velocities): column c' of A' is Σ_c Q[c'][c] A[:, c]
    for (double* q : {c->q0.data() + 12 * i, c->qd0.data() + 12 * i}) {
      double A[3][3], t[3];
      for (int r = 0; r < 3; ++r) {
        for (int k = 0; k < 3; ++k) A[r][k] = q[3 * k + r];
        t[r] = q[9 + r];
      }
      for (int cp = 0; cp < 3; ++cp)
        for (int r = 0; r < 3; ++r) q[3 * cp + r] = A[r][0] * Q[cp][0] + A[r][1] * Q[cp][1] + A[r][2] * Q[cp][2];
      for (int r = 0; r < 3; ++r) q[9 + r] = t[r] + A[r][0] * o[0] + A[r][1] * o[1] + A[r][2] * o[2];
    }
  }
  // material points on bodies: ȳ' = Q(ȳ − o)
  int64_t P = 0;
  for (int64_t k = 0; k < J->n_joints; ++k) P += J->npts[k];
  c->ya.assign(J->ybar_a, J->ybar_a + 3 * P);
  c->yb.assign(J->ybar_b, J->ybar_b + 3 * P);
  for (int64_t k = 0, pt = 0; k < J->n_joints; ++k)
    for (int q = 0; q < J->npts[k]; ++q, ++pt)
      for (int side = 0; side < 2; ++side) {
        const int64_t b = side ? J->body_b[k] : J->body_a[k];
        if (b < 0) continue;  // world point of an anchor
        const double* F = c->frame.data() + 12 * b;
        double* y = (side ? c->yb.data() : c->ya.data()) + 3 * pt;
        const double d[3] = {y[0] - F[9], y[1] - F[10], y[2] - F[11]};
        for (int r = 0; r < 3; ++r) y[r] = F[3 * r] * d[0] + F[3 * r + 1] * d[1] + F[3 * r + 2] * d[2];
      }
  c->B = *B;
  c->B.q0 = c->q0.data();
  c->B.qd0 = c->qd0.data();
  c->B.mbar = c->mbar.data();
  c->J = *J;
  c->J.ybar_a = c->ya.data();
  c->J.ybar_b = c->yb.data();
  return true;
}

// ------------------------------------------------------------------------------------------ validation
static mabd_status validate(const mabd_bodies* B, const mabd_joints* J, const mabd_options* o, std::string* msg) {
  if (!B || !J) return *msg = "bodies/joints NULL", MABD_EINVAL;
  if (B->n < 1) return *msg = "n must be >= 1", MABD_EINVAL;
  if (B->n > (int64_t)INT_MAX / 2) return *msg = "too many bodies", MABD_EINVAL;
  if (!B->q0 || !B->qd0 || !B->mbar || !B->volume || !B->youngs || !B->poisson)
    return *msg = "a body array is NULL", MABD_EINVAL;
  if (J->n_joints < 0) return *msg = "n_joints < 0", MABD_EINVAL;
  if (J->n_joints > 0 && (!J->body_a || !J->body_b || !J->npts || !J->ybar_a || !J->ybar_b))
    return *msg = "a joint array is NULL", MABD_EINVAL;
  if (o) {
    if (o->newton_iters < 0 || o->newton_iters > 16) return *msg = "newton_iters must be in [0, 16]", MABD_EINVAL;
    if (o->world > 1 && (o->rank < 0 || o->rank >= o->world)) return *msg = "rank outside [0, world)", MABD_EINVAL;
    if (o->world > 256) return *msg = "world > 256", MABD_EINVAL;
    if (o->solver < 0 || o->solver > MABD_SOLVER_LOOP_BREAKER) return *msg = "unknown solver", MABD_EINVAL;
    if (o->gs_sweeps < 0 || !(o->gs_tol >= 0.0)) return *msg = "gs_sweeps and gs_tol must be >= 0", MABD_EINVAL;
    if (o->host_exchange && (o->world < 2 || o->newton_iters > 1))
      return *msg = "host_exchange needs world >= 2 and one Newton iteration", MABD_EINVAL;
    if (o->rotation != MABD_ROTATION_POLAR && o->rotation != MABD_ROTATION_LENGTH_PRESERVING)
      return *msg = "rotation must be MABD_ROTATION_POLAR (0) or MABD_ROTATION_LENGTH_PRESERVING (1)", MABD_EINVAL;
    if (o->residual_rhs != 0 && o->residual_rhs != 1)
      return *msg = "residual_rhs must be 1 (0 = default = 1): -C(qn) is always in the dual rhs", MABD_EINVAL;
  }
  for (int64_t i = 0; i < B->n; ++i) {
    const double* m = B->mbar + 10 * i;
    double M[4][4];
    unpack_mbar(m, M);
    if (!spd4(M))
      return *msg = fmt("body %lld: mbar must be symmetric positive definite", (long long)i), MABD_EINVAL;
    if (!(B->volume[i] > 0) || !(B->youngs[i] > 0) || !(B->poisson[i] > -1.0 && B->poisson[i] < 0.5))
      return *msg = fmt("body %lld: need V > 0, E > 0, -1 < nu < 0.5", (long long)i), MABD_EINVAL;
    for (int c = 0; c < 12; ++c)
      if (!std::isfinite(B->q0[12 * i + c]) || !std::isfinite(B->qd0[12 * i + c]))
        return *msg = fmt("body %lld: non-finite initial state", (long long)i), MABD_EINVAL;
  }
  int64_t P = 0;
  for (int64_t k = 0; k < J->n_joints; ++k) {
    const int32_t a = J->body_a[k], b = J->body_b[k], np = J->npts[k];
    if (a < 0 || a >= B->n) return *msg = fmt("joint %lld: body_a out of range", (long long)k), MABD_EINVAL;
    if (b < -1 || b >= B->n) return *msg = fmt("joint %lld: body_b out of range", (long long)k), MABD_EINVAL;
    if (a == b) return *msg = fmt("joint %lld: both ends on body %lld", (long long)k, a), MABD_EINVAL;
    const int32_t kd = J->kind ? J->kind[k] : 0;
    if (kd < 0 || kd > 3)
      return *msg = fmt("joint %lld: kind must be 0 (point), 1 (five-row hinge), 2 (universal) or 3 (prismatic)",
                        (long long)k), MABD_EINVAL;
    if (kd == 3 ? np != 3 : (np != 1 && np != 2))
      return *msg = fmt("joint %lld: npts must be 1 or 2 (3 for a prismatic joint)", (long long)k), MABD_EINVAL;
    if ((kd == 1 || kd == 2) && np != 2)
      return *msg = fmt("joint %lld: five-row hinges and universal joints have npts = 2", (long long)k),
             MABD_EINVAL;
    P += np;
  }
  for (int64_t p = 0; p < 3 * P; ++p)
    if (!std::isfinite(J->ybar_a[p]) || !std::isfinite(J->ybar_b[p]))
      return *msg = "non-finite joint point", MABD_EINVAL;
  return MABD_OK;
}

// ------------------------------------------------------------------------------------------ materials
// Bodies that share (V, μ, λ, M̄/m) share a material; their mass ratio is a per-body scale.
static void detect_materials(const mabd_bodies* B, Plan* p, std::vector<int32_t>* mid_body,
                             std::vector<double>* msc_body) {
  std::unordered_map<Key48, int32_t, Key48Hash> map;
  const int64_t n = B->n;
  mid_body->resize(n);
  msc_body->resize(n);
  p->mats.clear();
  for (int64_t i = 0; i < n; ++i) {
    const double* m = B->mbar + 10 * i;
    const double E = B->youngs[i], nu = B->poisson[i];
    const double mu = E / (2.0 * (1.0 + nu));
    const double lam = E * nu / ((1.0 + nu) * (1.0 - 2.0 * nu));
    const double key[6] = {B->volume[i], mu, lam, m[0] / m[9], m[4] / m[9], m[7] / m[9]};
    Key48 kk = key_of(key);
    auto it = map.find(kk);
    int32_t id;
    if (it == map.end()) {
      id = (int32_t)p->mats.size();
      map.emplace(kk, id);
      Material M{m[0], m[4], m[7], m[9], B->volume[i], mu, lam, 0.0};
      p->mats.push_back(M);
    } else {
      id = it->second;
    }
    (*mid_body)[i] = id;
    (*msc_body)[i] = m[9] / p->mats[id].m;
  }
}

// ------------------------------------------------------------------------------------------ chain topology
// Forest of paths with ball joints only, each body in ≤ 2 joints, anchors only at path ends (A14).
static bool chain_build(const mabd_joints* J, int64_t n, Plan* p, std::vector<int64_t>* pos_of_body,
                        std::string* msg) {
  const int64_t K = J->n_joints;
  std::vector<int32_t> deg(n, 0), ideg(n, 0);
  std::vector<int64_t> pt_off(K + 1, 0);
  for (int64_t k = 0; k < K; ++k) {
    if (J->npts[k] != 1) return *msg = "chain solver needs ball joints (npts = 1)", false;
    pt_off[k + 1] = pt_off[k] + J->npts[k];
    deg[J->body_a[k]]++;
    if (J->body_b[k] >= 0) {
      deg[J->body_b[k]]++;
      ideg[J->body_a[k]]++;
      ideg[J->body_b[k]]++;
    }
  }
  for (int64_t i = 0; i < n; ++i)
    if (deg[i] > 2) return *msg = "a body has more than 2 joints", false;
  // incidence lists (≤ 2 per body)
  std::vector<int64_t> inc(2 * n, -1);
  std::vector<int32_t> cnt(n, 0);
  for (int64_t k = 0; k < K; ++k) {
    inc[2 * J->body_a[k] + cnt[J->body_a[k]]++] = k;
    if (J->body_b[k] >= 0) inc[2 * J->body_b[k] + cnt[J->body_b[k]]++] = k;
  }
  auto other = [&](int64_t k, int64_t b) -> int64_t { return J->body_a[k] == b ? J->body_b[k] : J->body_a[k]; };
  std::vector<char> seen(n, 0);
  // walk every path from an end (ideg ≤ 1); prefer the end that carries an anchor
  struct Chain {
    std::vector<int64_t> bodies;
    std::vector<int64_t> joints;  // interior joints, joints[i] links bodies[i] and bodies[i+1]
    int64_t start_anchor = -1, end_anchor = -1;
  };
  std::vector<Chain> chains;
  auto anchor_of = [&](int64_t b, int64_t skip) -> int64_t {
    for (int s = 0; s < cnt[b]; ++s) {
      const int64_t k = inc[2 * b + s];
      if (J->body_b[k] < 0 && k != skip) return k;
    }
    return -1;
  };
  std::vector<int64_t> starts;
  for (int64_t i = 0; i < n; ++i)
    if (ideg[i] <= 1 && anchor_of(i, -1) >= 0) starts.push_back(i);
  for (int64_t i = 0; i < n; ++i)
    if (ideg[i] <= 1 && anchor_of(i, -1) < 0) starts.push_back(i);
  for (int64_t s0 : starts) {
    if (seen[s0]) continue;
    Chain ch;
    int64_t b = s0, prevj = -1;
    ch.start_anchor = anchor_of(b, -1);
    while (true) {
      seen[b] = 1;
      ch.bodies.push_back(b);
      int64_t nextj = -1;
      for (int s = 0; s < cnt[b]; ++s) {
        const int64_t k = inc[2 * b + s];
        if (k != prevj && J->body_b[k] >= 0) nextj = k;
      }
      if (nextj < 0) break;
      ch.joints.push_back(nextj);
      prevj = nextj;
      b = other(nextj, b);
      if (seen[b]) return *msg = "cycle in the joint graph", false;
    }
    ch.end_anchor = anchor_of(b, ch.start_anchor);
    if (ch.bodies.size() > 1 || ch.end_anchor != ch.start_anchor) {
      // anchors at interior bodies are impossible here (deg ≤ 2 and interior bodies have ideg = 2)
    }
    if (ch.bodies.size() == 1 && ch.end_anchor == ch.start_anchor) ch.end_anchor = -1;
    chains.push_back(std::move(ch));
  }
  for (int64_t i = 0; i < n; ++i)
    if (!seen[i]) return *msg = "cycle in the joint graph", false;

  // ---- windows: short chains packed into 256-slot windows, long chains over consecutive windows
  std::vector<int64_t> chain_base(chains.size());
  int64_t nwin = 0, used = SEG;  // used = slots used in the current packed window (SEG = none open)
  std::vector<int32_t> flags;
  for (size_t c = 0; c < chains.size(); ++c) {
    const int64_t m = (int64_t)chains[c].bodies.size() + (chains[c].end_anchor >= 0 ? 1 : 0);
    if (m <= SEG) {
      if (used + m > SEG) {
        flags.push_back(0);
        ++nwin;
        used = 0;
      }
      chain_base[c] = (nwin - 1) * SEG + used;
      used += m;
    } else {
      const int64_t w = (m + SEG - 1) / SEG;
      chain_base[c] = nwin * SEG;
      for (int64_t i = 0; i < w; ++i) {
        int32_t f = SEG_LONG;
        if (i > 0) f |= SEG_LEFT_IFACE;
        if (i + 1 < w) f |= SEG_RIGHT_IFACE;
        flags.push_back(f);
      }
      nwin += w;
      used = SEG;  // do not pack after a long chain's last window
    }
  }
  p->n_windows = nwin;
  p->ld = nwin * SEG;
  p->seg_flags = flags;
  p->slot_info.assign(p->ld + 1, slot_pack(SIDE_NONE, SIDE_NONE, 0));
  p->geo.assign(6, 0.0);  // geometry 0: zeros (absent slots)
  std::unordered_map<Key48, uint32_t, Key48Hash> gmap;
  gmap.emplace(key_of(p->geo.data()), 0u);
  auto geo_id = [&](const double* yl, const double* yr) -> uint32_t {
    double v[6] = {yl[0], yl[1], yl[2], yr[0], yr[1], yr[2]};
    Key48 kk = key_of(v);
    auto it = gmap.find(kk);
    if (it != gmap.end()) return it->second;
    const uint32_t id = (uint32_t)(p->geo.size() / 6);
    p->geo.insert(p->geo.end(), v, v + 6);
    gmap.emplace(kk, id);
    return id;
  };
  pos_of_body->assign(n, -1);
  int64_t rows = 0;
  for (size_t c = 0; c < chains.size(); ++c) {
    const Chain& ch = chains[c];
    const int64_t base = chain_base[c];
    const int64_t L = (int64_t)ch.bodies.size();
    for (int64_t i = 0; i < L; ++i) (*pos_of_body)[ch.bodies[i]] = base + i;
    // slot 0: start anchor (world, body) or absent (none, body)
    if (ch.start_anchor >= 0) {
      const int64_t k = ch.start_anchor;  // body_a = body, body_b = world: C = x_a(ȳ_a) − p
      const uint32_t g = geo_id(J->ybar_b + 3 * k, J->ybar_a + 3 * k);
      p->slot_info[base] = slot_pack(SIDE_WORLD, SIDE_BODY, g);
      rows += 3;
    } else {
      p->slot_info[base] = slot_pack(SIDE_NONE, SIDE_BODY, 0);
    }
    for (int64_t i = 0; i + 1 < L; ++i) {
      const int64_t k = ch.joints[i];
      const bool a_left = J->body_a[k] == ch.bodies[i];
      const double* yl = a_left ? J->ybar_a + 3 * k : J->ybar_b + 3 * k;
      const double* yr = a_left ? J->ybar_b + 3 * k : J->ybar_a + 3 * k;
      p->slot_info[base + i + 1] = slot_pack(SIDE_BODY, SIDE_BODY, geo_id(yl, yr));
      rows += 3;
    }
    if (ch.end_anchor >= 0) {
      const int64_t k = ch.end_anchor;
      p->slot_info[base + L] = slot_pack(SIDE_BODY, SIDE_WORLD, geo_id(J->ybar_a + 3 * k, J->ybar_b + 3 * k));
      rows += 3;
    }
  }
  // pt_off unused for ball joints (one point per joint, indexed by joint id)
  (void)pt_off;
  p->n_dual_rows = rows;
  // long windows: ordinal, list, left-interface flags
  p->seg_red.assign(nwin, -1);
  p->long_list.clear();
  p->left_iface.clear();
  for (int64_t w = 0; w < nwin; ++w)
    if (p->seg_flags[w] & SEG_LONG) {
      p->seg_red[w] = (int32_t)p->long_list.size();
      p->long_list.push_back((int32_t)w);
      p->left_iface.push_back((p->seg_flags[w] & SEG_LEFT_IFACE) ? 1 : 0);
    }
  p->n_long = (int64_t)p->long_list.size();
  p->levels.clear();
  if (p->n_long > 0) {
    int64_t nu = p->n_long;
    while (true) {
      BtdLevel L;
      L.n_u = nu;
      L.windows = (nu + SEG - 1) / SEG;
      L.fused = nu <= SEG;
      p->levels.push_back(L);
      if (L.fused) break;
      nu = L.windows;
    }
  }
  const int64_t nl = (int64_t)p->levels.size();
  p->launches_per_step = 1 + (p->n_long > 0 ? (int32_t)(2 * nl - 1 + 1) : 0);
  // one window using at most SMALL_SLOTS slots: the one-warp kernel (latency-bound scenes such as config 1)
  p->small_chain = p->n_windows == 1 && p->n_long == 0;
  for (int64_t t = SMALL_SLOTS; t < (int64_t)p->slot_info.size() && p->small_chain; ++t)
    if (p->slot_info[t] != slot_pack(SIDE_NONE, SIDE_NONE, 0)) p->small_chain = false;
  return true;
}

// ------------------------------------------------------------------------------------------ chain parts
// W parts own contiguous window ranges (≈ nw/W each). A boundary may split a long chain; the part on its left
// is then "right-open" and must hold ≤ 256 or a multiple of 256 long windows, so that its last BTD window ends
// exactly on the next part's first slot (the boundary is moved left until that holds). Per step each part
// reduces its long windows to a 2-equation top (BTD level, then a sequential top); the W tops form a
// block-tridiagonal system solved redundantly after one all-gather.
static bool partition_chain(Plan* p, int W, int rank, bool emulate, std::string* msg) {
  p->n_parts = W;
  p->parts.clear();
  p->local_windows.clear();
  p->local_long.clear();
  p->part_left_open.assign(W, 0);
  if (W <= 1) {
    p->part_lo = 0;
    p->part_hi = 1;
    return true;
  }
  const int64_t nw = p->n_windows;
  std::vector<int64_t> long_before(nw + 1, 0);  // long windows in [0, w)
  for (int64_t w = 0; w < nw; ++w) long_before[w + 1] = long_before[w] + ((p->seg_flags[w] & SEG_LONG) ? 1 : 0);
  auto splits = [&](int64_t b) { return b > 0 && b < nw && (p->seg_flags[b] & SEG_LEFT_IFACE); };
  std::vector<int64_t> bnd(W + 1, 0);
  bnd[W] = nw;
  for (int q = 1; q < W; ++q) {
    int64_t b = std::max<int64_t>((int64_t)((double)q * nw / W + 0.5), bnd[q - 1]);
    b = std::min(b, nw);
    while (splits(b)) {
      const int64_t n1 = long_before[b] - long_before[bnd[q - 1]];
      if (n1 <= SEG || n1 % SEG == 0) break;
      --b;
    }
    bnd[q] = b;
  }
  for (int q = 0; q < W; ++q) {
    Plan::Part P;
    P.win_lo = bnd[q];
    P.win_hi = bnd[q + 1];
    P.long_lo = long_before[P.win_lo];
    P.long_hi = long_before[P.win_hi];
    P.left_open = splits(P.win_lo) ? 1 : 0;
    P.right_open = splits(P.win_hi) ? 1 : 0;
    P.n1 = P.long_hi - P.long_lo;
    P.btd1 = P.n1 > SEG;
    P.n2 = P.btd1 ? (P.n1 + SEG - 1) / SEG : P.n1;
    if (P.n2 > SEG) return *msg = "a part holds more than 65,536 long-chain segments", false;
    if (P.right_open && P.btd1 && P.n1 % SEG != 0) return *msg = "internal: unaligned right-open part", false;
    p->part_left_open[q] = P.left_open;
    if (P.left_open && P.n1 > 0) p->left_iface[P.long_lo] = 0;  // the left part enters via the rank-level system
    p->parts.push_back(P);
  }
  p->part_lo = emulate ? 0 : rank;
  p->part_hi = emulate ? W : rank + 1;
  for (int q = p->part_lo; q < p->part_hi; ++q) {
    for (int64_t w = p->parts[q].win_lo; w < p->parts[q].win_hi; ++w) p->local_windows.push_back((int32_t)w);
    for (int64_t u = p->parts[q].long_lo; u < p->parts[q].long_hi; ++u) p->local_long.push_back(p->long_list[u]);
  }
  int lps = p->n_long == 0 ? 1 : 1 + 1 + 1;  // chain pass 1 (+ global solve, chain finish if a chain is long)
  for (int q = p->part_lo; q < p->part_hi; ++q)
    if (p->parts[q].n1 > 0) lps += 2 + (p->parts[q].btd1 ? 2 : 0);
  p->launches_per_step = lps;
  return true;
}

// ------------------------------------------------------------------------------------------ build_plan
mabd_status build_plan(const mabd_bodies* B, const mabd_joints* J, const mabd_options* o, Plan* p, std::string* msg) {
  mabd_status st = validate(B, J, o, msg);
  if (st != MABD_OK) return st;
  *p = Plan();
  Canon canon;
  if (canonical_frames(B, J, &canon)) {  // from here on the scene is in the canonical body frames
    B = &canon.B;
    J = &canon.J;
    p->frame = std::move(canon.frame);
  }
  p->n = B->n;
  p->n_joints = J->n_joints;
  p->newton_iters = (o && o->newton_iters > 1) ? o->newton_iters : 1;
  p->rotation = o ? o->rotation : MABD_ROTATION_POLAR;
  for (int i = 0; i < 3; ++i) p->grav[i] = B->gravity[i];
  std::vector<int32_t> mid;
  std::vector<double> msc;
  detect_materials(B, p, &mid, &msc);

  int req = o ? o->solver : 0;
  std::vector<int64_t> pos;
  std::string why;
  bool ok = false;
  if (req == MABD_SOLVER_LOOP_BREAKER) {  // the paper's Case III: the forest by chain / tree, + breakers
    if (o && o->world > 1) return *msg = "loop breakers run on one GPU", MABD_EUNSUPPORTED;
    if (!loop_split(J, B->n, &p->loop, &why)) return *msg = "loop breakers: " + why, MABD_EINVAL;
    p->loop.active = true;
    J = &p->loop.forest;
    req = 0;  // chain if the forest is a set of ball-joint paths, else tree
  }
  if (req == 0 || req == MABD_SOLVER_CHAIN) {
    ok = chain_build(J, B->n, p, &pos, &why);
    if (ok) {
      p->solver = MABD_SOLVER_CHAIN;
      const int W = o && o->world > 1 ? o->world : 1;
      p->use_nccl = W > 1 && o->nccl_unique_id != nullptr && !o->host_exchange;
      p->host_exchange = W > 1 && o->host_exchange;
      if (!partition_chain(p, W, o ? o->rank : 0, W > 1 && !p->use_nccl && !p->host_exchange, msg))
        return MABD_EINVAL;
    }
    if (!ok && req == MABD_SOLVER_CHAIN) return *msg = "chain solver requested: " + why, MABD_EINVAL;
  }
  if (!ok && (req == 0 || req == MABD_SOLVER_TREE)) {
    std::string why2;
    ok = tree_build(J, B->n, p, &pos, &why2);
    if (ok) p->solver = MABD_SOLVER_TREE;
    if (!ok && req == MABD_SOLVER_TREE) return *msg = "tree solver requested: " + why2, MABD_EINVAL;
    if (!ok) why += "; " + why2;
  }
  if (!ok && req == MABD_SOLVER_LINE_GS) {  // the paper's Case IV, any topology
    ok = sparse_build(B, J, p, &pos, &why, false) && gs_build(B, p, o->gs_sweeps, o->gs_tol, &why);
    if (!ok) return *msg = "line Gauss-Seidel: " + why, MABD_EINVAL;
    p->solver = MABD_SOLVER_LINE_GS;
  }
  if (!ok && p->loop.active) return *msg = "loop breakers: the forest is neither chains nor trees", MABD_EINVAL;
  if (!ok && (req == 0 || req == MABD_SOLVER_SPARSE)) {
    std::string why3;
    ok = sparse_build(B, J, p, &pos, &why3);
    if (ok) p->solver = MABD_SOLVER_SPARSE;
    if (!ok) why += "; " + why3;
  }
  if (!ok) {
    *msg = "topology not supported by this build (" + why + ")";
    return MABD_EUNSUPPORTED;
  }
  p->step_end_folded = p->small_chain && p->newton_iters == 1 && !p->loop.active && p->n_parts <= 1;
  if (p->loop.active) {  // breaker points → internal positions; 2 + 3b forest runs + 2 kernels each, + solve, force
    for (auto* v : {&p->loop.pa, &p->loop.pb})
      for (int32_t& b : *v) b = (int32_t)pos[b];
    const int runs = 2 + 3 * (int)p->loop.pa.size();
    p->launches_per_step = runs * (p->launches_per_step + 2) - 1;
  }
  if (p->newton_iters > 1) p->launches_per_step = p->newton_iters * p->launches_per_step + 2;  // + prep, final
  if (o && o->world > 1 && p->solver == MABD_SOLVER_TREE) {
    const int W = o->world;
    p->use_nccl = o->nccl_unique_id != nullptr && !o->host_exchange;
    p->host_exchange = o->host_exchange != 0;
    if (!tree_partition(p, W, o->rank, !p->use_nccl && !p->host_exchange, msg)) return MABD_EINVAL;
  }
  if (o && o->world > 1 && (p->solver == MABD_SOLVER_SPARSE || p->solver == MABD_SOLVER_LINE_GS))
    return *msg = "world > 1 is implemented for the chain and tree solvers (run nets as replicas)",
           MABD_EUNSUPPORTED;
  // per-position arrays
  const int64_t ld = p->ld;
  p->perm.assign(B->n, 0);
  bool multi_mat = p->mats.size() > 1, any_scale = false;
  for (int64_t i = 0; i < B->n; ++i)
    if (msc[i] != 1.0) any_scale = true;
  if (multi_mat) p->mat_id.assign(ld, 0);
  if (any_scale) p->mscale.assign(ld, 1.0);
  p->q_soa.assign(12 * ld, 0.0);
  p->qd_soa.assign(12 * ld, 0.0);
  for (int64_t i = 0; i < B->n; ++i) {
    const int64_t s = pos[i];
    p->perm[i] = s;
    if (multi_mat) p->mat_id[s] = mid[i];
    if (any_scale) p->mscale[s] = msc[i];
    for (int c = 0; c < 12; ++c) {
      p->q_soa[c * ld + s] = B->q0[12 * i + c];
      p->qd_soa[c * ld + s] = B->qd0[12 * i + c];
    }
  }
  // ---- device layout
  size_t cur = 0;
  auto take = [&](size_t bytes) {
    const size_t o2 = cur;
    cur = align_up(cur + std::max<size_t>(bytes, 8));
    return o2;
  };
  Plan::Off& f = p->off;
  f.q = take(sizeof(double) * 12 * ld);
  f.qd = take(sizeof(double) * 12 * ld);
  f.rs = take(sizeof(double) * 9 * ld);
  f.z = p->newton_iters > 1 ? take(sizeof(double) * 12 * ld) : 0;
  f.wr = take(sizeof(double) * 9 * ld);
  f.mat_id = multi_mat ? take(sizeof(int32_t) * ld) : 0;
  f.mscale = any_scale ? take(sizeof(double) * ld) : 0;
  f.mats = take(sizeof(Material) * p->mats.size());
  f.hinv = take(sizeof(HinvBlk) * p->mats.size());
  f.perm = take(sizeof(int64_t) * B->n);
  f.io = take(sizeof(double) * 24 * B->n);
  f.err = take(sizeof(int32_t) * 4);
  f.frame = p->frame.empty() ? 0 : take(sizeof(double) * p->frame.size());
  if (p->loop.active) {
    LoopPlan& L = p->loop;
    const size_t m = 3 * L.pa.size();
    L.o_save = take(sizeof(double) * 24 * ld);
    L.o_M = take(sizeof(double) * (1 + m) * m);
    L.o_lam = take(sizeof(double) * m);
    L.o_pa = take(sizeof(int32_t) * L.pa.size());
    L.o_pb = take(sizeof(int32_t) * L.pb.size());
    L.o_ya = take(sizeof(double) * L.ya.size());
    L.o_yb = take(sizeof(double) * L.yb.size());
  }
  if (p->solver == MABD_SOLVER_CHAIN) {
    f.slot_info = take(sizeof(uint32_t) * (ld + 16));  // + padding: segments stage SEG + 4 slot codes
    f.geo = take(sizeof(double) * p->geo.size());
    f.seg_flags = take(sizeof(int32_t) * p->n_windows);
    f.seg_red = take(sizeof(int32_t) * p->n_windows);
    f.long_list = take(sizeof(int32_t) * std::max<int64_t>(1, p->n_long));
    f.left_iface = take(sizeof(int32_t) * std::max<int64_t>(1, p->n_long));
    f.tops.clear();
    f.lams.clear();
    f.tops.push_back(take(sizeof(Top) * std::max<int64_t>(1, p->n_long)));
    if (p->n_parts <= 1) {
      for (const BtdLevel& L : p->levels) {
        f.lams.push_back(take(sizeof(double) * 3 * L.n_u));
        if (!L.fused) f.tops.push_back(take(sizeof(Top) * L.windows));
      }
    } else {
      f.lams.push_back(take(sizeof(double) * 3 * (p->n_long + 1)));  // λ of every long window (+ one spare)
      f.all_tops = take(sizeof(Top) * p->n_parts);
      f.lam_g = take(sizeof(double) * 3 * (p->n_parts + 1));
      f.plo = take(sizeof(int32_t) * p->n_parts);
      f.lwin = take(sizeof(int32_t) * std::max<size_t>(1, p->local_windows.size()));
      f.llong = take(sizeof(int32_t) * std::max<size_t>(1, p->local_long.size()));
      f.p_tops1.assign(p->n_parts, 0);
      f.p_lam2.assign(p->n_parts, 0);
      f.p_scr.assign(p->n_parts, 0);
      for (int q = p->part_lo; q < p->part_hi; ++q) {
        const Plan::Part& P = p->parts[q];
        if (P.n1 == 0) continue;
        if (P.btd1) {
          f.p_tops1[q] = take(sizeof(Top) * P.n2);
          f.p_lam2[q] = take(sizeof(double) * 3 * P.n2);
        }
        f.p_scr[q] = take(sizeof(double) * 27 * (P.n2 + 1));
      }
    }
  }
  if (p->solver == MABD_SOLVER_TREE) {
    const TreePlan& t = p->tree;
    const int64_t K = p->n_joints, n = B->n;
    f.t_up = take(sizeof(int32_t) * n);
    f.t_coff = take(sizeof(int32_t) * (n + 1));
    f.t_cj = take(sizeof(int32_t) * std::max<size_t>(1, t.child_joint.size()));
    f.t_wsoff = take(sizeof(int64_t) * (n + 1));
    f.t_jnpts = take(sizeof(int32_t) * std::max<int64_t>(1, K));
    f.t_jchd = take(sizeof(int32_t) * std::max<int64_t>(1, K));
    f.t_jy = take(sizeof(double) * 12 * std::max<int64_t>(1, K));
    f.t_goff = take(sizeof(int32_t) * t.group_off.size());
    f.t_glp = take(sizeof(int32_t) * t.glev_ptr.size());
    f.t_glo = take(sizeof(int32_t) * t.glev_off.size());
    f.t_glnl = take(sizeof(int32_t) * std::max<size_t>(1, t.glev_nl.size()));
    f.t_fo = take(sizeof(int64_t) * std::max<int64_t>(1, n));
    f.t_fstr = take(sizeof(int32_t) * std::max<int64_t>(1, n));
    f.t_par = take(sizeof(int32_t) * std::max<int64_t>(1, n));
    f.t_uprow = take(sizeof(int32_t) * std::max<int64_t>(1, n));
    f.t_f0 = take(sizeof(double) * std::max<int64_t>(1, t.fo_total));
    f.t_shat = take(sizeof(double) * 28 * std::max<int64_t>(1, K));
    f.t_lam = take(sizeof(double) * 6 * std::max<int64_t>(1, K));
    f.t_bscr = take(sizeof(double) * 21 * n);
    f.t_ws = take(sizeof(double) * std::max<int64_t>(1, t.ws_total));
    f.t_ptoff = take(sizeof(int32_t) * (n + 1));
    f.t_ptcode = take(sizeof(int32_t) * std::max<size_t>(1, t.pt_code.size()));
    f.t_nn = take(sizeof(int32_t) * n);
    f.t_rootj = take(sizeof(int32_t) * std::max<size_t>(1, t.root_joint.size()));
    f.t_rslot = take(sizeof(int32_t) * std::max<size_t>(1, t.root_slot.size()));
    f.t_xbuf = take(sizeof(double) * 42 * (size_t)std::max(1, t.parts * t.rpp));
  }
  if (p->solver == MABD_SOLVER_SPARSE || p->solver == MABD_SOLVER_LINE_GS) sparse_layout(p, take);
  p->workspace_bytes = cur;
  return MABD_OK;
}

// ------------------------------------------------------------------------------------------ device side
template <class T>
static cudaError_t put(T* dst, const std::vector<T>& v, cudaStream_t st) {
  if (v.empty()) return cudaSuccess;
  return cudaMemcpyAsync(dst, v.data(), sizeof(T) * v.size(), cudaMemcpyHostToDevice, st);
}

cudaError_t upload_plan(const Plan& p, char* ws, cudaStream_t st, DevPtrs* d) {
  const Plan::Off& f = p.off;
  d->b.q = (double*)(ws + f.q);
  d->b.qd = (double*)(ws + f.qd);
  d->b.rs = (double*)(ws + f.rs);
  d->b.z = p.newton_iters > 1 ? (double*)(ws + f.z) : nullptr;
  d->wr_buf = (double*)(ws + f.wr);
  d->b.wr = nullptr;
  d->b.ld = p.ld;
  d->b.mat_id = p.mat_id.empty() ? nullptr : (const int32_t*)(ws + f.mat_id);
  d->b.mscale = p.mscale.empty() ? nullptr : (const double*)(ws + f.mscale);
  d->mats = (Material*)(ws + f.mats);
  d->b.mats = d->mats;
  d->hinv = (HinvBlk*)(ws + f.hinv);
  d->perm = (int64_t*)(ws + f.perm);
  d->io = (double*)(ws + f.io);
  d->err = (int32_t*)(ws + f.err);
  d->frame = p.frame.empty() ? nullptr : (double*)(ws + f.frame);
  cudaError_t e;
  if (d->frame && (e = put(d->frame, p.frame, st))) return e;
  if (p.loop.active) {  // the breaker forces ride on the wrench buffer, zero elsewhere
    const LoopPlan& L = p.loop;
    d->loop_save = (double*)(ws + L.o_save);
    d->loop_M = (double*)(ws + L.o_M);
    d->loop_lam = (double*)(ws + L.o_lam);
    d->loop_pa = (int32_t*)(ws + L.o_pa);
    d->loop_pb = (int32_t*)(ws + L.o_pb);
    d->loop_ya = (double*)(ws + L.o_ya);
    d->loop_yb = (double*)(ws + L.o_yb);
    if ((e = put(d->loop_pa, L.pa, st)) || (e = put(d->loop_pb, L.pb, st)) || (e = put(d->loop_ya, L.ya, st)) ||
        (e = put(d->loop_yb, L.yb, st)))
      return e;
    if ((e = cudaMemsetAsync(d->wr_buf, 0, sizeof(double) * 9 * p.ld, st))) return e;
    d->b.wr = d->wr_buf;
  }
  if ((e = put(d->b.q, p.q_soa, st))) return e;
  if ((e = put(d->b.qd, p.qd_soa, st))) return e;
  if (!p.mat_id.empty() && (e = put((int32_t*)d->b.mat_id, p.mat_id, st))) return e;
  if (!p.mscale.empty() && (e = put((double*)d->b.mscale, p.mscale, st))) return e;
  if ((e = put(d->mats, p.mats, st))) return e;
  if ((e = put(d->perm, p.perm, st))) return e;
  if (p.solver == MABD_SOLVER_CHAIN) {
    d->slot_info = (uint32_t*)(ws + f.slot_info);
    d->geo = (double*)(ws + f.geo);
    d->seg_flags = (int32_t*)(ws + f.seg_flags);
    d->seg_red = (int32_t*)(ws + f.seg_red);
    d->long_list = (int32_t*)(ws + f.long_list);
    d->left_iface = (int32_t*)(ws + f.left_iface);
    if ((e = put(d->slot_info, p.slot_info, st))) return e;
    if ((e = put(d->geo, p.geo, st))) return e;
    if ((e = put(d->seg_flags, p.seg_flags, st))) return e;
    if ((e = put(d->seg_red, p.seg_red, st))) return e;
    if ((e = put(d->long_list, p.long_list, st))) return e;
    if ((e = put(d->left_iface, p.left_iface, st))) return e;
    d->tops.clear();
    d->lams.clear();
    for (size_t o : f.tops) d->tops.push_back((Top*)(ws + o));
    for (size_t o : f.lams) d->lams.push_back((double*)(ws + o));
    if (p.n_parts > 1) {
      d->all_tops = (Top*)(ws + f.all_tops);
      d->lam_g = (double*)(ws + f.lam_g);
      d->part_left_open = (int32_t*)(ws + f.plo);
      d->local_windows = (int32_t*)(ws + f.lwin);
      d->local_long = (int32_t*)(ws + f.llong);
      if ((e = put(d->part_left_open, p.part_left_open, st))) return e;
      if ((e = put(d->local_windows, p.local_windows, st))) return e;
      if ((e = put(d->local_long, p.local_long, st))) return e;
      // parts without long windows keep an identity top (their rank-level unknown gets λ = 0)
      std::vector<Top> ident(p.n_parts);
      for (Top& T : ident) {
        std::memset(&T, 0, sizeof(T));
        T.D0[0] = T.D0[3] = T.D0[5] = 1.0;
        T.D1[0] = T.D1[3] = T.D1[5] = 1.0;
      }
      if ((e = put(d->all_tops, ident, st))) return e;
      if ((e = cudaMemsetAsync(d->lam_g, 0, sizeof(double) * 3 * (p.n_parts + 1), st))) return e;
      d->p_tops1.assign(p.n_parts, nullptr);
      d->p_lam2.assign(p.n_parts, nullptr);
      d->p_scr.assign(p.n_parts, nullptr);
      for (int q = p.part_lo; q < p.part_hi; ++q) {
        if (p.parts[q].n1 == 0) continue;
        if (p.parts[q].btd1) {
          d->p_tops1[q] = (Top*)(ws + f.p_tops1[q]);
          d->p_lam2[q] = (double*)(ws + f.p_lam2[q]);
        }
        d->p_scr[q] = (double*)(ws + f.p_scr[q]);
      }
    }
  }
  if (p.solver == MABD_SOLVER_TREE) {
    const TreePlan& t = p.tree;
    TreeArgs& A = d->tree;
    A.b = d->b;
    A.hinv_tab = p.mscale.empty() ? d->hinv : nullptr;
    A.up_joint = (const int32_t*)(ws + f.t_up);
    A.child_off = (const int32_t*)(ws + f.t_coff);
    A.child_joint = (const int32_t*)(ws + f.t_cj);
    A.ws_off = (const int64_t*)(ws + f.t_wsoff);
    A.jnpts = (const int32_t*)(ws + f.t_jnpts);
    A.jchd = (const int32_t*)(ws + f.t_jchd);
    A.jy = (const double*)(ws + f.t_jy);
    A.group_off = (const int32_t*)(ws + f.t_goff);
    A.glev_ptr = (const int32_t*)(ws + f.t_glp);
    A.glev_off = (const int32_t*)(ws + f.t_glo);
    A.glev_nl = (const int32_t*)(ws + f.t_glnl);
    A.fo_off = (const int64_t*)(ws + f.t_fo);
    A.fo_str = (const int32_t*)(ws + f.t_fstr);
    A.parent = (const int32_t*)(ws + f.t_par);
    A.up_row = (const int32_t*)(ws + f.t_uprow);
    A.f0 = (double*)(ws + f.t_f0);
    A.cap = t.cap;
    A.Shat = (double*)(ws + f.t_shat);
    A.lam = (double*)(ws + f.t_lam);
    A.bscr = (double*)(ws + f.t_bscr);
    A.ws = (double*)(ws + f.t_ws);
    A.group0 = 0;
    A.front_rows = t.max_m;
    A.n = p.n;
    A.pt_off = (const int32_t*)(ws + f.t_ptoff);
    A.pt_code = (const int32_t*)(ws + f.t_ptcode);
    A.body_nn = (const int32_t*)(ws + f.t_nn);
    A.root_joint = (const int32_t*)(ws + f.t_rootj);
    A.root_slot = (const int32_t*)(ws + f.t_rslot);
    A.xbuf = (double*)(ws + f.t_xbuf);
    if ((e = put((int32_t*)A.root_joint, t.root_joint, st))) return e;
    if ((e = put((int32_t*)A.root_slot, t.root_slot, st))) return e;
    if ((e = put((int32_t*)A.pt_off, t.pt_off, st))) return e;
    if ((e = put((int32_t*)A.pt_code, t.pt_code, st))) return e;
    if ((e = put((int32_t*)A.body_nn, t.body_nn, st))) return e;
    if ((e = put((int32_t*)A.up_joint, t.up_joint, st))) return e;
    if ((e = put((int32_t*)A.child_off, t.child_off, st))) return e;
    if ((e = put((int32_t*)A.child_joint, t.child_joint, st))) return e;
    if ((e = put((int64_t*)A.ws_off, t.ws_off, st))) return e;
    if ((e = put((int32_t*)A.jnpts, t.jnpts, st))) return e;
    if ((e = put((int32_t*)A.jchd, t.jchd, st))) return e;
    if ((e = put((double*)A.jy, t.jy, st))) return e;
    if ((e = put((int32_t*)A.group_off, t.group_off, st))) return e;
    if ((e = put((int32_t*)A.glev_ptr, t.glev_ptr, st))) return e;
    if ((e = put((int32_t*)A.glev_off, t.glev_off, st))) return e;
    if ((e = put((int32_t*)A.glev_nl, t.glev_nl, st))) return e;
    if ((e = put((int64_t*)A.fo_off, t.fo_off, st))) return e;
    if ((e = put((int32_t*)A.fo_str, t.fo_str, st))) return e;
    if ((e = put((int32_t*)A.parent, t.parent, st))) return e;
    if ((e = put((int32_t*)A.up_row, t.up_row, st))) return e;
    if ((e = cudaMemsetAsync(A.lam, 0, sizeof(double) * 6 * std::max<int64_t>(1, p.n_joints), st))) return e;
  }
  if (p.solver == MABD_SOLVER_SPARSE || p.solver == MABD_SOLVER_LINE_GS) return sparse_upload(p, ws, st, d);
  return cudaSuccess;
}

cudaError_t prefactor_device(const Plan& p, const DevPtrs& d, double h, cudaStream_t st) {
  return launch_hinv_table(d.mats, (int)p.mats.size(), 1.0 / (h * h), d.hinv, st);
}

// Device error word: [0] flags (ERR_*, set by any kernel), [1] step index as the kernels saw it (unused by the host),
// [2] first step after which [0] was non-zero (set by step_end_kernel), [3] steps enqueued since the last reset.
__global__ void err_reset_kernel(int32_t* e) {
  e[0] = 0;
  e[1] = INT_MAX;
  e[2] = INT_MAX;
  e[3] = 0;
}

cudaError_t reset_err(const DevPtrs& d, cudaStream_t st) {
  err_reset_kernel<<<1, 1, 0, st>>>(d.err);
  return cudaGetLastError();
}

// The last node of every step (also inside a captured graph, where the step index cannot be a kernel argument):
// attributes a new error to this step and counts it.
__global__ void step_end_kernel(int32_t* e) {
  if (e[0] != 0 && e[2] == INT_MAX) e[2] = e[3];
  e[3] += 1;
}

cudaError_t launch_step_end(const Plan& p, const DevPtrs& d, cudaStream_t st) {
  if (p.step_end_folded) return cudaSuccess;  // done by the step's only kernel
  step_end_kernel<<<1, 1, 0, st>>>(d.err);
  return cudaGetLastError();
}

// one step of a multi-part chain scene for the parts [part_lo, part_hi) of this process
static cudaError_t launch_step_parts(const Plan& p, const DevPtrs& d, ChainArgs a, cudaStream_t st) {
  cudaError_t e;
  const StepConsts& k = a.k;
  if (k.phase == 2) goto after_exchange;  // host exchange: the caller has filled all_tops
  a.seg_list = d.local_windows;
  if ((e = launch_chain(a, (int)p.local_windows.size(), false, st))) return e;
  if (p.n_long == 0) return cudaSuccess;  // independent short chains (config 2): no exchange, nothing to finish
  for (int q = p.part_lo; q < p.part_hi; ++q) {
    const Plan::Part& P = p.parts[q];
    if (P.n1 == 0) continue;
    const Top* lvl = d.tops[0] + P.long_lo;
    if (P.btd1) {
      BtdArgs b{};
      b.top_in = lvl;
      b.left_iface = d.left_iface + P.long_lo;
      b.n_u = P.n1;
      b.mode = BTD_REDUCE;
      b.top_out = d.p_tops1[q];
      b.right_open = P.right_open;
      b.k = k;
      if ((e = launch_btd(b, (int)P.n2, st))) return e;
      lvl = d.p_tops1[q];
    }
    SeqArgs sq{};
    sq.top_in = lvl;
    sq.n = (int32_t)P.n2;
    sq.right_open = P.right_open;
    sq.top_out = d.all_tops + q;
    sq.scratch = d.p_scr[q];
    sq.k = k;
    if ((e = launch_seq_top(sq, st))) return e;
  }
  if (k.phase == 1) return cudaSuccess;  // host exchange: the caller all-gathers all_tops now
  if (p.use_nccl) {
    const int rc = nccl_allgather_doubles(d.nccl_comm, (double*)d.all_tops, sizeof(Top) / sizeof(double), p.part_lo, st);
    if (rc != 0) return nccl_step_failed(rc), cudaErrorUnknown;  // mabd_step reports MABD_ENCCL
  }
after_exchange:
  {
    BtdArgs b{};
    b.top_in = d.all_tops;
    b.left_iface = d.part_left_open;
    b.n_u = p.n_parts;
    b.mode = BTD_FUSED;
    b.lam_out = d.lam_g;
    b.k = k;
    if ((e = launch_btd(b, 1, st))) return e;
  }
  double* lam1 = d.lams[0];
  for (int q = p.part_lo; q < p.part_hi; ++q) {
    const Plan::Part& P = p.parts[q];
    if (P.n1 == 0) continue;
    if (P.right_open) {  // λ of the next part's first long window, for this part's last segment
      if ((e = cudaMemcpyAsync(lam1 + 3 * P.long_hi, d.lam_g + 3 * (q + 1), 3 * sizeof(double),
                               cudaMemcpyDeviceToDevice, st)))
        return e;
    }
    SeqArgs sq{};
    sq.top_in = P.btd1 ? d.p_tops1[q] : d.tops[0] + P.long_lo;
    sq.n = (int32_t)P.n2;
    sq.right_open = P.right_open;
    sq.scratch = d.p_scr[q];
    sq.lam_ends = d.lam_g + 3 * q;
    sq.lam_out = P.btd1 ? d.p_lam2[q] : lam1 + 3 * P.long_lo;
    sq.k = k;
    if ((e = launch_seq_finish(sq, st))) return e;
    if (P.btd1) {
      BtdArgs b{};
      b.top_in = d.tops[0] + P.long_lo;
      b.left_iface = d.left_iface + P.long_lo;
      b.n_u = P.n1;
      b.mode = BTD_FINISH;
      b.lam_in = d.p_lam2[q];
      b.lam_out = lam1 + 3 * P.long_lo;
      b.right_open = P.right_open;
      b.lam_remote = d.lam_g + 3 * (q + 1);
      b.k = k;
      if ((e = launch_btd(b, (int)P.n2, st))) return e;
    }
  }
  a.seg_list = d.local_long;
  a.lam_in = lam1;
  return launch_chain(a, (int)p.local_long.size(), true, st);
}

// K > 1 Newton iterations: iteration 0 is the plain step's linearisation at qⁿ (velocity
// form, gravity explicit); iteration i ≥ 1 is linearised at q⁽ⁱ⁾ with the velocity buffer holding
// v⁽ⁱ⁾ = (q̂ − q⁽ⁱ⁾)/h and zero explicit gravity (q̂ = qⁿ + hq̇ⁿ + h²[0;g] carries it). Each iteration's update
// writes q⁽ⁱ⁺¹⁾ = q⁽ⁱ⁾ + δq and v⁽ⁱ⁺¹⁾ = v⁽ⁱ⁾ − δq/h + h·grav (t-components); after the last one,
// q̇ⁿ⁺¹ = z − v⁽ᴷ⁾ with z = q̇ⁿ + h[0;g] saved before the first.
__global__ void iter_prep_kernel(const double* qd, double* z, int64_t ld, double h, double g0, double g1, double g2) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= 12 * ld) return;
  const int c = (int)(i / ld);
  z[i] = qd[i] + (c == 9 ? h * g0 : c == 10 ? h * g1 : c == 11 ? h * g2 : 0.0);
}
__global__ void iter_final_kernel(double* qd, const double* z, int64_t ld) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < 12 * ld) qd[i] = z[i] - qd[i];
}

static cudaError_t launch_iteration(const Plan& p, const DevPtrs& d, const StepConsts& k, cudaStream_t st);

static ChainArgs chain_args(const Plan& p, const DevPtrs& d, const StepConsts& k) {
  ChainArgs a;
  a.step_end = 0;
  a.nsteps = 1;
  a.b = d.b;
  a.slot_info = d.slot_info;
  a.geo = d.geo;
  a.seg_flags = d.seg_flags;
  a.seg_red = d.seg_red;
  a.seg_list = nullptr;
  a.hinv_tab = p.mscale.empty() ? d.hinv : nullptr;
  a.n_mats = (int32_t)p.mats.size();
  a.top_out = d.tops.empty() ? nullptr : d.tops[0];
  a.lam_in = d.lams.empty() ? nullptr : d.lams[0];
  a.k = k;
  return a;
}

static StepConsts step_consts(const Plan& p, const DevPtrs& d, double h, int32_t step, int phase) {
  StepConsts k;
  k.h = h;
  k.ih = 1.0 / h;
  k.ih2 = 1.0 / (h * h);
  for (int i = 0; i < 3; ++i) k.grav[i] = p.grav[i];
  k.step_index = step;
  k.err = d.err;
  k.iter = 0;
  k.niter = std::max(1, p.newton_iters);
  k.lp = p.rotation == MABD_ROTATION_LENGTH_PRESERVING ? 1 : 0;
  k.phase = phase;
  return k;
}

// nsteps steps of a one-warp chain scene (Plan::step_end_folded) in one launch: the state stays in the warp's
// registers between the steps and each step does its own step_end bookkeeping.
cudaError_t launch_steps_small(const Plan& p, const DevPtrs& d, double h, int32_t nsteps, cudaStream_t st) {
  if (!p.step_end_folded) return cudaErrorNotSupported;
  ChainArgs a = chain_args(p, d, step_consts(p, d, h, 0, 0));
  a.step_end = 1;
  a.nsteps = nsteps;
  return launch_small_chain(a, st);
}

cudaError_t launch_step(const Plan& p, const DevPtrs& d, double h, int32_t step, cudaStream_t st, int phase) {
  StepConsts k = step_consts(p, d, h, step, phase);
  if (k.niter == 1) return launch_iteration(p, d, k, st);
  const int64_t tot = 12 * d.b.ld;
  const unsigned grid = (unsigned)((tot + 255) / 256);
  iter_prep_kernel<<<grid, 256, 0, st>>>(d.b.qd, d.b.z, d.b.ld, h, p.grav[0], p.grav[1], p.grav[2]);
  cudaError_t e;
  for (int i = 0; i < k.niter; ++i) {
    k.iter = i;
    if (i == 1)
      for (int c = 0; c < 3; ++c) k.grav[c] = 0.0;
    if ((e = launch_iteration(p, d, k, st))) return e;
  }
  iter_final_kernel<<<grid, 256, 0, st>>>(d.b.qd, d.b.z, d.b.ld);
  return cudaGetLastError();
}

static cudaError_t forest_iteration(const Plan& p, const DevPtrs& d, const StepConsts& k, cudaStream_t st);

static cudaError_t launch_iteration(const Plan& p, const DevPtrs& d, const StepConsts& k, cudaStream_t st) {
  if (p.loop.active) return loop_step(p, d, k, st, forest_iteration);
  return forest_iteration(p, d, k, st);
}

static cudaError_t forest_iteration(const Plan& p, const DevPtrs& d, const StepConsts& k, cudaStream_t st) {
  if (p.solver == MABD_SOLVER_TREE) return tree_step(p, d, k, st);
  if (p.solver == MABD_SOLVER_SPARSE) return sparse_step(p, d, k, st);
  if (p.solver == MABD_SOLVER_LINE_GS) return gs_step(p, d, k, st);
  if (p.solver != MABD_SOLVER_CHAIN) return cudaErrorNotSupported;
  ChainArgs a = chain_args(p, d, k);
  if (p.n_parts > 1) return launch_step_parts(p, d, a, st);
  if (p.small_chain) {
    a.step_end = p.step_end_folded ? 1 : 0;
    return launch_small_chain(a, st);
  }
  cudaError_t e = launch_chain(a, (int)p.n_windows, false, st);
  if (e != cudaSuccess || p.n_long == 0) return e;
  const int nl = (int)p.levels.size();
  // levels i = 0..nl-1 (BTD level i+1): REDUCE for i < nl-1, FUSED at nl-1
  for (int i = 0; i < nl; ++i) {
    BtdArgs b{};
    b.top_in = d.tops[i];
    b.left_iface = (i == 0) ? d.left_iface : nullptr;
    b.n_u = p.levels[i].n_u;
    b.mode = p.levels[i].fused ? BTD_FUSED : BTD_REDUCE;
    b.top_out = p.levels[i].fused ? nullptr : d.tops[i + 1];
    b.lam_in = nullptr;
    b.lam_out = d.lams[i];
    b.k = k;
    if ((e = launch_btd(b, (int)p.levels[i].windows, st)) != cudaSuccess) return e;
  }
  for (int i = nl - 2; i >= 0; --i) {
    BtdArgs b{};
    b.top_in = d.tops[i];
    b.left_iface = (i == 0) ? d.left_iface : nullptr;
    b.n_u = p.levels[i].n_u;
    b.mode = BTD_FINISH;
    b.top_out = nullptr;
    b.lam_in = d.lams[i + 1];
    b.lam_out = d.lams[i];
    b.k = k;
    if ((e = launch_btd(b, (int)p.levels[i].windows, st)) != cudaSuccess) return e;
  }
  a.seg_list = d.long_list;
  return launch_chain(a, (int)p.n_long, true, st);
}

}  // namespace mabd
