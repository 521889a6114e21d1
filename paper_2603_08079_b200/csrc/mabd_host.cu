// libmabd.so host runtime: the C ABI of include/mabd.h.
//
// mabd_create: validates the scene, detects shared materials, classifies the joint topology (SURVEY §8(c)
// A14: forest of paths → chain solver, forest of trees → tree solver, otherwise sparse), orders bodies and
// joints for the chosen solver, and uploads everything into one device workspace.
// mabd_prefactor: per-material closed-form H̄⁻¹ and the solver plan.
// mabd_step: launches the step kernels nsteps times on the handle's stream (no host sync inside the loop).
#include <cuda_runtime.h>

#include <algorithm>
#include <climits>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <string>
#include <unordered_map>
#include <vector>

#include "../../include/mabd.h"
#include "mabd_kernels.h"
#include "mabd_plan.h"

using namespace mabd;

static thread_local std::string g_thread_err;

struct mabd_ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  std::string err;
  bool prefactored = false;
  double h_pref = 0.0;
  Plan plan;                 // host-side plan (kept for introspection / sizes)
  // device memory
  char* ws = nullptr;
  size_t ws_bytes = 0;
  bool own_ws = false;
  DevPtrs d;
  int32_t* h_err = nullptr;  // pinned [4]
  int64_t steps_done = 0;
  int64_t steps_pending = 0;   // enqueued by mabd_step_async since the last mabd_check
  bool use_graphs = true;      // options.no_graphs == 0 and a non-default stream
  double exchange_h = 0.0;     // a host-exchange step in progress (mabd_step_exchange_begin)
  cudaGraphExec_t graph = nullptr;
  double graph_h = 0.0;
};

static mabd_status fail(mabd_ctx* c, mabd_status st, const char* fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  if (c)
    c->err = buf;
  else
    g_thread_err = buf;
  return st;
}

// One step as a CUDA graph (captured on the handle's stream at the first step after create / prefactor /
// set_wrench, replayed nsteps times): the plan's launch sequence plus the step_end node. Kernel arguments (h, the
// pointers, the wrench) are baked into the graph, so it is rebuilt when any of them changes.
static void drop_graph(mabd_ctx* c) {
  if (c->graph) cudaGraphExecDestroy(c->graph);
  c->graph = nullptr;
}

#define CUDA_TRY(c, expr)                                                                          \
  do {                                                                                             \
    cudaError_t e_ = (expr);                                                                       \
    if (e_ != cudaSuccess) return fail((c), MABD_ECUDA, "%s: %s", #expr, cudaGetErrorString(e_)); \
  } while (0)

extern "C" {

mabd_status mabd_workspace_size(const mabd_bodies* bodies, const mabd_joints* joints, const mabd_options* opts,
                                size_t* bytes) {
  if (!bytes) return fail(nullptr, MABD_EINVAL, "bytes is NULL");
  Plan p;
  std::string msg;
  mabd_status st = build_plan(bodies, joints, opts, &p, &msg);
  if (st != MABD_OK) return fail(nullptr, st, "%s", msg.c_str());
  *bytes = p.workspace_bytes;
  return MABD_OK;
}

mabd_status mabd_create(const mabd_bodies* bodies, const mabd_joints* joints, const mabd_options* opts,
                        mabd_handle* out) {
  if (!out) return fail(nullptr, MABD_EINVAL, "out is NULL");
  *out = nullptr;
  mabd_ctx* c = new mabd_ctx();
  std::string msg;
  mabd_status st = build_plan(bodies, joints, opts, &c->plan, &msg);
  if (st != MABD_OK) {
    delete c;
    return fail(nullptr, st, "%s", msg.c_str());
  }
  cudaError_t e = cudaGetDevice(&c->device);
  if (e != cudaSuccess) {
    delete c;
    return fail(nullptr, MABD_ECUDA, "cudaGetDevice: %s", cudaGetErrorString(e));
  }
  c->stream = opts ? (cudaStream_t)opts->cuda_stream : nullptr;
  if (opts && opts->workspace) {
    if (opts->workspace_bytes < c->plan.workspace_bytes) {
      size_t need = c->plan.workspace_bytes;
      delete c;
      return fail(nullptr, MABD_ENOMEM, "workspace too small: %zu < %zu bytes", opts->workspace_bytes, need);
    }
    c->ws = (char*)opts->workspace;
    c->ws_bytes = opts->workspace_bytes;
  } else {
    e = cudaMalloc(&c->ws, c->plan.workspace_bytes);
    if (e != cudaSuccess) {
      delete c;
      return fail(nullptr, MABD_ENOMEM, "cudaMalloc(%zu): %s", c->plan.workspace_bytes, cudaGetErrorString(e));
    }
    c->own_ws = true;
    c->ws_bytes = c->plan.workspace_bytes;
  }
  c->use_graphs = c->stream != nullptr && !(opts && opts->no_graphs);
  e = cudaMallocHost(&c->h_err, 4 * sizeof(int32_t));
  if (e == cudaSuccess) e = chain_kernels_init();
  if (e == cudaSuccess && (c->plan.solver == MABD_SOLVER_SPARSE || c->plan.solver == MABD_SOLVER_LINE_GS))
    e = sparse_init();
  if (e == cudaSuccess && c->plan.solver == MABD_SOLVER_TREE) e = tree_init();
  if (e == cudaSuccess) e = upload_plan(c->plan, c->ws, c->stream, &c->d);
  if (e == cudaSuccess) e = reset_err(c->d, c->stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(c->stream);
  if (e != cudaSuccess) {
    mabd_destroy(c);
    return fail(nullptr, MABD_ECUDA, "create: %s", cudaGetErrorString(e));
  }
  if (c->plan.use_nccl) {  // collective: every rank of the world calls mabd_create
    std::string why;
    if (!nccl_load(&why)) {
      mabd_destroy(c);
      return fail(nullptr, MABD_ENCCL, "%s", why.c_str());
    }
    const int rc = nccl_comm_init(&c->d.nccl_comm, opts->world, opts->nccl_unique_id, opts->rank);
    if (rc != 0) {
      mabd_destroy(c);
      return fail(nullptr, MABD_ENCCL, "ncclCommInitRank: %s", nccl_err(rc));
    }
  }
  *out = c;
  return MABD_OK;
}

mabd_status mabd_prefactor(mabd_handle c, double h) {
  if (!c) return fail(nullptr, MABD_EINVAL, "NULL handle");
  if (!(h > 0.0) || !std::isfinite(h)) return fail(c, MABD_EINVAL, "h must be > 0 (got %g)", h);
  CUDA_TRY(c, cudaSetDevice(c->device));
  CUDA_TRY(c, prefactor_device(c->plan, c->d, h, c->stream));
  drop_graph(c);
  c->prefactored = true;
  c->h_pref = h;
  return MABD_OK;
}

static cudaError_t enqueue_one_step(mabd_ctx* c, double h, int32_t s) {
  cudaError_t e = launch_step(c->plan, c->d, h, s, c->stream);
  if (e == cudaSuccess) e = launch_step_end(c->plan, c->d, c->stream);
  return e;
}

static cudaError_t build_graph(mabd_ctx* c, double h) {
  drop_graph(c);
  cudaError_t e = cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeThreadLocal);
  if (e != cudaSuccess) return e;
  const cudaError_t e1 = enqueue_one_step(c, h, 0);
  cudaGraph_t g = nullptr;
  e = cudaStreamEndCapture(c->stream, &g);
  if (e1 != cudaSuccess || e != cudaSuccess) {
    if (g) cudaGraphDestroy(g);
    return e1 != cudaSuccess ? e1 : e;
  }
  e = cudaGraphInstantiate(&c->graph, g, 0);
  cudaGraphDestroy(g);
  if (e != cudaSuccess) c->graph = nullptr;
  c->graph_h = h;
  return e;
}

static mabd_status enqueue_steps(mabd_ctx* c, double h, int64_t nsteps) {
  if (!c->prefactored) return fail(c, MABD_ESTATE, "mabd_step before mabd_prefactor");
  if (!(h > 0.0) || !std::isfinite(h)) return fail(c, MABD_EINVAL, "h must be > 0 (got %g)", h);
  if (nsteps < 0) return fail(c, MABD_EINVAL, "nsteps < 0");
  if (nsteps == 0) return MABD_OK;
  CUDA_TRY(c, cudaSetDevice(c->device));
  if (h != c->h_pref) {
    mabd_status st = mabd_prefactor(c, h);
    if (st != MABD_OK) return st;
  }
  nccl_take_step_error();
  if (c->plan.step_end_folded && nsteps > 1) {  // one-warp chain scene: all the call's steps in one launch
    for (int64_t s0 = 0; s0 < nsteps; s0 += INT_MAX) {
      const cudaError_t e = launch_steps_small(c->plan, c->d, h, (int32_t)std::min<int64_t>(nsteps - s0, INT_MAX),
                                               c->stream);
      if (e != cudaSuccess) return fail(c, MABD_ECUDA, "launch_steps_small: %s", cudaGetErrorString(e));
    }
    c->steps_pending += nsteps;
    return MABD_OK;
  }
  const bool graphs = c->use_graphs;
  if (graphs && (!c->graph || c->graph_h != h)) {
    const cudaError_t e = build_graph(c, h);
    if (e != cudaSuccess) {
      if (const int rc = nccl_take_step_error()) return fail(c, MABD_ENCCL, "NCCL exchange (capture): %s", nccl_err(rc));
      return fail(c, MABD_ECUDA, "step graph capture: %s", cudaGetErrorString(e));
    }
  }
  for (int64_t s = 0; s < nsteps; ++s) {
    const cudaError_t e = graphs ? cudaGraphLaunch(c->graph, c->stream)
                                 : enqueue_one_step(c, h, (int32_t)std::min<int64_t>(s, INT_MAX - 1));
    if (e != cudaSuccess) {
      if (const int rc = nccl_take_step_error())
        return fail(c, MABD_ENCCL, "NCCL exchange in step %lld of this call: %s", (long long)s, nccl_err(rc));
      return fail(c, MABD_ECUDA, "launch_step (step %lld of this call): %s", (long long)s, cudaGetErrorString(e));
    }
  }
  c->steps_pending += nsteps;
  return MABD_OK;
}

mabd_status mabd_check(mabd_handle c) {
  if (!c) return fail(nullptr, MABD_EINVAL, "NULL handle");
  CUDA_TRY(c, cudaSetDevice(c->device));
  CUDA_TRY(c, cudaMemcpyAsync(c->h_err, c->d.err, 4 * sizeof(int32_t), cudaMemcpyDeviceToHost, c->stream));
  CUDA_TRY(c, cudaStreamSynchronize(c->stream));
  const int64_t pending = c->steps_pending;
  c->steps_done += pending;
  c->steps_pending = 0;
  const int32_t flags = c->h_err[0], at = c->h_err[2];
  CUDA_TRY(c, reset_err(c->d, c->stream));
  if (flags & ERR_NONFINITE)
    return fail(c, MABD_ENONFINITE, "non-finite state or det(A) <= 1e-9 at step %d of the %lld steps enqueued",
                at, (long long)pending);
  if (flags & ERR_SINGULAR)
    return fail(c, MABD_ESINGULAR,
                "dual matrix not positive definite (redundant joints?) at step %d of the %lld steps enqueued", at,
                (long long)pending);
  return MABD_OK;
}

mabd_status mabd_step_async(mabd_handle c, double h, int64_t nsteps) {
  if (!c) return fail(nullptr, MABD_EINVAL, "NULL handle");
  if (c->plan.host_exchange && nsteps > 0)
    return fail(c, MABD_ESTATE, "host_exchange: step with mabd_step_exchange_begin / end");
  return enqueue_steps(c, h, nsteps);
}

// ---- caller-driven exchange (options.host_exchange; SURVEY §8(e) split scenes without NCCL)
static mabd_status exchange_view(mabd_ctx* c, double** buf, int64_t* per_rank, int32_t* ranks, int32_t* slot) {
  const Plan& p = c->plan;
  if (p.solver == MABD_SOLVER_CHAIN && p.n_parts > 1) {
    *buf = (double*)c->d.all_tops;
    *per_rank = sizeof(Top) / sizeof(double);
    *ranks = p.n_parts;
    *slot = p.part_lo;
    return MABD_OK;
  }
  if (p.solver == MABD_SOLVER_TREE && p.tree.parts > 1) {
    *buf = c->d.tree.xbuf;
    *per_rank = (int64_t)p.tree.rpp * TREE_TSLOT;
    *ranks = p.tree.parts;
    *slot = p.tree.part;
    return MABD_OK;
  }
  return fail(c, MABD_ESTATE, "no exchange: the scene is not split across ranks");
}

mabd_status mabd_exchange_info(mabd_handle c, int64_t* doubles_per_rank, int32_t* ranks, int32_t* my_slot) {
  if (!c || !doubles_per_rank || !ranks || !my_slot) return fail(c, MABD_EINVAL, "NULL argument");
  double* buf;
  return exchange_view(c, &buf, doubles_per_rank, ranks, my_slot);
}

mabd_status mabd_exchange_copy(mabd_handle c, double* host_all, int32_t to_device) {
  if (!c || !host_all) return fail(c, MABD_EINVAL, "NULL argument");
  double* buf;
  int64_t per;
  int32_t ranks, slot;
  mabd_status st = exchange_view(c, &buf, &per, &ranks, &slot);
  if (st != MABD_OK) return st;
  CUDA_TRY(c, cudaSetDevice(c->device));
  if (to_device)
    CUDA_TRY(c, cudaMemcpyAsync(buf, host_all, sizeof(double) * per * ranks, cudaMemcpyHostToDevice, c->stream));
  else
    CUDA_TRY(c, cudaMemcpyAsync(host_all + per * slot, buf + per * slot, sizeof(double) * per,
                                cudaMemcpyDeviceToHost, c->stream));
  CUDA_TRY(c, cudaStreamSynchronize(c->stream));
  return MABD_OK;
}

mabd_status mabd_step_exchange_begin(mabd_handle c, double h) {
  if (!c) return fail(nullptr, MABD_EINVAL, "NULL handle");
  if (!c->plan.host_exchange) return fail(c, MABD_ESTATE, "options.host_exchange is not set");
  if (!c->prefactored) return fail(c, MABD_ESTATE, "step before mabd_prefactor");
  if (!(h > 0.0) || !std::isfinite(h)) return fail(c, MABD_EINVAL, "h must be > 0 (got %g)", h);
  CUDA_TRY(c, cudaSetDevice(c->device));
  if (h != c->h_pref) {
    mabd_status st = mabd_prefactor(c, h);
    if (st != MABD_OK) return st;
  }
  c->exchange_h = h;
  CUDA_TRY(c, launch_step(c->plan, c->d, h, 0, c->stream, 1));
  CUDA_TRY(c, cudaStreamSynchronize(c->stream));
  return MABD_OK;
}

mabd_status mabd_step_exchange_end(mabd_handle c) {
  if (!c) return fail(nullptr, MABD_EINVAL, "NULL handle");
  if (!(c->exchange_h > 0.0)) return fail(c, MABD_ESTATE, "mabd_step_exchange_end without begin");
  CUDA_TRY(c, cudaSetDevice(c->device));
  CUDA_TRY(c, launch_step(c->plan, c->d, c->exchange_h, 0, c->stream, 2));
  CUDA_TRY(c, launch_step_end(c->plan, c->d, c->stream));
  c->exchange_h = 0.0;
  c->steps_pending += 1;
  return mabd_check(c);
}

mabd_status mabd_step(mabd_handle c, double h, int64_t nsteps) {
  if (!c) return fail(nullptr, MABD_EINVAL, "NULL handle");
  if (c->plan.host_exchange && nsteps > 0)
    return fail(c, MABD_ESTATE, "host_exchange: step with mabd_step_exchange_begin / end");
  const mabd_status st = enqueue_steps(c, h, nsteps);
  if (st != MABD_OK) return st;
  if (nsteps == 0 && c->steps_pending == 0) return MABD_OK;
  return mabd_check(c);
}

mabd_status mabd_get_state(mabd_handle c, double* q_out, double* qd_out, int out_on_device) {
  if (!c) return fail(nullptr, MABD_EINVAL, "NULL handle");
  CUDA_TRY(c, cudaSetDevice(c->device));
  const int64_t n = c->plan.n;
  if (c->plan.use_nccl) {  // every rank advanced only its windows: share them (outside any timed loop)
    std::vector<std::pair<int64_t, int64_t>> ranges;
    if (c->plan.solver == MABD_SOLVER_TREE) {  // each rank advanced its bottom groups (the top is replicated)
      const TreePlan& t = c->plan.tree;
      for (int r = 0; r < t.parts; ++r) {
        const int lo = std::min(t.n_bottom, r * t.gpr), hi = std::min(t.n_bottom, (r + 1) * t.gpr);
        ranges.push_back({t.group_off[lo], t.group_off[hi]});
      }
    } else {
      for (const auto& P : c->plan.parts) ranges.push_back({P.win_lo * SEG, P.win_hi * SEG});
    }
    int rc = nccl_bcast_ranges(c->d.nccl_comm, c->d.b.q, ranges, c->d.b.ld, 12, c->stream);
    if (rc == 0) rc = nccl_bcast_ranges(c->d.nccl_comm, c->d.b.qd, ranges, c->d.b.ld, 12, c->stream);
    if (rc != 0) return fail(c, MABD_ENCCL, "state broadcast: %s", nccl_err(rc));
  }
  double* dq = out_on_device ? q_out : (q_out ? c->d.io : nullptr);
  double* dqd = out_on_device ? qd_out : (qd_out ? c->d.io + 12 * n : nullptr);
  CUDA_TRY(c, launch_gather(c->d.b.q, c->d.b.qd, c->d.b.ld, c->d.perm, n, c->d.frame, dq, dqd, c->stream));
  if (!out_on_device) {
    if (q_out) CUDA_TRY(c, cudaMemcpyAsync(q_out, dq, 12 * n * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
    if (qd_out)
      CUDA_TRY(c, cudaMemcpyAsync(qd_out, dqd, 12 * n * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
  }
  CUDA_TRY(c, cudaStreamSynchronize(c->stream));
  return MABD_OK;
}

mabd_status mabd_set_state(mabd_handle c, const double* q, const double* qd, int in_on_device) {
  if (!c) return fail(nullptr, MABD_EINVAL, "NULL handle");
  CUDA_TRY(c, cudaSetDevice(c->device));
  const int64_t n = c->plan.n;
  const double* sq = q;
  const double* sqd = qd;
  if (!in_on_device) {
    if (q) {
      CUDA_TRY(c, cudaMemcpyAsync(c->d.io, q, 12 * n * sizeof(double), cudaMemcpyHostToDevice, c->stream));
      sq = c->d.io;
    }
    if (qd) {
      CUDA_TRY(c, cudaMemcpyAsync(c->d.io + 12 * n, qd, 12 * n * sizeof(double), cudaMemcpyHostToDevice, c->stream));
      sqd = c->d.io + 12 * n;
    }
  }
  CUDA_TRY(c, launch_scatter(c->d.b.q, c->d.b.qd, c->d.b.ld, c->d.perm, n, c->d.frame, sq, sqd, c->stream));
  if (!in_on_device) CUDA_TRY(c, cudaStreamSynchronize(c->stream));
  return MABD_OK;
}

mabd_status mabd_set_wrench(mabd_handle c, const double* W, int in_on_device) {
  if (!c) return fail(nullptr, MABD_EINVAL, "NULL handle");
  if (c->plan.loop.active)
    return fail(c, MABD_EUNSUPPORTED, "external wrenches are not available with the loop-breaker solver");
  CUDA_TRY(c, cudaSetDevice(c->device));
  const double* wr = nullptr;
  if (W) {
    const int64_t n = c->plan.n;
    const double* src = W;
    if (!in_on_device) {
      CUDA_TRY(c, cudaMemcpyAsync(c->d.io, W, 6 * n * sizeof(double), cudaMemcpyHostToDevice, c->stream));
      src = c->d.io;
    }
    CUDA_TRY(c, cudaMemsetAsync(c->d.wr_buf, 0, 9 * c->d.b.ld * sizeof(double), c->stream));
    CUDA_TRY(c, launch_scatter_rows(c->d.wr_buf, c->d.b.ld, c->d.perm, n, src, 6, c->stream));
    CUDA_TRY(c, launch_wrench_point(c->d.wr_buf, c->d.b.ld, c->d.perm, n, c->d.frame, c->stream));
    if (!in_on_device) CUDA_TRY(c, cudaStreamSynchronize(c->stream));
    wr = c->d.wr_buf;
  }
  drop_graph(c);   // the wrench pointer is a kernel argument baked into the step graph
  c->d.b.wr = wr;  // every solver reads the wrench through its copy of the body arrays
  c->d.tree.b.wr = wr;
  c->d.sparse.b.wr = wr;
  return MABD_OK;
}

mabd_status mabd_query(mabd_handle c, int32_t* solver, int32_t* launches_per_step, int64_t* n_bodies,
                       int64_t* n_dual_rows) {
  if (!c) return fail(nullptr, MABD_EINVAL, "NULL handle");
  if (solver) *solver = c->plan.loop.active ? MABD_SOLVER_LOOP_BREAKER : c->plan.solver;
  if (launches_per_step)  // + the step_end node (folded into the one-warp chain kernel when that runs alone)
    *launches_per_step = c->plan.launches_per_step + (c->plan.step_end_folded ? 0 : 1);
  if (n_bodies) *n_bodies = c->plan.n;
  if (n_dual_rows) *n_dual_rows = c->plan.n_dual_rows;
  return MABD_OK;
}

mabd_status mabd_solver_stats(mabd_handle c, int64_t* last_iterations) {
  if (!c) return fail(nullptr, MABD_EINVAL, "NULL handle");
  if (!last_iterations) return fail(c, MABD_EINVAL, "last_iterations is NULL");
  *last_iterations = 0;
  if (c->plan.solver == MABD_SOLVER_SPARSE || c->plan.solver == MABD_SOLVER_LINE_GS) {
    int32_t it = 0;
    CUDA_TRY(c, cudaSetDevice(c->device));
    CUDA_TRY(c, cudaMemcpyAsync(&it, c->d.sparse.iters, sizeof(int32_t), cudaMemcpyDeviceToHost, c->stream));
    CUDA_TRY(c, cudaStreamSynchronize(c->stream));
    *last_iterations = it;
  }
  return MABD_OK;
}

// developer probe (not in the header): the line Gauss-Seidel residual history of the last step
// (out[0] = max|r|, then per sweep max|r − Sλ|, max|Sλ|); returns the number of doubles written
int mabd_dbg_gs_trace(mabd_handle c, double* out, int n) {
  if (!c || c->plan.solver != MABD_SOLVER_LINE_GS) return 0;
  const int m = std::min(n, 1 + 2 * c->plan.sparse.gs_sweeps);
  cudaMemcpyAsync(out, c->d.sparse.gs.resmax, sizeof(double) * m, cudaMemcpyDeviceToHost, c->stream);
  cudaStreamSynchronize(c->stream);
  return m;
}

// developer probe (not in the header): the sparse solver's last max|r − Sλ| / max|r| before a refinement pass
int mabd_dbg_refine_ratio(mabd_handle c, double* out) {
  if (!c || c->plan.solver != MABD_SOLVER_SPARSE || !c->d.sparse.rmax) return 0;
  cudaMemcpyAsync(out, c->d.sparse.rmax + 2, sizeof(double), cudaMemcpyDeviceToHost, c->stream);
  cudaStreamSynchronize(c->stream);
  return 1;
}

mabd_status mabd_nccl_unique_id(void* out, size_t bytes) {
  if (!out || bytes < 128) return fail(nullptr, MABD_EINVAL, "need a 128-byte buffer");
  std::string why;
  if (!nccl_load(&why)) return fail(nullptr, MABD_ENCCL, "%s", why.c_str());
  const int rc = nccl_unique_id(out);
  if (rc != 0) return fail(nullptr, MABD_ENCCL, "ncclGetUniqueId: %s", nccl_err(rc));
  return MABD_OK;
}

mabd_status mabd_partition_info(const mabd_bodies* bodies, const mabd_joints* joints, const mabd_options* opts,
                                int64_t* out, int64_t n_out) {
  if (!out || n_out < 10) return fail(nullptr, MABD_EINVAL, "need 10 output slots");
  Plan p;
  std::string msg;
  mabd_status st = build_plan(bodies, joints, opts, &p, &msg);
  if (st != MABD_OK) return fail(nullptr, st, "%s", msg.c_str());
  const int r = opts && opts->world > 1 ? opts->rank : 0;
  out[0] = p.n_parts;
  out[1] = p.n_windows;
  out[2] = p.n_long;
  if (p.n_parts > 1) {
    const auto& P = p.parts[r];
    out[3] = P.win_lo; out[4] = P.win_hi; out[5] = P.long_lo; out[6] = P.long_hi;
    out[7] = P.left_open; out[8] = P.right_open; out[9] = P.n2;
  } else {
    out[3] = 0; out[4] = p.n_windows; out[5] = 0; out[6] = p.n_long; out[7] = 0; out[8] = 0; out[9] = 0;
  }
  if (n_out >= 20) {  // tree split: solver, parts, bottom groups, groups per part, gather slots per part, this
                      // part's group range and body range, first top body, joints into the bottom groups
    for (int i = 10; i < 20; ++i) out[i] = 0;
    out[10] = p.solver;
    if (p.solver == MABD_SOLVER_TREE) {
      const TreePlan& t = p.tree;
      const int lo = std::min(t.n_bottom, t.part * t.gpr), hi = std::min(t.n_bottom, (t.part + 1) * t.gpr);
      out[11] = t.parts; out[12] = t.n_bottom; out[13] = t.gpr; out[14] = t.rpp;
      out[15] = lo; out[16] = hi; out[17] = t.group_off[lo]; out[18] = t.group_off[hi];
      out[19] = t.parts > 1 ? (int64_t)t.root_joint.size() : 0;
    }
  }
  return MABD_OK;
}

mabd_status mabd_destroy(mabd_handle c) {
  if (!c) return MABD_OK;
  cudaSetDevice(c->device);
  if (c->stream) cudaStreamSynchronize(c->stream);
  drop_graph(c);
  nccl_comm_destroy(c->d.nccl_comm);
  if (c->own_ws && c->ws) cudaFree(c->ws);
  if (c->h_err) cudaFreeHost(c->h_err);
  delete c;
  return MABD_OK;
}

const char* mabd_last_error(mabd_handle c) {
  if (c) return c->err.c_str();
  return g_thread_err.c_str();
}

}  // extern "C"
