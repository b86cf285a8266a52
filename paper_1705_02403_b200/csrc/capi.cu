// capi.cu -- the C ABI of include/gmt_b200.h: contexts, device-resident
// instances, single and batched GMT* solves.  Host code here only marshals
// (validation, pointer arithmetic, cudaMemcpyAsync); every computation on
// the path runs in the CUDA kernels of solve.cu / graph.cu / sample.cu.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "common.cuh"
#include "gmt_b200.h"
#include "internal.cuh"
#include "solve.cuh"

using namespace gmtb;

// ---- errors ---------------------------------------------------------------
namespace gmtb {
thread_local std::string g_last_error;

int set_error(int code, const std::string& msg) {
  g_last_error = msg;
  return code;
}

int cuda_error(cudaError_t e, const char* what) {
  return set_error(GMT_E_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}
}  // namespace gmtb

#define GMT_CUDA(call)                                     \
  do {                                                     \
    cudaError_t _e = (call);                               \
    if (_e != cudaSuccess) return cuda_error(_e, #call);   \
  } while (0)

#define GMT_TRY(call)          \
  do {                         \
    int _rc = (call);          \
    if (_rc != GMT_OK) return _rc; \
  } while (0)

// ---- device arena -----------------------------------------------------------
namespace gmtb {

thread_local cudaStream_t g_alloc_stream = nullptr;

AllocScope::AllocScope(gmt_ctx* ctx) : prev(g_alloc_stream) {
  g_alloc_stream = ctx ? ctx->stream : nullptr;
}

int Arena::reserve(size_t bytes) {
  if (bytes <= cap) return GMT_OK;
  release();
  size_t want = std::max(bytes, static_cast<size_t>(1) << 20);
  const cudaError_t e = g_alloc_stream ? cudaMallocAsync(&ptr, want, g_alloc_stream) : cudaMalloc(&ptr, want);
  if (e != cudaSuccess) {
    ptr = nullptr;
    return cuda_error(e, "device allocation");
  }
  cap = want;
  return GMT_OK;
}

void Arena::release() {
  if (ptr) {
    if (g_alloc_stream)
      cudaFreeAsync(ptr, g_alloc_stream);
    else
      cudaFree(ptr);
  }
  ptr = nullptr;
  cap = 0;
}

int HostPinned::reserve(size_t bytes) {
  if (bytes <= cap) return GMT_OK;
  if (ptr) cudaFreeHost(ptr);
  ptr = nullptr;
  cap = 0;
  size_t want = std::max(bytes, static_cast<size_t>(1) << 16);
  cudaError_t e = cudaHostAlloc(&ptr, want, cudaHostAllocDefault);
  if (e != cudaSuccess) return cuda_error(e, "cudaHostAlloc");
  cap = want;
  return GMT_OK;
}

void HostPinned::release() {
  if (ptr) cudaFreeHost(ptr);
  ptr = nullptr;
  cap = 0;
}

}  // namespace gmtb

// Sequential carving of one allocation into 16-byte aligned sections.
struct Carver {
  size_t off = 0;
  template <typename T>
  size_t take(size_t count) {
    size_t o = off;
    off = align16(off + sizeof(T) * count);
    return o;
  }
};

template <typename T>
static T* at(void* base, size_t off) {
  return reinterpret_cast<T*>(static_cast<char*>(base) + off);
}

// ---- context ----------------------------------------------------------------
extern "C" const char* gmt_last_error(void) { return g_last_error.c_str(); }
extern "C" int gmt_abi_version(void) { return GMT_B200_ABI_VERSION; }

extern "C" int gmt_struct_sizes(int64_t* out, int32_t count) {
  const int64_t sizes[] = {sizeof(gmt_scene),        sizeof(gmt_sample_source), sizeof(gmt_graph_view),
                           sizeof(gmt_plan_out),     sizeof(gmt_plan_summary),  sizeof(gmt_problem),
                           sizeof(gmt_di_params),    sizeof(gmt_batch_host),    sizeof(gmt_quad_params),
                           sizeof(gmt_scenario),     sizeof(gmt_trial_outcome), sizeof(gmt_dubins_params)};
  const int32_t n = static_cast<int32_t>(sizeof(sizes) / sizeof(sizes[0]));
  for (int32_t i = 0; i < count && i < n; ++i) out[i] = sizes[i];
  return n;
}

extern "C" int gmt_ctx_create(int device, gmt_ctx** out) {
  *out = nullptr;
  int count = 0;
  cudaError_t e = cudaGetDeviceCount(&count);
  if (e != cudaSuccess || count == 0) {
    return set_error(GMT_E_NO_DEVICE, std::string("no CUDA device: ") +
                                          (e != cudaSuccess ? cudaGetErrorString(e) : "0 devices"));
  }
  if (device < 0 || device >= count) return set_error(GMT_E_INVALID_INPUT, "device out of range");
  cudaDeviceProp prop;
  GMT_CUDA(cudaGetDeviceProperties(&prop, device));
  if (prop.major != 10) {
    return set_error(GMT_E_NO_DEVICE, std::string("device ") + prop.name +
                                          " is not sm_100 (Blackwell B200); this library is built "
                                          "for sm_100a only");
  }
  GMT_CUDA(cudaSetDevice(device));
  {  // keep freed pool memory for reuse instead of returning it at every sync
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
      uint64_t keep = UINT64_MAX;
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
    }
  }
  auto* ctx = new gmt_ctx;
  ctx->device = device;
  ctx->sm_count = prop.multiProcessorCount;
  ctx->smem_optin = prop.sharedMemPerBlockOptin;
  e = cudaMalloc(&ctx->counters, sizeof(int64_t) * 16);  // [0..2] traffic, [4..15] phase timing (debug)
  if (e == cudaSuccess) e = cudaMemset(ctx->counters, 0, sizeof(int64_t) * 16);
  if (e != cudaSuccess) {
    delete ctx;
    return cuda_error(e, "counters");
  }
  e = cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking);
  if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&ctx->copy_stream, cudaStreamNonBlocking);
  for (int k = 0; k < kMaxCopyChunks && e == cudaSuccess; ++k)
    e = cudaEventCreateWithFlags(&ctx->copy_done[k], cudaEventDisableTiming);
  if (e != cudaSuccess) {
    delete ctx;
    return cuda_error(e, "cudaStreamCreate");
  }
  *out = ctx;
  return GMT_OK;
}

extern "C" void gmt_ctx_destroy(gmt_ctx* ctx) {
  if (!ctx) return;
  cudaSetDevice(ctx->device);
  cudaStreamSynchronize(ctx->stream);
  {
    AllocScope scope(ctx);
    ctx->res.release();
    ctx->scratch.release();
    ctx->jobs.release();
    ctx->pp_work.release();
    ctx->pool_work.release();
    ctx->pool_rows.release();
    ctx->pool_res.release();
    ctx->gstate.release();
    destroy_pool(ctx->pool);
    ctx->pool = nullptr;
    ctx->plan_inst.mem.release();
    ctx->plan_inst.desc_mem.release();
    ctx->plan_inst.aux.release();
    ctx->plan_inst.mem2.release();
    ctx->plan_inst.mem3.release();
  }
  cudaStreamSynchronize(ctx->stream);
  ctx->pinned.release();
  ctx->pinned2.release();
  ctx->pinned_jobs.release();
  ctx->pool_pinned.release();
  cudaFree(ctx->counters);
  for (int k = 0; k < kMaxCopyChunks; ++k)
    if (ctx->copy_done[k]) cudaEventDestroy(ctx->copy_done[k]);
  if (ctx->copy_stream) cudaStreamDestroy(ctx->copy_stream);
  cudaStreamDestroy(ctx->stream);
  delete ctx;
}

extern "C" void* gmt_ctx_stream(gmt_ctx* ctx) { return ctx ? ctx->stream : nullptr; }

extern "C" int gmt_ctx_synchronize(gmt_ctx* ctx) {
  gmtb::AllocScope alloc_scope_(ctx);
  GMT_CUDA(cudaStreamSynchronize(ctx->stream));
  return GMT_OK;
}

extern "C" int64_t gmt_launch_count(const gmt_ctx* ctx) { return ctx ? ctx->launches : 0; }

extern "C" int gmt_ctx_set_option(gmt_ctx* ctx, int option, int64_t value) {
  gmtb::AllocScope alloc_scope_(ctx);
  switch (option) {
    case GMT_OPT_CLUSTER:
      if (value != 0 && value != 1 && value != 2 && value != 4 && value != 8 && value != 16)
        return set_error(GMT_E_INVALID_INPUT, "cluster size must be 0, 1, 2, 4, 8 or 16");
      ctx->cluster = static_cast<int>(value);
      return GMT_OK;
    case GMT_OPT_THREADS:
    case GMT_OPT_BATCH_THREADS: {
      const int cap = 512;  // <= 256: narrow CTA shape, above: wide (solve.cu)
      // (768: the 24-warp batched double-integrator shape, GMT_OPT_BATCH_THREADS only)
      const bool di24 = option == GMT_OPT_BATCH_THREADS && value == 768;
      if (value != 0 && !di24 && (value < 32 || value > cap || value % 32 != 0))
        return set_error(GMT_E_INVALID_INPUT, "threads must be 0, a multiple of 32 up to " +
                                                  std::to_string(cap) + ", or 768 (batched 6D)");
      (option == GMT_OPT_THREADS ? ctx->threads : ctx->batch_threads) = static_cast<int>(value);
      return GMT_OK;
    }
    case GMT_OPT_COUNTERS:
      ctx->counting = value ? 1 : 0;
      return GMT_OK;
    case GMT_OPT_BATCH_CLUSTER:
      if (value != 0 && value != 1 && value != 2 && value != 4 && value != 8 && value != 16)
        return set_error(GMT_E_INVALID_INPUT, "batch cluster size must be 0 (auto), 1, 2, 4, 8 or 16");
      ctx->batch_cluster = static_cast<int>(value);
      return GMT_OK;
    default:
      return set_error(GMT_E_INVALID_INPUT, "unknown option");
  }
}

extern "C" int gmt_ctx_counters(gmt_ctx* ctx, int64_t* out, int32_t reset) {
  gmtb::AllocScope alloc_scope_(ctx);
  GMT_CUDA(cudaStreamSynchronize(ctx->stream));
#ifdef GMT_PHASE_TIMING  // debug builds: out[4..15] = per-phase clock sums
  GMT_CUDA(cudaMemcpy(out, ctx->counters, sizeof(int64_t) * 16, cudaMemcpyDeviceToHost));
#else
  GMT_CUDA(cudaMemcpy(out, ctx->counters, sizeof(int64_t) * 3, cudaMemcpyDeviceToHost));
#endif
  if (reset) GMT_CUDA(cudaMemset(ctx->counters, 0, sizeof(int64_t) * 16));
  return GMT_OK;
}

extern "C" int gmt_host_alloc(size_t bytes, void** out) {
  GMT_CUDA(cudaHostAlloc(out, bytes, cudaHostAllocDefault));
  return GMT_OK;
}

extern "C" void gmt_host_free(void* p) {
  if (p) cudaFreeHost(p);
}

// ---- radius (host scalar; graph.cpp:14-32 with the same libm calls) --------
extern "C" int gmt_unit_ball_volume(int32_t d, double* out) {
  if (d < 1) return set_error(GMT_E_INVALID_INPUT, "dimension must be >= 1");
  *out = std::pow(M_PI, 0.5 * d) / std::tgamma(0.5 * d + 1.0);
  return GMT_OK;
}

extern "C" int gmt_connection_radius(int32_t dim, int64_t n_, double eta, double mu,
                                     double* out) {
  if (dim < 1) return set_error(GMT_E_INVALID_INPUT, "dimension must be >= 1");
  if (n_ < 2) return set_error(GMT_E_INVALID_INPUT, "connection radius needs n >= 2");
  if (!(eta >= 0.0)) return set_error(GMT_E_INVALID_INPUT, "eta must be >= 0");
  if (!(mu > 0.0 && mu <= 1.0)) return set_error(GMT_E_INVALID_INPUT, "mu_free must be in (0, 1]");
  double zeta;
  gmt_unit_ball_volume(dim, &zeta);
  const double d = static_cast<double>(dim), n = static_cast<double>(n_);
  const double inv_d = 1.0 / d;
  *out = 4.0 * std::pow(1.0 + eta, inv_d) * std::pow(inv_d, inv_d) * std::pow(mu / zeta, inv_d) *
         std::pow(std::log(n) / n, inv_d);
  return GMT_OK;
}

// ---- instances ----------------------------------------------------------------
namespace gmtb {

int validate_scene(const gmt_scene* s) {  // validate_obstacles / validate_box (space.cpp:18-38)
  if (!s) return set_error(GMT_E_INVALID_INPUT, "scene is null");
  if (s->dim < 1) return set_error(GMT_E_INVALID_INPUT, "obstacle set dimension must be >= 1");
  if (s->num_boxes < 0) return set_error(GMT_E_INVALID_INPUT, "negative box count");
  for (int b = 0; b < s->num_boxes; ++b)
    for (int k = 0; k < s->dim; ++k)
      if (!(s->box_lo[b * s->dim + k] <= s->box_hi[b * s->dim + k]))
        return set_error(GMT_E_INVALID_INPUT, "box has lo > hi on axis " + std::to_string(k));
  for (int k = 0; k < s->dim; ++k)
    if (!(s->goal_lo[k] <= s->goal_hi[k]))
      return set_error(GMT_E_INVALID_INPUT, "box has lo > hi on axis " + std::to_string(k));
  return GMT_OK;
}

// Lay an instance out in `arena` and copy the host arrays in (async on the
// ctx stream).  Fills `desc` with device pointers.
int fill_instance(gmt_ctx* ctx, Arena& arena, DevInstance& desc, const gmt_scene* scene,
                  const double* coords, int32_t n, int32_t goal_count, const gmt_graph_view* g) {
  GMT_TRY(validate_scene(scene));
  if (n < 1) return set_error(GMT_E_INVALID_INPUT, "instance needs at least one sample");
  if (!g) return set_error(GMT_E_INVALID_INPUT, "graph is null");
  const int d = scene->dim, nb = scene->num_boxes;
  const int gn = g->n;
  if (gn < 0) return set_error(GMT_E_INVALID_INPUT, "graph node count is negative");
  const int64_t E = g->out_ptr[gn];
  const bool directed = g->directed != 0;
  const int64_t Ein = directed ? g->in_ptr[gn] : E;
  const bool paths = g->num_paths > 0;
  const int64_t npts = paths ? g->path_ptr[g->num_paths] : 0;
  if (paths && g->dim != d) return set_error(GMT_E_INVALID_INPUT, "path points differ in dimension");

  Carver c;
  const size_t o_coords = c.take<double>(static_cast<size_t>(n) * d);
  const size_t o_lo = c.take<double>(static_cast<size_t>(nb) * d);
  const size_t o_hi = c.take<double>(static_cast<size_t>(nb) * d);
  const size_t o_glo = c.take<double>(d);
  const size_t o_ghi = c.take<double>(d);
  const size_t o_optr = c.take<int64_t>(gn + 1);
  const size_t o_ocol = c.take<int32_t>(E);
  const size_t o_ocost = c.take<double>(E);
  size_t o_iptr = 0, o_icol = 0, o_icost = 0;
  if (directed) {
    o_iptr = c.take<int64_t>(gn + 1);
    o_icol = c.take<int32_t>(Ein);
    o_icost = c.take<double>(Ein);
  }
  const bool has_in_path = paths && (directed ? g->in_path != nullptr : g->out_path != nullptr);
  const size_t o_ipath = has_in_path ? c.take<int32_t>(Ein) : 0;
  const bool has_out_path = paths && directed && g->out_path != nullptr;
  const size_t o_opath = has_out_path ? c.take<int32_t>(E) : 0;
  const size_t o_pptr = paths ? c.take<int64_t>(g->num_paths + 1) : 0;
  const size_t o_ppts = paths ? c.take<double>(static_cast<size_t>(npts) * d) : 0;
  GMT_TRY(arena.reserve(c.off));

  void* base = arena.ptr;
  cudaStream_t s = ctx->stream;
  auto put = [&](size_t off, const void* src, size_t bytes) -> int {
    if (bytes == 0) return GMT_OK;
    GMT_CUDA(cudaMemcpyAsync(at<char>(base, off), src, bytes, cudaMemcpyHostToDevice, s));
    return GMT_OK;
  };
  GMT_TRY(put(o_coords, coords, sizeof(double) * n * d));
  GMT_TRY(put(o_lo, scene->box_lo, sizeof(double) * nb * d));
  GMT_TRY(put(o_hi, scene->box_hi, sizeof(double) * nb * d));
  GMT_TRY(put(o_glo, scene->goal_lo, sizeof(double) * d));
  GMT_TRY(put(o_ghi, scene->goal_hi, sizeof(double) * d));
  GMT_TRY(put(o_optr, g->out_ptr, sizeof(int64_t) * (gn + 1)));
  GMT_TRY(put(o_ocol, g->out_col, sizeof(int32_t) * E));
  GMT_TRY(put(o_ocost, g->out_cost, sizeof(double) * E));
  if (directed) {
    GMT_TRY(put(o_iptr, g->in_ptr, sizeof(int64_t) * (gn + 1)));
    GMT_TRY(put(o_icol, g->in_col, sizeof(int32_t) * Ein));
    GMT_TRY(put(o_icost, g->in_cost, sizeof(double) * Ein));
  }
  if (has_in_path) GMT_TRY(put(o_ipath, directed ? g->in_path : g->out_path, sizeof(int32_t) * Ein));
  if (has_out_path) GMT_TRY(put(o_opath, g->out_path, sizeof(int32_t) * E));
  if (paths) {
    GMT_TRY(put(o_pptr, g->path_ptr, sizeof(int64_t) * (g->num_paths + 1)));
    GMT_TRY(put(o_ppts, g->path_pts, sizeof(double) * npts * d));
  }

  desc = DevInstance{};
  desc.n = n;
  desc.dim = d;
  desc.num_boxes = nb;
  desc.directed = directed ? 1 : 0;
  desc.goal_count = goal_count;
  desc.init_index = -1;
  desc.radius = g->radius;
  desc.num_edges = E;
  desc.coords = at<double>(base, o_coords);
  desc.box_lo = at<double>(base, o_lo);
  desc.box_hi = at<double>(base, o_hi);
  desc.goal_lo = at<double>(base, o_glo);
  desc.goal_hi = at<double>(base, o_ghi);
  desc.out_ptr = at<int64_t>(base, o_optr);
  desc.out_col = at<int32_t>(base, o_ocol);
  desc.out_cost = at<double>(base, o_ocost);
  desc.in_ptr = directed ? at<int64_t>(base, o_iptr) : desc.out_ptr;
  desc.in_col = directed ? at<int32_t>(base, o_icol) : desc.out_col;
  desc.in_cost = directed ? at<double>(base, o_icost) : desc.out_cost;
  desc.in_path = has_in_path ? at<int32_t>(base, o_ipath) : nullptr;
  desc.out_path = has_out_path ? at<int32_t>(base, o_opath) : (directed ? nullptr : desc.in_path);
  desc.path_ptr = paths ? at<int64_t>(base, o_pptr) : nullptr;
  desc.path_pts = paths ? at<double>(base, o_ppts) : nullptr;
  return GMT_OK;
}

int push_desc(gmt_ctx* ctx, gmt_instance* inst) {
  GMT_TRY(inst->desc_mem.reserve(sizeof(DevInstance)));
  GMT_CUDA(cudaMemcpyAsync(inst->desc_mem.ptr, &inst->desc, sizeof(DevInstance),
                           cudaMemcpyHostToDevice, ctx->stream));
  return GMT_OK;
}

}  // namespace gmtb

extern "C" int gmt_instance_upload(gmt_ctx* ctx, const gmt_scene* scene, const double* coords,
                                   int32_t n, int32_t goal_count, const gmt_graph_view* graph,
                                   gmt_instance** out) {
  gmtb::AllocScope alloc_scope_(ctx);
  *out = nullptr;
  auto* inst = new gmt_instance;
  int rc = fill_instance(ctx, inst->mem, inst->desc, scene, coords, n, goal_count, graph);
  if (rc == GMT_OK) rc = push_desc(ctx, inst);
  if (rc == GMT_OK) {
    cudaError_t e = cudaStreamSynchronize(ctx->stream);
    if (e != cudaSuccess) rc = cuda_error(e, "upload");
  }
  if (rc != GMT_OK) {
    delete inst;
    return rc;
  }
  inst->graph_n = graph->n;
  *out = inst;
  return GMT_OK;
}

extern "C" int gmt_instance_info(const gmt_instance* inst, int32_t* n, int32_t* dim,
                                 int32_t* init_index, double* radius, int64_t* num_edges,
                                 int32_t* goal_count) {
  if (!inst) return set_error(GMT_E_INVALID_INPUT, "instance is null");
  if (n) *n = inst->desc.n;
  if (dim) *dim = inst->desc.dim;
  if (init_index) *init_index = inst->desc.init_index;
  if (radius) *radius = inst->desc.radius;
  if (num_edges) *num_edges = inst->desc.num_edges;
  if (goal_count) *goal_count = inst->desc.goal_count;
  return GMT_OK;
}

extern "C" int gmt_instance_download(gmt_ctx* ctx, const gmt_instance* inst, double* coords,
                                     int32_t* goal_idx, int64_t* out_ptr, int32_t* out_col,
                                     double* out_cost) {
  gmtb::AllocScope alloc_scope_(ctx);
  const DevInstance& D = inst->desc;
  cudaStream_t s = ctx->stream;
  if (coords)
    GMT_CUDA(cudaMemcpyAsync(coords, D.coords, sizeof(double) * D.n * D.dim, cudaMemcpyDeviceToHost, s));
  if (out_ptr)
    GMT_CUDA(cudaMemcpyAsync(out_ptr, D.out_ptr, sizeof(int64_t) * (inst->graph_n + 1),
                             cudaMemcpyDeviceToHost, s));
  if (out_col)
    GMT_CUDA(cudaMemcpyAsync(out_col, D.out_col, sizeof(int32_t) * D.num_edges, cudaMemcpyDeviceToHost, s));
  if (out_cost)
    GMT_CUDA(cudaMemcpyAsync(out_cost, D.out_cost, sizeof(double) * D.num_edges, cudaMemcpyDeviceToHost, s));
  if (goal_idx && D.goal_count > 0) {
    if (!inst->goal_idx_dev)
      return set_error(GMT_E_INVALID_INPUT, "goal indices are only kept for device-built instances");
    GMT_CUDA(cudaMemcpyAsync(goal_idx, inst->goal_idx_dev, sizeof(int32_t) * D.goal_count,
                             cudaMemcpyDeviceToHost, s));
  }
  GMT_CUDA(cudaStreamSynchronize(s));
  return GMT_OK;
}

extern "C" void gmt_instance_destroy(gmt_instance* inst) { delete inst; }

// ---- exact geometry on the device -------------------------------------------------
extern "C" int gmt_segment_free(gmt_ctx* ctx, int32_t dim, int32_t num_boxes, const double* box_lo,
                                const double* box_hi, const double* a, const double* b, int64_t count,
                                uint8_t* free_out) {
  gmtb::AllocScope alloc_scope_(ctx);
  if (!ctx) return set_error(GMT_E_INVALID_INPUT, "context is null");
  // validate_obstacles / validate_box (space.cpp:18-38) and the dimension
  // checks of segment_free (space.cpp:81-83).
  if (dim < 1) return set_error(GMT_E_INVALID_INPUT, "obstacle set dimension must be >= 1");
  if (dim > kMaxSolveDim) return set_error(GMT_E_INVALID_INPUT, "dimension above 16 is not supported");
  if (num_boxes < 0 || count < 0) return set_error(GMT_E_INVALID_INPUT, "negative count");
  for (int64_t i = 0; i < static_cast<int64_t>(num_boxes) * dim; ++i)
    if (!(box_lo[i] <= box_hi[i]))
      return set_error(GMT_E_INVALID_INPUT, "box has lo > hi on axis " + std::to_string(i % dim));
  if (count == 0) return GMT_OK;
  const size_t nbx = static_cast<size_t>(num_boxes) * dim, nseg = static_cast<size_t>(count) * dim;
  Carver c;
  const size_t o_lo = c.take<double>(nbx), o_hi = c.take<double>(nbx);
  const size_t o_a = c.take<double>(nseg), o_b = c.take<double>(nseg);
  const size_t o_out = c.take<uint8_t>(count);
  Arena buf;
  GMT_TRY(buf.reserve(c.off));
  cudaStream_t s = ctx->stream;
  void* base = buf.ptr;
  int rc = GMT_OK;
  auto cu = [&](cudaError_t e, const char* what) {
    if (rc == GMT_OK && e != cudaSuccess) rc = cuda_error(e, what);
  };
  if (nbx) {
    cu(cudaMemcpyAsync(at<double>(base, o_lo), box_lo, sizeof(double) * nbx, cudaMemcpyHostToDevice, s), "copy");
    cu(cudaMemcpyAsync(at<double>(base, o_hi), box_hi, sizeof(double) * nbx, cudaMemcpyHostToDevice, s), "copy");
  }
  cu(cudaMemcpyAsync(at<double>(base, o_a), a, sizeof(double) * nseg, cudaMemcpyHostToDevice, s), "copy");
  cu(cudaMemcpyAsync(at<double>(base, o_b), b, sizeof(double) * nseg, cudaMemcpyHostToDevice, s), "copy");
  if (rc == GMT_OK) {
    cu(launch_segment_free(at<double>(base, o_a), at<double>(base, o_b), count, dim, at<double>(base, o_lo),
                           at<double>(base, o_hi), num_boxes, at<uint8_t>(base, o_out), ctx->sm_count, s),
       "segment_free launch");
    ++ctx->launches;
  }
  cu(cudaMemcpyAsync(free_out, at<uint8_t>(base, o_out), count, cudaMemcpyDeviceToHost, s), "copy");
  cu(cudaStreamSynchronize(s), "segment_free");
  buf.release();
  return rc;
}

// ---- single-query solve ---------------------------------------------------------
namespace gmtb {

int validate_plan(const gmt_instance* inst, int32_t init_index, double lambda, double radius) {
  // validate_plan_inputs (planner.cpp:17-23) and planner.cpp:98-103.
  if (!inst) return set_error(GMT_E_INVALID_INPUT, "instance is null");
  if (inst->graph_n != inst->desc.n)
    return set_error(GMT_E_INVALID_INPUT, "graph was built over a different sample count");
  if (init_index < 0 || init_index >= inst->desc.n)
    return set_error(GMT_E_INVALID_INPUT, "init_index " + std::to_string(init_index) + " out of range");
  if (!(lambda > 0.0 && lambda <= 1.0)) return set_error(GMT_E_INVALID_INPUT, "lambda must be in (0, 1]");
  if (radius != inst->desc.radius)
    return set_error(GMT_E_INVALID_INPUT, "params.radius differs from the graph's connection radius");
  return GMT_OK;
}

// Shared-memory plan for a set of queries; errors when a query's wavefront
// cannot live on chip.
// gstate (may be null): when the state exceeds the opt-in, *gstate receives
// the per-query bytes of a global-memory wavefront (one wide CTA per query,
// launch_solve's gstate mode) instead of an error; 0 when it fits on chip.
int plan_smem(gmt_ctx* ctx, int max_n, int max_d, int max_nb, int cluster, size_t* smem,
              int* obs_in_smem, size_t* gstate = nullptr) {
  if (gstate) *gstate = 0;
  if (max_d > kMaxSolveDim)
    return set_error(GMT_E_INVALID_INPUT, "dimension above 16 is not supported");
  if (max_n > kMaxSolveNodes) {
    if (!gstate)
      return set_error(GMT_E_INVALID_INPUT, "n = " + std::to_string(max_n) + " exceeds the " +
                                                std::to_string(kMaxSolveNodes) +
                                                "-node limit of the on-chip wavefront");
    *obs_in_smem = 1;  // global-memory wavefront with 32-bit work lists
    *gstate = solve_layout(max_n, max_d, max_nb, true, false, 4).total;
    *smem = 0;
    return GMT_OK;
  }
  const bool parent_smem = cluster > 1;
  const size_t obs_bytes = sizeof(double) * 4 * static_cast<size_t>(max_nb) * max_d;
  *obs_in_smem = obs_bytes <= 48 * 1024 ? 1 : 0;
  SolveLayout L = solve_layout(max_n, max_d, max_nb, *obs_in_smem != 0, parent_smem);
  if (L.total > ctx->smem_optin && *obs_in_smem) {
    *obs_in_smem = 0;
    L = solve_layout(max_n, max_d, max_nb, false, parent_smem);
  }
  if (L.total > ctx->smem_optin && gstate) {
    *obs_in_smem = 1;  // (the boxes are staged into the global buffer)
    L = solve_layout(max_n, max_d, max_nb, true, false, 4);
    *gstate = L.total;
    *smem = 0;
    return GMT_OK;
  }
  if (L.total > ctx->smem_optin) {
    return set_error(GMT_E_INVALID_INPUT,
                     "n = " + std::to_string(max_n) + " needs " + std::to_string(L.total) +
                         " bytes of on-chip wavefront state; the limit is " +
                         std::to_string(ctx->smem_optin));
  }
  *smem = L.total;
  return GMT_OK;
}

// Result buffers for `count` queries of up to `n` nodes each.
int carve_results(Arena& arena, int count, const int64_t* node_off, bool tree, bool stats,
                  std::vector<DevResult>& out, ResultScalars** scalars_base, int64_t* counters) {
  const int64_t total = node_off[count];
  Carver c;
  const size_t o_sc = c.take<ResultScalars>(count);
  const size_t o_path = c.take<int32_t>(total);
  size_t o_label = 0, o_cost = 0, o_iter = 0, o_gs = 0, o_na = 0, o_ck = 0;
  const size_t o_parent = c.take<int32_t>(total);  // always: batched solves walk it
  if (tree) {
    o_label = c.take<uint8_t>(total);
    o_cost = c.take<double>(total);
    o_iter = c.take<int64_t>(total);
  }
  if (stats) {
    o_gs = c.take<int32_t>(total + count);
    o_na = c.take<int32_t>(total + count);
    o_ck = c.take<int64_t>(total + count);
  }
  GMT_TRY(arena.reserve(c.off));
  void* b = arena.ptr;
  out.resize(count);
  for (int q = 0; q < count; ++q) {
    const int64_t o = node_off[q];
    DevResult& r = out[q];
    r.scalars = at<ResultScalars>(b, o_sc) + q;
    r.path = at<int32_t>(b, o_path) + o;
    r.label = tree ? at<uint8_t>(b, o_label) + o : nullptr;
    r.tree_cost = tree ? at<double>(b, o_cost) + o : nullptr;
    r.parent = at<int32_t>(b, o_parent) + o;
    r.iter_added = tree ? at<int64_t>(b, o_iter) + o : nullptr;
    r.group_sizes = stats ? at<int32_t>(b, o_gs) + o + q : nullptr;
    r.nodes_added = stats ? at<int32_t>(b, o_na) + o + q : nullptr;
    r.checks = stats ? at<int64_t>(b, o_ck) + o + q : nullptr;
    r.counters = counters;
  }
  *scalars_base = at<ResultScalars>(b, o_sc);
  return GMT_OK;
}

// One global wavefront buffer per job (stride aligned to 256 bytes).
int assign_gstate(Arena& arena, std::vector<SolveJob>& jobs, size_t bytes) {
  const size_t stride = (bytes + 255) & ~static_cast<size_t>(255);
  GMT_TRY(arena.reserve(stride * jobs.size()));
  for (size_t q = 0; q < jobs.size(); ++q) jobs[q].gstate = static_cast<unsigned char*>(arena.ptr) + q * stride;
  return GMT_OK;
}

int launch_jobs(gmt_ctx* ctx, const std::vector<SolveJob>& jobs, int cluster, int threads,
                size_t smem, int obs_in_smem, int dim) {
  const size_t bytes = sizeof(SolveJob) * jobs.size();
  GMT_TRY(ctx->jobs.reserve(bytes));
  GMT_TRY(ctx->pinned_jobs.reserve(bytes));
  std::memcpy(ctx->pinned_jobs.ptr, jobs.data(), bytes);
  GMT_CUDA(cudaMemcpyAsync(ctx->jobs.ptr, ctx->pinned_jobs.ptr, bytes, cudaMemcpyHostToDevice,
                           ctx->stream));
  const bool gs = jobs[0].gstate != nullptr;
  const cudaError_t e = launch_solve(static_cast<const SolveJob*>(ctx->jobs.ptr), static_cast<int>(jobs.size()),
                                     gs ? 1 : cluster, gs ? 512 : threads, smem, obs_in_smem, dim, ctx->stream,
                                     !gs && jobs[0].res.counters != nullptr, gs);
  if (e != cudaSuccess) {
    return set_error(GMT_E_CUDA, std::string("solve launch (cluster ") + std::to_string(cluster) + ", " +
                                     std::to_string(threads) + " threads, " + std::to_string(smem) +
                                     " B smem, dim " + std::to_string(dim) + "): " + cudaGetErrorString(e));
  }
  ++ctx->launches;
  return GMT_OK;
}

int download_result(gmt_ctx* ctx, const DevResult& r, int n, gmt_plan_out* out) {
  cudaStream_t s = ctx->stream;
  ResultScalars sc;
  GMT_CUDA(cudaMemcpyAsync(&sc, r.scalars, sizeof(sc), cudaMemcpyDeviceToHost, s));
  if (out->label && r.label) GMT_CUDA(cudaMemcpyAsync(out->label, r.label, n, cudaMemcpyDeviceToHost, s));
  if (out->tree_cost && r.tree_cost)
    GMT_CUDA(cudaMemcpyAsync(out->tree_cost, r.tree_cost, sizeof(double) * n, cudaMemcpyDeviceToHost, s));
  if (out->parent && r.parent)
    GMT_CUDA(cudaMemcpyAsync(out->parent, r.parent, sizeof(int32_t) * n, cudaMemcpyDeviceToHost, s));
  if (out->iteration_added && r.iter_added)
    GMT_CUDA(cudaMemcpyAsync(out->iteration_added, r.iter_added, sizeof(int64_t) * n,
                             cudaMemcpyDeviceToHost, s));
  GMT_CUDA(cudaStreamSynchronize(s));
  out->status = sc.status;
  out->goal_node = sc.goal_node;
  out->cost = sc.cost;
  out->iterations = sc.iterations;
  out->total_collision_checks = sc.total_checks;
  out->path_len = sc.path_len;
  out->num_stats = sc.num_stats;
  out->tree_size = sc.tree_size;
  if (out->path && sc.path_len > 0)
    GMT_CUDA(cudaMemcpyAsync(out->path, r.path, sizeof(int32_t) * sc.path_len, cudaMemcpyDeviceToHost, s));
  const int ns = std::min(sc.num_stats, out->stats_cap);
  if (ns > 0 && r.group_sizes) {
    if (out->group_sizes)
      GMT_CUDA(cudaMemcpyAsync(out->group_sizes, r.group_sizes, sizeof(int32_t) * ns, cudaMemcpyDeviceToHost, s));
    if (out->nodes_added)
      GMT_CUDA(cudaMemcpyAsync(out->nodes_added, r.nodes_added, sizeof(int32_t) * ns, cudaMemcpyDeviceToHost, s));
    if (out->collision_checks)
      GMT_CUDA(cudaMemcpyAsync(out->collision_checks, r.checks, sizeof(int64_t) * ns, cudaMemcpyDeviceToHost, s));
  }
  GMT_CUDA(cudaStreamSynchronize(s));
  return GMT_OK;
}

int plan_on(gmt_ctx* ctx, const gmt_instance* inst, int32_t init_index, double lambda,
            double radius, gmt_plan_out* out, int mode = kModeGmt) {
  GMT_TRY(validate_plan(inst, init_index, lambda, radius));
  const DevInstance& D = inst->desc;
  size_t smem, gs = 0;
  int obs;
  GMT_TRY(plan_smem(ctx, D.n, D.dim, D.num_boxes, ctx->cluster ? ctx->cluster : 8, &smem, &obs, &gs));
  int64_t node_off[2] = {0, D.n};
  std::vector<DevResult> res;
  ResultScalars* sc;
  GMT_TRY(carve_results(ctx->res, 1, node_off, true, true, res, &sc,
                        ctx->counting ? ctx->counters : nullptr));
  SolveJob job{};
  job.inst = static_cast<const DevInstance*>(inst->desc_mem.ptr);
  job.res = res[0];
  job.init_index = init_index;
  job.mode = mode;
  job.lambda = lambda;
  job.radius = radius;
  const int cluster = ctx->cluster ? ctx->cluster : 8;
  int threads = ctx->threads ? ctx->threads : 512;
  std::vector<SolveJob> jobs{job};
  if (gs) GMT_TRY(assign_gstate(ctx->gstate, jobs, gs));  // (too large for shared memory)
  GMT_TRY(launch_jobs(ctx, jobs, cluster, threads, smem, obs, D.dim));
  return download_result(ctx, res[0], D.n, out);
}

}  // namespace gmtb

extern "C" int gmt_plan(gmt_ctx* ctx, const gmt_instance* inst, int32_t init_index, double lambda,
                        double radius, gmt_plan_out* out) {
  gmtb::AllocScope alloc_scope_(ctx);
  return plan_on(ctx, inst, init_index, lambda, radius, out);
}

extern "C" int gmt_fmt_plan(gmt_ctx* ctx, const gmt_instance* inst, int32_t init_index,
                            gmt_plan_out* out) {
  gmtb::AllocScope alloc_scope_(ctx);
  if (!inst) return set_error(GMT_E_INVALID_INPUT, "instance is null");
  return plan_on(ctx, inst, init_index, 1.0, inst->desc.radius, out, kModeFmt);
}

extern "C" int gmt_dijkstra_oracle(gmt_ctx* ctx, const gmt_instance* inst, int32_t init_index,
                                   gmt_plan_out* out) {
  gmtb::AllocScope alloc_scope_(ctx);
  // validate_plan_inputs (planner.cpp:17-23), then eager checks + Dijkstra.
  if (!inst) return set_error(GMT_E_INVALID_INPUT, "instance is null");
  if (inst->graph_n != inst->desc.n)
    return set_error(GMT_E_INVALID_INPUT, "graph was built over a different sample count");
  if (init_index < 0 || init_index >= inst->desc.n)
    return set_error(GMT_E_INVALID_INPUT, "init_index " + std::to_string(init_index) + " out of range");
  const DevInstance& D = inst->desc;
  if (D.dim > kMaxSolveDim) return set_error(GMT_E_INVALID_INPUT, "dimension above 16 is not supported");
  int64_t node_off[2] = {0, D.n};
  std::vector<DevResult> res;
  ResultScalars* sc;
  GMT_TRY(carve_results(ctx->res, 1, node_off, true, false, res, &sc, nullptr));
  SolveJob job{};
  job.inst = static_cast<const DevInstance*>(inst->desc_mem.ptr);
  job.res = res[0];
  job.init_index = init_index;
  job.mode = kModeGmt;
  job.lambda = 1.0;
  job.radius = D.radius;
  GMT_TRY(ctx->jobs.reserve(sizeof(SolveJob)));
  GMT_TRY(ctx->pinned_jobs.reserve(sizeof(SolveJob)));
  std::memcpy(ctx->pinned_jobs.ptr, &job, sizeof(SolveJob));
  cudaStream_t s = ctx->stream;
  GMT_CUDA(cudaMemcpyAsync(ctx->jobs.ptr, ctx->pinned_jobs.ptr, sizeof(SolveJob), cudaMemcpyHostToDevice, s));
  Arena buf;
  GMT_TRY(buf.reserve(16 + static_cast<size_t>(D.num_edges)));
  auto* checks = static_cast<unsigned long long*>(buf.ptr);
  auto* ok = static_cast<uint8_t*>(buf.ptr) + 16;
  GMT_CUDA(cudaMemsetAsync(checks, 0, sizeof(unsigned long long), s));
  GMT_CUDA(launch_dijkstra(job.inst, static_cast<const SolveJob*>(ctx->jobs.ptr), D.n, D.dim, ok, checks,
                           ctx->sm_count, s));
  ctx->launches += 2;
  const int rc = download_result(ctx, res[0], D.n, out);
  buf.release();
  return rc;
}

extern "C" int gmt_plan_host(gmt_ctx* ctx, const gmt_scene* scene, const double* coords, int32_t n,
                             int32_t goal_count, const gmt_graph_view* graph, int32_t init_index,
                             double lambda, double radius, gmt_plan_out* out) {
  gmtb::AllocScope alloc_scope_(ctx);
  // planner.cpp:17-23 checks come first, before anything is uploaded.
  if (!graph) return set_error(GMT_E_INVALID_INPUT, "graph is null");
  if (graph->n != n) return set_error(GMT_E_INVALID_INPUT, "graph was built over a different sample count");
  if (init_index < 0 || init_index >= n)
    return set_error(GMT_E_INVALID_INPUT, "init_index " + std::to_string(init_index) + " out of range");
  if (!(lambda > 0.0 && lambda <= 1.0)) return set_error(GMT_E_INVALID_INPUT, "lambda must be in (0, 1]");
  if (radius != graph->radius)
    return set_error(GMT_E_INVALID_INPUT, "params.radius differs from the graph's connection radius");
  gmt_instance& inst = ctx->plan_inst;
  GMT_TRY(fill_instance(ctx, inst.mem, inst.desc, scene, coords, n, goal_count, graph));
  inst.graph_n = graph->n;
  GMT_TRY(push_desc(ctx, &inst));
  return plan_on(ctx, &inst, init_index, lambda, radius, out);
}

// ---- batches (struct gmt_batch: internal.cuh) -------------------------------------------
// The common dimension of a batch's instances (0: mixed).
static int b_dim_of(gmt_instance* const* insts, int count) {
  int d = insts[0]->desc.dim;
  for (int q = 1; q < count; ++q)
    if (insts[q]->desc.dim != d) return 0;
  return d;
}

extern "C" int gmt_batch_create(gmt_ctx* ctx, int32_t count, gmt_instance* const* insts,
                                const int32_t* init_index, double lambda, gmt_batch** out) {
  gmtb::AllocScope alloc_scope_(ctx);
  *out = nullptr;
  if (count < 1) return set_error(GMT_E_INVALID_INPUT, "batch needs at least one query");
  auto* b = new gmt_batch;
  b->ctx = ctx;
  b->node_off.assign(count + 1, 0);
  int max_n = 0, max_d = 0, max_nb = 0;
  for (int q = 0; q < count; ++q) {
    const gmt_instance* inst = insts[q];
    const int ii = init_index ? init_index[q] : (inst ? inst->desc.init_index : -1);
    int rc = validate_plan(inst, ii, lambda, inst ? inst->desc.radius : 0.0);
    if (rc != GMT_OK) {
      delete b;
      return set_error(rc, "query " + std::to_string(q) + ": " + g_last_error);
    }
    b->node_off[q + 1] = b->node_off[q] + inst->desc.n;
    max_n = std::max(max_n, inst->desc.n);
    max_d = std::max(max_d, inst->desc.dim);
    max_nb = std::max(max_nb, inst->desc.num_boxes);
  }
  b->dim = insts[0]->desc.dim;
  for (int q = 1; q < count; ++q)
    if (insts[q]->desc.dim != b->dim) b->dim = 0;
  // Auto shape (batch cluster 0): a few kinodynamic queries (eight polyline
  // segments per lazy check) run on 2-CTA clusters of wide CTAs; Euclidean
  // queries, and kinodynamic batches that fill the SMs several times over,
  // on single narrow CTAs (4096 DI queries: 47 ms vs 52 ms on wide CTAs and
  // 66 ms on 2-CTA clusters, tools/di_sweep.py).
  b->cluster = ctx->batch_cluster;
  bool kino = false;
  for (int q = 0; q < count; ++q) kino = kino || insts[q]->desc.steering != GMT_STEER_EUCLIDEAN;
  const bool di6 = kino && b_dim_of(insts, count) == 6;
  if (b->cluster == 0) b->cluster = di6 ? 1 : (kino && count < 4 * ctx->sm_count ? 2 : 1);
  size_t gs = 0;
  int rc = plan_smem(ctx, max_n, max_d, max_nb, b->cluster, &b->smem, &b->obs, &gs);
  if (rc == GMT_OK && gs) b->cluster = 1;
  if (rc == GMT_OK)
    rc = carve_results(b->res, count, b->node_off.data(), true, true, b->results, &b->scalars,
                       ctx->counting ? ctx->counters : nullptr);
  if (rc != GMT_OK) {
    delete b;
    return rc;
  }
  b->jobs.resize(count);
  for (int q = 0; q < count; ++q) {
    SolveJob& j = b->jobs[q];
    j = SolveJob{};
    j.inst = static_cast<const DevInstance*>(insts[q]->desc_mem.ptr);
    j.res = b->results[q];
    j.init_index = init_index ? init_index[q] : insts[q]->desc.init_index;
    j.lambda = lambda;
    j.radius = insts[q]->desc.radius;
  }
  b->threads = ctx->batch_threads ? ctx->batch_threads : (b->cluster > 1 ? 512 : (di6 ? 768 : 256));
  if (b->threads == 768 && (b->cluster != 1 || !di6)) b->threads = b->cluster > 1 ? 512 : 256;
  if (!gs && solve_dyn_scratch(b->threads, b->dim)) {  // (the 24-warp shape's scratch)
    const size_t total = align16(b->smem) + solve_dyn_scratch(b->threads, b->dim);
    if (total <= ctx->smem_optin) {
      b->smem = total;
    } else {
      b->threads = 256;
    }
  }
  if (gs) {
    b->threads = 512;
    rc = assign_gstate(b->gstate_mem, b->jobs, gs);
    if (rc != GMT_OK) {
      delete b;
      return rc;
    }
  }
  rc = b->jobs_mem.reserve(sizeof(SolveJob) * count);
  if (rc == GMT_OK) {
    // jobs_mem comes from the stream-ordered pool of ctx->stream: write it on
    // that stream (a block freed there earlier may still be read by work in
    // flight on it) and wait, since b->jobs is pageable.
    cudaError_t e = cudaMemcpyAsync(b->jobs_mem.ptr, b->jobs.data(), sizeof(SolveJob) * count,
                                    cudaMemcpyHostToDevice, ctx->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(ctx->stream);
    if (e != cudaSuccess) rc = cuda_error(e, "batch jobs");
  }
  if (rc != GMT_OK) {
    delete b;
    return rc;
  }
  *out = b;
  return GMT_OK;
}

extern "C" int gmt_batch_launch(gmt_ctx* ctx, gmt_batch* b) {
  gmtb::AllocScope alloc_scope_(ctx);
  const bool gs = b->jobs[0].gstate != nullptr;
  GMT_CUDA(launch_solve(static_cast<const SolveJob*>(b->jobs_mem.ptr), static_cast<int>(b->jobs.size()),
                        b->cluster, b->threads, b->smem, b->obs, b->dim, ctx->stream,
                        !gs && b->jobs[0].res.counters != nullptr, gs, b->pool && !gs));
  ++ctx->launches;
  return GMT_OK;
}

static void to_summary(const ResultScalars& s, gmt_plan_summary* o) {
  o->status = s.status;
  o->goal_node = s.goal_node;
  o->cost = s.cost;
  o->iterations = s.iterations;
  o->total_collision_checks = s.total_checks;
  o->path_len = s.path_len;
  o->num_stats = s.num_stats;
}

extern "C" int gmt_batch_summaries(gmt_ctx* ctx, gmt_batch* b, gmt_plan_summary* out) {
  gmtb::AllocScope alloc_scope_(ctx);
  const size_t count = b->jobs.size();
  std::vector<ResultScalars> sc(count);
  GMT_CUDA(cudaMemcpyAsync(sc.data(), b->scalars, sizeof(ResultScalars) * count,
                           cudaMemcpyDeviceToHost, ctx->stream));
  GMT_CUDA(cudaStreamSynchronize(ctx->stream));
  for (size_t q = 0; q < count; ++q) to_summary(sc[q], &out[q]);
  // Adaptive launch order: a batch that spans several waves of CTAs ends with
  // a partial wave, shortest when the longest queries start first.  After the
  // first results are known, later launches dispatch the queries by their
  // collision checks, largest first (results are per query and unaffected;
  // 4096 DI queries: 37.8 -> 36.2 ms).
  if (!b->lpt_done && count >= static_cast<size_t>(2 * ctx->sm_count)) {
    std::vector<size_t> order(count);
    for (size_t q = 0; q < count; ++q) order[q] = q;
    std::stable_sort(order.begin(), order.end(),
                     [&](size_t a, size_t c) { return sc[a].total_checks > sc[c].total_checks; });
    std::vector<SolveJob> lpt(count);
    for (size_t k = 0; k < count; ++k) lpt[k] = b->jobs[order[k]];
    GMT_CUDA(cudaMemcpyAsync(b->jobs_mem.ptr, lpt.data(), sizeof(SolveJob) * count, cudaMemcpyHostToDevice,
                             ctx->stream));
    GMT_CUDA(cudaStreamSynchronize(ctx->stream));
    b->lpt_done = true;
  }
  return GMT_OK;
}

extern "C" int gmt_batch_result(gmt_ctx* ctx, gmt_batch* b, int32_t q, gmt_plan_out* out) {
  gmtb::AllocScope alloc_scope_(ctx);
  if (q < 0 || q >= static_cast<int32_t>(b->jobs.size()))
    return set_error(GMT_E_INVALID_INPUT, "query index out of range");
  const int n = static_cast<int>(b->node_off[q + 1] - b->node_off[q]);
  return download_result(ctx, b->results[q], n, out);
}

extern "C" void gmt_batch_destroy(gmt_batch* b) { delete b; }

// ---- packed host batch (the batched drop-in) ------------------------------------------
extern "C" int gmt_plan_batch_host(gmt_ctx* ctx, const gmt_batch_host* B, double lambda,
                                   gmt_plan_summary* summaries, int32_t* paths, uint8_t* label,
                                   double* tree_cost, int32_t* parent, int64_t* iteration_added) {
  gmtb::AllocScope alloc_scope_(ctx);
  const int count = B->count, d = B->dim;
  if (count < 1) return set_error(GMT_E_INVALID_INPUT, "batch needs at least one query");
  if (d < 1) return set_error(GMT_E_INVALID_INPUT, "dimension must be >= 1");
  if (!(lambda > 0.0 && lambda <= 1.0)) return set_error(GMT_E_INVALID_INPUT, "lambda must be in (0, 1]");
  const int64_t total_nodes = B->node_off[count];
  const int64_t total_edges = B->edge_off[count];
  const int64_t total_boxes = B->box_off[count];
  int max_n = 0, max_nb = 0;
  for (int q = 0; q < count; ++q) {
    const int n = static_cast<int>(B->node_off[q + 1] - B->node_off[q]);
    const int ii = B->init_index[q];
    if (n < 1) return set_error(GMT_E_INVALID_INPUT, "query " + std::to_string(q) + " has no samples");
    if (ii < 0 || ii >= n)
      return set_error(GMT_E_INVALID_INPUT, "query " + std::to_string(q) + ": init_index out of range");
    max_n = std::max(max_n, n);
    max_nb = std::max(max_nb, B->box_off[q + 1] - B->box_off[q]);
  }
  size_t smem;
  int obs;
  const int cluster = ctx->batch_cluster ? ctx->batch_cluster : 1;
  GMT_TRY(plan_smem(ctx, max_n, d, max_nb, cluster, &smem, &obs));

  // Device layout: every array of the batch back to back, one descriptor
  // per query; the host side only computes offsets.
  Carver c;
  const size_t o_coords = c.take<double>(total_nodes * d);
  const size_t o_lo = c.take<double>(total_boxes * d);
  const size_t o_hi = c.take<double>(total_boxes * d);
  const size_t o_glo = c.take<double>(static_cast<size_t>(count) * d);
  const size_t o_ghi = c.take<double>(static_cast<size_t>(count) * d);
  const size_t o_rp = c.take<int64_t>(total_nodes + count);
  const size_t o_col = c.take<int32_t>(total_edges);
  const size_t o_cost = c.take<double>(total_edges);
  const size_t o_desc = c.take<DevInstance>(count);
  GMT_TRY(ctx->scratch.reserve(c.off));
  // The (stream-ordered) scratch allocation happens on ctx->stream; the
  // copy stream may only write it after that point.
  GMT_CUDA(cudaEventRecord(ctx->copy_done[0], ctx->stream));
  GMT_CUDA(cudaStreamWaitEvent(ctx->copy_stream, ctx->copy_done[0], 0));
  void* base = ctx->scratch.ptr;
  cudaStream_t s = ctx->stream, cs = ctx->copy_stream;

  const bool tree = label || tree_cost || parent || iteration_added;
  std::vector<DevResult> res;
  ResultScalars* sc_dev;
  GMT_TRY(carve_results(ctx->res, count, B->node_off, tree, false, res, &sc_dev,
                        ctx->counting ? ctx->counters : nullptr));

  std::vector<DevInstance> descs(count);
  std::vector<SolveJob> jobs(count);
  DevInstance* d_desc = at<DevInstance>(base, o_desc);
  for (int q = 0; q < count; ++q) {
    DevInstance& D = descs[q];
    const int64_t no = B->node_off[q], eo = B->edge_off[q];
    const int32_t bo = B->box_off[q];
    D = DevInstance{};
    D.n = static_cast<int32_t>(B->node_off[q + 1] - no);
    D.dim = d;
    D.num_boxes = B->box_off[q + 1] - bo;
    D.directed = 0;
    D.goal_count = B->goal_count[q];
    D.init_index = B->init_index[q];
    D.radius = B->radius[q];
    D.num_edges = B->edge_off[q + 1] - eo;
    D.coords = at<double>(base, o_coords) + no * d;
    D.box_lo = at<double>(base, o_lo) + static_cast<int64_t>(bo) * d;
    D.box_hi = at<double>(base, o_hi) + static_cast<int64_t>(bo) * d;
    D.goal_lo = at<double>(base, o_glo) + static_cast<int64_t>(q) * d;
    D.goal_hi = at<double>(base, o_ghi) + static_cast<int64_t>(q) * d;
    D.out_ptr = at<int64_t>(base, o_rp) + no + q;
    D.out_col = at<int32_t>(base, o_col) + eo;
    D.out_cost = at<double>(base, o_cost) + eo;
    D.in_ptr = D.out_ptr;
    D.in_col = D.out_col;
    D.in_cost = D.out_cost;
    SolveJob& j = jobs[q];
    j = SolveJob{};
    j.inst = d_desc + q;
    j.res = res[q];
    j.init_index = D.init_index;
    j.lambda = lambda;
    j.radius = D.radius;
  }
  GMT_TRY(ctx->pinned.reserve(sizeof(DevInstance) * count));
  std::memcpy(ctx->pinned.ptr, descs.data(), sizeof(DevInstance) * count);
  GMT_CUDA(cudaMemcpyAsync(at<char>(base, o_desc), ctx->pinned.ptr, sizeof(DevInstance) * count,
                           cudaMemcpyHostToDevice, s));
  const size_t job_bytes = sizeof(SolveJob) * count;
  GMT_TRY(ctx->jobs.reserve(job_bytes));
  GMT_TRY(ctx->pinned_jobs.reserve(job_bytes));
  std::memcpy(ctx->pinned_jobs.ptr, jobs.data(), job_bytes);
  GMT_CUDA(cudaMemcpyAsync(ctx->jobs.ptr, ctx->pinned_jobs.ptr, job_bytes, cudaMemcpyHostToDevice, s));
  GMT_TRY(ctx->pinned2.reserve(sizeof(ResultScalars) * count));
  auto* sc_host = static_cast<ResultScalars*>(ctx->pinned2.ptr);
  const int threads = ctx->batch_threads ? ctx->batch_threads : (cluster > 1 ? 512 : 256);

  // Pipeline: the queries go in chunks; chunk k's host->device copies run
  // on the copy stream while chunk k-1 solves on the compute stream, and
  // each chunk's results come back right after its solve.
  const int nchunks = std::max(1, std::min(kMaxCopyChunks, count / 64));
  for (int ch = 0; ch < nchunks; ++ch) {
    const int q0 = static_cast<int>(static_cast<int64_t>(count) * ch / nchunks);
    const int q1 = static_cast<int>(static_cast<int64_t>(count) * (ch + 1) / nchunks);
    const int64_t n0 = B->node_off[q0], n1 = B->node_off[q1];
    const int64_t e0 = B->edge_off[q0], e1 = B->edge_off[q1];
    const int64_t b0 = B->box_off[q0], b1 = B->box_off[q1];
    auto put = [&](size_t off, size_t elem, int64_t first, int64_t last, const void* src) -> int {
      if (last <= first) return GMT_OK;
      GMT_CUDA(cudaMemcpyAsync(at<char>(base, off) + elem * first,
                               static_cast<const char*>(src) + elem * first, elem * (last - first),
                               cudaMemcpyHostToDevice, cs));
      return GMT_OK;
    };
    GMT_TRY(put(o_coords, sizeof(double), n0 * d, n1 * d, B->coords));
    GMT_TRY(put(o_lo, sizeof(double), b0 * d, b1 * d, B->box_lo));
    GMT_TRY(put(o_hi, sizeof(double), b0 * d, b1 * d, B->box_hi));
    GMT_TRY(put(o_glo, sizeof(double), static_cast<int64_t>(q0) * d, static_cast<int64_t>(q1) * d, B->goal_lo));
    GMT_TRY(put(o_ghi, sizeof(double), static_cast<int64_t>(q0) * d, static_cast<int64_t>(q1) * d, B->goal_hi));
    GMT_TRY(put(o_rp, sizeof(int64_t), n0 + q0, n1 + q1, B->row_ptr));
    GMT_TRY(put(o_col, sizeof(int32_t), e0, e1, B->col));
    GMT_TRY(put(o_cost, sizeof(double), e0, e1, B->cost));
    GMT_CUDA(cudaEventRecord(ctx->copy_done[ch], cs));
    GMT_CUDA(cudaStreamWaitEvent(s, ctx->copy_done[ch], 0));
    GMT_CUDA(launch_solve(static_cast<const SolveJob*>(ctx->jobs.ptr) + q0, q1 - q0, cluster, threads,
                          smem, obs, d, s, jobs[q0].res.counters != nullptr));
    ++ctx->launches;
    auto get = [&](void* dst, const void* src, size_t elem, int64_t first, int64_t last) -> int {
      if (!dst || last <= first) return GMT_OK;
      GMT_CUDA(cudaMemcpyAsync(static_cast<char*>(dst) + elem * first,
                               static_cast<const char*>(src) + elem * first, elem * (last - first),
                               cudaMemcpyDeviceToHost, s));
      return GMT_OK;
    };
    GMT_TRY(get(sc_host, sc_dev, sizeof(ResultScalars), q0, q1));
    GMT_TRY(get(paths, res[0].path, sizeof(int32_t), n0, n1));
    GMT_TRY(get(label, res[0].label, sizeof(uint8_t), n0, n1));
    GMT_TRY(get(tree_cost, res[0].tree_cost, sizeof(double), n0, n1));
    GMT_TRY(get(parent, res[0].parent, sizeof(int32_t), n0, n1));
    GMT_TRY(get(iteration_added, res[0].iter_added, sizeof(int64_t), n0, n1));
  }
  GMT_CUDA(cudaStreamSynchronize(s));
  for (int q = 0; q < count; ++q) to_summary(sc_host[q], &summaries[q]);
  return GMT_OK;
}
