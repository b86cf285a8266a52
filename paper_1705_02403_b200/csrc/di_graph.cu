// di_graph.cu -- the directed r-disk graphs of the kinodynamic steering
// models (the 6D double integrator, di.cuh, and the
// 12D linearised quadrotor, quad.cuh) built on the device, in the reference's
// NeighborGraph conventions (graph.cpp:117-188): out-row u = targets v != u
// with cost(u -> v) <= r ascending, in-row x = sources u with
// cost(u -> x) <= r ascending (the sequential merge order), path ids in
// (source, target) order (graph.cpp:172-183).
//
// Kernels (templated on the model): warp per row, lanes over 32 consecutive
// columns, the model's exact-safe prefilter then its steering solve per
// pair, ballot + popc ordered compaction; a count pass,
// an exclusive scan, a fill pass, for the out-rows and (roles swapped) the
// in-rows; optionally every out-edge's waypoint polyline.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <vector>

#include "common.cuh"
#include "di.cuh"
#include "quad.cuh"
#include "dubins.cuh"
#include "internal.cuh"
#include "offline.cuh"

namespace gmtb {

namespace {

constexpr uint32_t kFull = 0xffffffffu;

#define GMT_CUDA(call)                                   \
  do {                                                   \
    cudaError_t _e = (call);                             \
    if (_e != cudaSuccess) return cuda_error(_e, #call); \
  } while (0)

// Necessary condition for cost(x0 -> x1) <= r (no false rejections): the
// effort term is >= 3w (2D - (v0+v1) tau)^2 / tau^3 per axis and tau <= r, so
// |D| > vmax r + r^2 / (2 sqrt(3w)) on any axis rules the pair out.
__device__ __forceinline__ bool di_may_connect(const double* x0, const double* x1, double bound) {
  for (int k = 0; k < 3; ++k) {
    const double D = x1[k] - x0[k];
    if (D > bound || -D > bound) return false;
  }
  return true;
}

// The |dp| test, then the quartic lower bound of di_cost_exceeds (di.cuh).
__device__ __forceinline__ bool di_may_connect(const double* x0, const double* x1, double bound,
                                               const DiParams& P, double r) {
  if (!di_may_connect(x0, x1, bound)) return false;
  return !di_cost_exceeds(di_coef(x0, x1, P), r);
}

struct DiModel {
  static constexpr int kDim = kDiDim;
  DiParams P;
  double bound;  // di_prefilter_bound
  double radius;
  __device__ bool may(const double* a, const double* b) const { return di_may_connect(a, b, bound, P, radius); }
  // may == may_quick && may_confirm (di_cost_exceeds = whole || parts):
  // the cheap part first, the 12-part bound only for the pairs it passes
  __device__ bool may_quick(const double* a, const double* b) const {
    return di_may_connect(a, b, bound) && !di_cost_exceeds_whole(di_coef(a, b, P), radius);
  }
  __device__ bool may_confirm(const double* a, const double* b) const {
    return !di_cost_exceeds_parts(di_coef(a, b, P), radius);
  }
  __device__ double cost_tau(const double* a, const double* b, double* t) const {
    return di_cost_tau(a, b, P, t);
  }
  __device__ double cost_within(const double* a, const double* b, double r, double* t) const {
    return di_cost_tau(a, b, P, t, r);
  }
  __device__ double coord(const double* a, const double* b, double tau, int k, int i) const {
    return di_coord(a, b, tau, k, i, P);
  }
  int segments() const { return P.segments; }
};

struct QuadModel {
  static constexpr int kDim = kQuadDim;
  QuadParams P;
  double radius;
  __device__ bool may(const double* a, const double* b) const { return quad_may_connect(a, b, P, radius); }
  __device__ bool may_quick(const double* a, const double* b) const { return may(a, b); }
  __device__ bool may_confirm(const double*, const double*) const { return true; }
  __device__ double cost_tau(const double* a, const double* b, double* t) const {
    return quad_cost_tau(a, b, P, t);
  }
  __device__ double cost_within(const double* a, const double* b, double r, double* t) const {
    return quad_cost_tau(a, b, P, t, r);
  }
  __device__ double coord(const double* a, const double* b, double tau, int k, int i) const {
    return quad_coord(a, b, tau, k, i, P);
  }
  int segments() const { return P.segments; }
};

// Dubins airplane (dubins.cuh) over augmented states (x, y[, z], heading);
// `tau` carries connect()'s segment count (0 = degenerate pair).
template <int PD>
struct DubinsModel {
  static constexpr int kDim = PD + 1;
  DubinsParams P;
  double radius;
  // The reference's candidate set, exactly: the 3^axes grid cells around u
  // (graph.cpp:56-101: cell = max(r, 1e-9) on the first min(dim, 3) axes,
  // 21-bit cell keys) -- which bounds |dz| even when the cost ignores the
  // climb -- then within_radius's straight-line prune (steering.cpp:112-118):
  // hypot of the planar offsets (glibc's, libm_port.cuh) when the cost
  // ignores the climb, else euclidean_distance (space.cpp:126-133).
  __device__ bool may(const double* a, const double* b) const {
    const double cell = radius > 1e-9 ? radius : 1e-9;
    for (int k = 0; k < PD; ++k) {
      const int ca = static_cast<int>(floor(a[k] / cell)), cb = static_cast<int>(floor(b[k] / cell));
      const unsigned dk = static_cast<unsigned>(ca - cb) & 0x1fffffu;
      if (dk > 1u && dk != 0x1fffffu) return false;
    }
    double lb;
    if (P.planar_cost_only) {
      lb = lmport::lm_hypot(a[0] - b[0], a[1] - b[1]);
    } else {
      double sq = 0.0;
      for (int k = 0; k < PD; ++k) {
        const double d = a[k] - b[k];
        sq += d * d;
      }
      lb = sqrt(sq);
    }
    return !(lb > radius);
  }
  __device__ double cost_tau(const double* a, const double* b, double* t) const {
    int segs;
    DubinsPath path;
    double dz;
    const double c = dubins_connect(a, a[PD], b, b[PD], P, &segs, &path, &dz);
    *t = static_cast<double>(segs);
    return c;
  }
  __device__ double cost_within(const double* a, const double* b, double, double* t) const {
    return cost_tau(a, b, t);
  }
  __device__ double coord(const double*, const double*, double, int, int) const { return 0.0; }
  __device__ bool may_quick(const double* a, const double* b) const { return may(a, b); }
  __device__ bool may_confirm(const double*, const double*) const { return true; }
  int segments() const { return 0; }
};

// SWAP = false: row r lists targets c with cost(r -> c) <= radius.
// SWAP = true:  row r lists sources c with cost(c -> r) <= radius.
template <class Model, bool SWAP, bool FILL>
__global__ void __launch_bounds__(256) kino_rows_kernel(const double* __restrict__ coords, int n,
                                                        Model model, double radius,
                                                        int64_t* __restrict__ counts,
                                                      const int64_t* __restrict__ row_ptr,
                                                      int32_t* __restrict__ col,
                                                      double* __restrict__ cost,
                                                      double* __restrict__ tau) {
  const int lane = threadIdx.x & 31;
  const int warps = (blockDim.x >> 5) * gridDim.x;
  for (int r = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); r < n; r += warps) {
    constexpr int kD = Model::kDim;
    double xr[kD];
    for (int k = 0; k < kD; ++k) xr[k] = __ldg(coords + static_cast<int64_t>(r) * kD + k);
    int64_t out = FILL ? row_ptr[r] : 0;
    for (int base = 0; base < n; base += 32) {
      const int c = base + lane;
      bool keep = false;
      double cc = 0.0, tc = 0.0;
      if (c < n && c != r) {
        double xc[kD];
        for (int k = 0; k < kD; ++k) xc[k] = __ldg(coords + static_cast<int64_t>(c) * kD + k);
        const double* from = SWAP ? xc : xr;
        const double* to = SWAP ? xr : xc;
        if (model.may(from, to)) {
          cc = model.cost_within(from, to, radius, &tc);
          keep = cc <= radius;
        }
      }
      const uint32_t m = __ballot_sync(kFull, keep);
      if (FILL && keep) {
        const int64_t slot = out + __popc(m & ((1u << lane) - 1u));
        col[slot] = c;
        cost[slot] = cc;
        if (tau) tau[slot] = tc;
      }
      out += __popc(m);
    }
    if (!FILL && lane == 0) counts[r] = out;
  }
}

// in_path[e] for in-edge (u -> x): the out-edge index of (u -> x), found by
// binary search in u's sorted out-row (NeighborGraph::edge_path, graph.cpp:34-40).
__global__ void in_path_kernel(const int64_t* __restrict__ in_ptr, const int32_t* __restrict__ in_col,
                               const int64_t* __restrict__ out_ptr,
                               const int32_t* __restrict__ out_col, int n,
                               int32_t* __restrict__ in_path) {
  for (int x = blockIdx.x * blockDim.x + threadIdx.x; x < n; x += gridDim.x * blockDim.x) {
    for (int64_t e = in_ptr[x]; e < in_ptr[x + 1]; ++e) {
      const int u = in_col[e];
      int64_t lo = out_ptr[u], hi = out_ptr[u + 1];
      while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if (out_col[mid] < x) lo = mid + 1; else hi = mid;
      }
      in_path[e] = static_cast<int32_t>(lo);
    }
  }
}

// Waypoints of every out-edge: path e = pts[e*(M+1)*D ...] (M+1 states,
// the degenerate zero-duration edge repeats its single state).
template <class Model>
__global__ void kino_paths_kernel(const double* __restrict__ coords, const int64_t* __restrict__ out_ptr,
                                  const int32_t* __restrict__ out_col, const double* __restrict__ out_tau,
                                  int n, Model model, int M, double* __restrict__ pts) {
  constexpr int kD = Model::kDim;
  for (int u = blockIdx.x; u < n; u += gridDim.x) {
    const double* x0 = coords + static_cast<int64_t>(u) * kD;
    for (int64_t e = out_ptr[u] + threadIdx.x; e < out_ptr[u + 1]; e += blockDim.x) {
      const double* x1 = coords + static_cast<int64_t>(out_col[e]) * kD;
      double* p = pts + e * (M + 1) * kD;
      for (int k = 0; k <= M; ++k)
        for (int i = 0; i < kD; ++i) p[k * kD + i] = model.coord(x0, x1, out_tau[e], k, i);
    }
  }
}

template <class Model>
__global__ void kino_pairs_kernel(const double* __restrict__ x0s, const double* __restrict__ x1s,
                                  int64_t count, Model model, double* __restrict__ cost,
                                  double* __restrict__ tau) {
  constexpr int kD = Model::kDim;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < count;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    double t;
    cost[i] = model.cost_tau(x0s + i * kD, x1s + i * kD, &t);
    tau[i] = t;
  }
}

__global__ void __launch_bounds__(1024) scan_rows_kernel(const int64_t* __restrict__ counts, int n,
                                                         int64_t* __restrict__ row_ptr) {
  __shared__ int64_t warp_sum[32];
  __shared__ int64_t carry;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) carry = 0;
  __syncthreads();
  for (int base = 0; base < n; base += blockDim.x) {
    const int i = base + tid;
    const int64_t x = i < n ? counts[i] : 0;
    int64_t incl = x;
    for (int o = 1; o < 32; o <<= 1) {
      const int64_t y = __shfl_up_sync(kFull, incl, o);
      if (lane >= o) incl += y;
    }
    if (lane == 31) warp_sum[warp] = incl;
    __syncthreads();
    if (warp == 0) {
      int64_t w = lane < (blockDim.x >> 5) ? warp_sum[lane] : 0;
      for (int o = 1; o < 32; o <<= 1) {
        const int64_t y = __shfl_up_sync(kFull, w, o);
        if (lane >= o) w += y;
      }
      warp_sum[lane] = w;
    }
    __syncthreads();
    const int64_t before = carry + (warp > 0 ? warp_sum[warp - 1] : 0) + incl - x;
    if (i < n) row_ptr[i] = before;
    __syncthreads();
    if (tid == blockDim.x - 1) carry = before + x;
    __syncthreads();
  }
  if (tid == 0) row_ptr[n] = carry;
}

// Dubins edge paths (graph.cpp:152-156, 172-183): path e = out-edge e,
// segments + 1 states (the degenerate pair: its single state); positions
// only (the lazy check reads coordinates).
__global__ void dubins_path_count_kernel(const double* __restrict__ out_tau, int64_t E,
                                         int64_t* __restrict__ counts) {
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < E;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int segs = static_cast<int>(out_tau[e]);
    counts[e] = segs == 0 ? 1 : segs + 1;
  }
}

template <int PD>
__global__ void dubins_path_fill_kernel(const double* __restrict__ aug, const int64_t* __restrict__ out_ptr,
                                        const int32_t* __restrict__ out_col, int n, DubinsParams P,
                                        const int64_t* __restrict__ path_ptr, double* __restrict__ pts,
                                        int32_t* __restrict__ out_path) {
  for (int u = blockIdx.x; u < n; u += gridDim.x) {
    const double* a = aug + static_cast<int64_t>(u) * (PD + 1);
    for (int64_t e = out_ptr[u] + threadIdx.x; e < out_ptr[u + 1]; e += blockDim.x) {
      out_path[e] = static_cast<int32_t>(e);
      const double* b = aug + static_cast<int64_t>(out_col[e]) * (PD + 1);
      int segs;
      DubinsPath path;
      double dz;
      dubins_connect(a, a[PD], b, b[PD], P, &segs, &path, &dz);
      double* out = pts + path_ptr[e] * PD;
      if (segs == 0) {
        for (int k = 0; k < PD; ++k) out[k] = a[k];
        continue;
      }
      for (int i = 0; i <= segs; ++i) dubins_waypoint(a, b, path, dz, segs, i, P, out + i * PD);
    }
  }
}

// Segment counts of given out-edges (a cache hit): the builder's tau.
template <int PD>
__global__ void dubins_tau_kernel(const double* __restrict__ aug, const int64_t* __restrict__ out_ptr,
                                  const int32_t* __restrict__ out_col, int n, DubinsParams P,
                                  double* __restrict__ tau) {
  for (int u = blockIdx.x; u < n; u += gridDim.x) {
    const double* a = aug + static_cast<int64_t>(u) * (PD + 1);
    for (int64_t e = out_ptr[u] + threadIdx.x; e < out_ptr[u + 1]; e += blockDim.x) {
      const double* b = aug + static_cast<int64_t>(out_col[e]) * (PD + 1);
      int segs;
      DubinsPath path;
      double dz;
      dubins_connect(a, a[PD], b, b[PD], P, &segs, &path, &dz);
      tau[e] = static_cast<double>(segs);
    }
  }
}

__global__ void augment_kernel(const double* __restrict__ coords, const double* __restrict__ heading, int n,
                               int pd, double* __restrict__ aug) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    for (int k = 0; k < pd; ++k) aug[static_cast<int64_t>(i) * (pd + 1) + k] = coords[static_cast<int64_t>(i) * pd + k];
    aug[static_cast<int64_t>(i) * (pd + 1) + pd] = heading[i];
  }
}

template <class Model>
int rows_pass(gmt_ctx* ctx, bool swap, const double* coords, int n, const Model& model, double radius,
              Arena& mem, DiRows* rows, bool with_tau) {
  cudaStream_t s = ctx->stream;
  const int blocks = std::max(1, std::min((n + 7) / 8, ctx->sm_count * 8));
  Arena cnt;
  int rc = cnt.reserve(sizeof(int64_t) * (n + 1));
  if (rc) return rc;
  int64_t* counts = static_cast<int64_t*>(cnt.ptr);
  if (swap)
    kino_rows_kernel<Model, true, false><<<blocks, 256, 0, s>>>(coords, n, model, radius, counts, nullptr,
                                                                nullptr, nullptr, nullptr);
  else
    kino_rows_kernel<Model, false, false><<<blocks, 256, 0, s>>>(coords, n, model, radius, counts, nullptr,
                                                                 nullptr, nullptr, nullptr);
  GMT_CUDA(cudaGetLastError());
  Arena rp;
  rc = rp.reserve(sizeof(int64_t) * (n + 1));
  if (rc) {
    cnt.release();
    return rc;
  }
  scan_rows_kernel<<<1, 1024, 0, s>>>(counts, n, static_cast<int64_t*>(rp.ptr));
  GMT_CUDA(cudaGetLastError());
  ctx->launches += 2;
  int64_t E = 0;
  GMT_CUDA(cudaMemcpyAsync(&E, static_cast<int64_t*>(rp.ptr) + n, sizeof(E), cudaMemcpyDeviceToHost, s));
  GMT_CUDA(cudaStreamSynchronize(s));
  const size_t o_ptr = 0;
  const size_t o_col = align16(sizeof(int64_t) * (n + 1));
  const size_t o_cost = o_col + align16(sizeof(int32_t) * E);
  const size_t o_tau = o_cost + align16(sizeof(double) * E);
  const size_t total = o_tau + (with_tau ? align16(sizeof(double) * E) : 0);
  rc = mem.reserve(total);
  if (rc) {
    cnt.release();
    rp.release();
    return rc;
  }
  char* b = static_cast<char*>(mem.ptr);
  rows->ptr = reinterpret_cast<int64_t*>(b + o_ptr);
  rows->col = reinterpret_cast<int32_t*>(b + o_col);
  rows->cost = reinterpret_cast<double*>(b + o_cost);
  rows->tau = with_tau ? reinterpret_cast<double*>(b + o_tau) : nullptr;
  rows->edges = E;
  GMT_CUDA(cudaMemcpyAsync(rows->ptr, rp.ptr, sizeof(int64_t) * (n + 1), cudaMemcpyDeviceToDevice, s));
  if (swap)
    kino_rows_kernel<Model, true, true><<<blocks, 256, 0, s>>>(coords, n, model, radius, nullptr, rows->ptr,
                                                               rows->col, rows->cost, rows->tau);
  else
    kino_rows_kernel<Model, false, true><<<blocks, 256, 0, s>>>(coords, n, model, radius, nullptr,
                                                                rows->ptr, rows->col, rows->cost, rows->tau);
  GMT_CUDA(cudaGetLastError());
  ++ctx->launches;
  GMT_CUDA(cudaStreamSynchronize(s));
  cnt.release();
  rp.release();
  return GMT_OK;
}

// One evaluation per pair: warp per source row u, the keep bit of every
// target chunk goes into an n x ceil(n/32) bit matrix (the ballot word),
// with out-degrees and in-degrees counted on the way.
template <class Model>
__global__ void __launch_bounds__(256) kino_eval_kernel(const double* __restrict__ coords, int n,
                                                        Model model, double radius,
                                                        uint32_t* __restrict__ bits, int W,
                                                        int64_t* __restrict__ out_counts,
                                                        int64_t* __restrict__ in_counts) {
  // The few columns that pass the cheap prefilter (may_quick) are queued
  // per warp and run through the rest of the test and the capped 2BVP
  // search 32 at a time, so no 32-column chunk waits on one lane's search.
  // Same keep bits and counts as testing every pair in place.
  constexpr int kD = Model::kDim;
  __shared__ int32_t queue_s[8][64];
  const int lane = threadIdx.x & 31;
  int32_t* const queue = queue_s[(threadIdx.x >> 5) & 7];
  const int warps = (blockDim.x >> 5) * gridDim.x;
  for (int r = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); r < n; r += warps) {
    double xr[kD];
    for (int k = 0; k < kD; ++k) xr[k] = __ldg(coords + static_cast<int64_t>(r) * kD + k);
    uint32_t* const brow = bits + static_cast<int64_t>(r) * W;
    int64_t cnt = 0;
    int qn = 0;
    auto drain = [&](int take) {  // evaluate queue[0, take), keep the rest
      bool keep = false;
      int c = 0;
      if (lane < take) {
        c = queue[lane];
        double xc[kD];
        for (int k = 0; k < kD; ++k) xc[k] = __ldg(coords + static_cast<int64_t>(c) * kD + k);
        if (model.may_confirm(xr, xc)) {
          double tc;
          keep = model.cost_within(xr, xc, radius, &tc) <= radius;
        }
      }
      if (keep) {
        atomicOr(brow + (c >> 5), 1u << (c & 31));
        atomicAdd(reinterpret_cast<unsigned long long*>(in_counts + c), 1ull);
      }
      cnt += __popc(__ballot_sync(kFull, keep));
      const int rest = lane + take < qn ? queue[lane + take] : 0;
      __syncwarp();
      if (lane + take < qn) queue[lane] = rest;
      qn -= take;
      __syncwarp();
    };
    for (int w = 0; w < W; ++w) {
      const int c = w * 32 + lane;
      bool may = false;
      if (c < n && c != r) {
        double xc[kD];
        for (int k = 0; k < kD; ++k) xc[k] = __ldg(coords + static_cast<int64_t>(c) * kD + k);
        may = model.may_quick(xr, xc);
      }
      if (lane == 0) brow[w] = 0u;  // (before any atomicOr into this word: queued columns are >= 32 w)
      const uint32_t m = __ballot_sync(kFull, may);
      if (may) queue[qn + __popc(m & ((1u << lane) - 1u))] = c;
      qn += __popc(m);
      __syncwarp();
      if (qn >= 32) drain(32);
    }
    while (qn > 0) drain(qn < 32 ? qn : 32);
    if (lane == 0) out_counts[r] = cnt;
  }
}

// Out-rows from the bit matrix: only kept pairs are evaluated again (the
// same capped search, so the same cost and duration).
template <class Model>
__global__ void __launch_bounds__(256) kino_out_fill_kernel(const double* __restrict__ coords, int n,
                                                            Model model, double radius,
                                                            const uint32_t* __restrict__ bits, int W,
                                                            const int64_t* __restrict__ row_ptr,
                                                            int32_t* __restrict__ col,
                                                            double* __restrict__ cost,
                                                            double* __restrict__ tau) {
  // The row's kept columns are queued in order and solved 32 at a time
  // (lane i -> slot out + i), not one word's few set bits per warp step.
  constexpr int kD = Model::kDim;
  __shared__ int32_t queue_s[8][64];
  const int lane = threadIdx.x & 31;
  int32_t* const queue = queue_s[(threadIdx.x >> 5) & 7];
  const int warps = (blockDim.x >> 5) * gridDim.x;
  for (int r = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); r < n; r += warps) {
    double xr[kD];
    for (int k = 0; k < kD; ++k) xr[k] = __ldg(coords + static_cast<int64_t>(r) * kD + k);
    int64_t out = row_ptr[r];
    int qn = 0;
    auto drain = [&](int take) {
      if (lane < take) {
        const int c = queue[lane];
        double xc[kD];
        for (int k = 0; k < kD; ++k) xc[k] = __ldg(coords + static_cast<int64_t>(c) * kD + k);
        double tc;
        const double cc = model.cost_within(xr, xc, radius, &tc);
        col[out + lane] = c;
        cost[out + lane] = cc;
        tau[out + lane] = tc;
      }
      const int rest = lane + take < qn ? queue[lane + take] : 0;
      __syncwarp();
      if (lane + take < qn) queue[lane] = rest;
      out += take;
      qn -= take;
      __syncwarp();
    };
    for (int w = 0; w < W; ++w) {
      const uint32_t m = __ldg(bits + static_cast<int64_t>(r) * W + w);
      if (!m) continue;
      if ((m >> lane) & 1u) queue[qn + __popc(m & ((1u << lane) - 1u))] = w * 32 + lane;
      qn += __popc(m);
      __syncwarp();
      if (qn >= 32) drain(32);
    }
    while (qn > 0) drain(qn < 32 ? qn : 32);
  }
}

// In-rows = the bit matrix's columns, sources ascending (the reference's
// sequential merge order, graph.cpp:184-186); each entry copies the
// out-edge's cost and duration (the same pair, the same computation).
__global__ void __launch_bounds__(256) kino_in_fill_kernel(const uint32_t* __restrict__ bits, int W, int n,
                                                           const int64_t* __restrict__ out_ptr,
                                                           const int32_t* __restrict__ out_col,
                                                           const double* __restrict__ out_cost,
                                                           const double* __restrict__ out_tau,
                                                           const int64_t* __restrict__ in_ptr,
                                                           int32_t* __restrict__ in_col,
                                                           double* __restrict__ in_cost,
                                                           double* __restrict__ in_tau) {
  const int lane = threadIdx.x & 31;
  const int warps = (blockDim.x >> 5) * gridDim.x;
  for (int x = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); x < n; x += warps) {
    const int wx = x >> 5;
    const uint32_t bx = 1u << (x & 31);
    int64_t out = in_ptr[x];
    for (int base = 0; base < n; base += 32) {
      const int u = base + lane;
      const bool kept = u < n && (__ldg(bits + static_cast<int64_t>(u) * W + wx) & bx);
      const uint32_t m = __ballot_sync(kFull, kept);
      if (kept) {
        int64_t lo = out_ptr[u], hi = out_ptr[u + 1];
        while (lo < hi) {  // NeighborGraph::edge_path lookup (graph.cpp:34-40)
          const int64_t mid = (lo + hi) >> 1;
          if (out_col[mid] < x) lo = mid + 1; else hi = mid;
        }
        const int64_t slot = out + __popc(m & ((1u << lane) - 1u));
        in_col[slot] = u;
        in_cost[slot] = out_cost[lo];
        in_tau[slot] = out_tau[lo];
      }
      out += __popc(m);
    }
  }
}

int carve_rows(Arena& mem, int n, int64_t E, DiRows* rows) {
  const size_t o_col = align16(sizeof(int64_t) * (n + 1));
  const size_t o_cost = o_col + align16(sizeof(int32_t) * E);
  const size_t o_tau = o_cost + align16(sizeof(double) * E);
  const size_t total = o_tau + align16(sizeof(double) * E);
  const int rc = mem.reserve(total);
  if (rc) return rc;
  char* b = static_cast<char*>(mem.ptr);
  rows->ptr = reinterpret_cast<int64_t*>(b);
  rows->col = reinterpret_cast<int32_t*>(b + o_col);
  rows->cost = reinterpret_cast<double*>(b + o_cost);
  rows->tau = reinterpret_cast<double*>(b + o_tau);
  rows->edges = E;
  return GMT_OK;
}

template <class Model>
int build_kino_graph_dev(gmt_ctx* ctx, const double* d_coords, int n, const Model& model, double radius,
                         Arena& out_mem, DiRows* out, Arena& in_mem, DiRows* in) {
  if (!(radius > 0.0)) return set_error(GMT_E_INVALID_INPUT, "connection radius must be positive");
  if (n < 1) return set_error(GMT_E_INVALID_INPUT, "cannot build a graph over zero samples");
  const int W = (n + 31) / 32;
  const size_t bit_bytes = sizeof(uint32_t) * static_cast<size_t>(n) * W;
  if (bit_bytes > (size_t(1) << 31)) {  // very large n: two evaluations per pair per direction
    int rc = rows_pass(ctx, false, d_coords, n, model, radius, out_mem, out, true);
    if (rc) return rc;
    return rows_pass(ctx, true, d_coords, n, model, radius, in_mem, in, true);
  }
  cudaStream_t s = ctx->stream;
  const size_t o_oc = align16(bit_bytes);
  const size_t o_ic = o_oc + align16(sizeof(int64_t) * (n + 1));
  const size_t o_op = o_ic + align16(sizeof(int64_t) * (n + 1));
  const size_t o_ip = o_op + align16(sizeof(int64_t) * (n + 1));
  Arena tmp;
  int rc = tmp.reserve(o_ip + sizeof(int64_t) * (n + 1));
  if (rc) return rc;
  char* b = static_cast<char*>(tmp.ptr);
  auto* bits = reinterpret_cast<uint32_t*>(b);
  auto* oc = reinterpret_cast<int64_t*>(b + o_oc);
  auto* ic = reinterpret_cast<int64_t*>(b + o_ic);
  auto* op = reinterpret_cast<int64_t*>(b + o_op);
  auto* ip = reinterpret_cast<int64_t*>(b + o_ip);
  GMT_CUDA(cudaMemsetAsync(ic, 0, sizeof(int64_t) * (n + 1), s));
  const int blocks = std::max(1, std::min((n + 7) / 8, ctx->sm_count * 8));
  kino_eval_kernel<Model><<<blocks, 256, 0, s>>>(d_coords, n, model, radius, bits, W, oc, ic);
  GMT_CUDA(cudaGetLastError());
  scan_rows_kernel<<<1, 1024, 0, s>>>(oc, n, op);
  scan_rows_kernel<<<1, 1024, 0, s>>>(ic, n, ip);
  GMT_CUDA(cudaGetLastError());
  ctx->launches += 3;
  int64_t E = 0;
  GMT_CUDA(cudaMemcpyAsync(&E, op + n, sizeof(E), cudaMemcpyDeviceToHost, s));
  GMT_CUDA(cudaStreamSynchronize(s));
  rc = carve_rows(out_mem, n, E, out);
  if (rc == GMT_OK) rc = carve_rows(in_mem, n, E, in);
  if (rc) {
    tmp.release();
    return rc;
  }
  GMT_CUDA(cudaMemcpyAsync(out->ptr, op, sizeof(int64_t) * (n + 1), cudaMemcpyDeviceToDevice, s));
  GMT_CUDA(cudaMemcpyAsync(in->ptr, ip, sizeof(int64_t) * (n + 1), cudaMemcpyDeviceToDevice, s));
  kino_out_fill_kernel<Model><<<blocks, 256, 0, s>>>(d_coords, n, model, radius, bits, W, out->ptr, out->col,
                                                     out->cost, out->tau);
  GMT_CUDA(cudaGetLastError());
  kino_in_fill_kernel<<<blocks, 256, 0, s>>>(bits, W, n, out->ptr, out->col, out->cost, out->tau, in->ptr,
                                             in->col, in->cost, in->tau);
  GMT_CUDA(cudaGetLastError());
  ctx->launches += 2;
  GMT_CUDA(cudaStreamSynchronize(s));
  tmp.release();
  return GMT_OK;
}


}  // namespace

double di_prefilter_bound(const DiParams& P, double radius) {
  // vmax r + r^2 / (2 sqrt(3 w)), widened by 1e-9 relative against rounding.
  return (P.vmax * radius + radius * radius / (2.0 * std::sqrt(3.0 * P.weight))) * (1.0 + 1e-9) + 1e-12;
}

namespace {

DiModel di_model(const gmt_di_params* p, double radius) {
  DiModel m;
  m.P = to_di(p);
  m.bound = di_prefilter_bound(m.P, radius);
  m.radius = radius;
  return m;
}

QuadModel quad_model(const gmt_quad_params* p, double radius) {
  QuadModel m;
  m.P = to_quad(p);
  m.radius = radius;
  return m;
}

template <class Model>
int kino_costs(gmt_ctx* ctx, const double* x0s, const double* x1s, int64_t count, const Model& model,
               double* cost_out, double* tau_out) {
  if (count <= 0) return GMT_OK;
  constexpr int kD = Model::kDim;
  Arena buf;
  const size_t xs = sizeof(double) * kD * static_cast<size_t>(count);
  int rc = buf.reserve(2 * xs + 2 * sizeof(double) * count);
  if (rc) return rc;
  double* d0 = static_cast<double*>(buf.ptr);
  double* d1 = d0 + kD * count;
  double* dc = d1 + kD * count;
  double* dt = dc + count;
  cudaStream_t s = ctx->stream;
  GMT_CUDA(cudaMemcpyAsync(d0, x0s, xs, cudaMemcpyHostToDevice, s));
  GMT_CUDA(cudaMemcpyAsync(d1, x1s, xs, cudaMemcpyHostToDevice, s));
  const int blocks = static_cast<int>(std::min<int64_t>((count + 255) / 256, 4096));
  kino_pairs_kernel<Model><<<blocks, 256, 0, s>>>(d0, d1, count, model, dc, dt);
  GMT_CUDA(cudaGetLastError());
  ++ctx->launches;
  GMT_CUDA(cudaMemcpyAsync(cost_out, dc, sizeof(double) * count, cudaMemcpyDeviceToHost, s));
  GMT_CUDA(cudaMemcpyAsync(tau_out, dt, sizeof(double) * count, cudaMemcpyDeviceToHost, s));
  GMT_CUDA(cudaStreamSynchronize(s));
  buf.release();
  return GMT_OK;
}

template <class Model>
int build_kino_graph_host(gmt_ctx* ctx, const double* coords, int32_t n, const Model& model, double radius,
                          int64_t* num_edges, int64_t* out_ptr, int32_t* out_col, double* out_cost,
                          double* out_tau, int64_t* in_ptr, int32_t* in_col, double* in_cost,
                          int32_t* in_path, double* path_pts) {
  if (n < 1) return set_error(GMT_E_INVALID_INPUT, "cannot build a graph over zero samples");
  constexpr int kD = Model::kDim;
  const int M = model.segments();
  cudaStream_t s = ctx->stream;
  Arena cbuf;
  int rc = cbuf.reserve(sizeof(double) * kD * static_cast<size_t>(n));
  if (rc) return rc;
  GMT_CUDA(cudaMemcpyAsync(cbuf.ptr, coords, sizeof(double) * kD * n, cudaMemcpyHostToDevice, s));
  const double* dc = static_cast<const double*>(cbuf.ptr);
  Arena om, im;
  DiRows o, in;
  rc = build_kino_graph_dev(ctx, dc, n, model, radius, om, &o, im, &in);
  if (rc) {
    cbuf.release();
    return rc;
  }
  *num_edges = o.edges;
  if (out_ptr) {
    auto get = [&](void* dst, const void* src, size_t bytes) -> int {
      if (dst && bytes) GMT_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, s));
      return GMT_OK;
    };
    const size_t E = static_cast<size_t>(o.edges);
    get(out_ptr, o.ptr, sizeof(int64_t) * (n + 1));
    get(out_col, o.col, sizeof(int32_t) * E);
    get(out_cost, o.cost, sizeof(double) * E);
    get(out_tau, o.tau, sizeof(double) * E);
    get(in_ptr, in.ptr, sizeof(int64_t) * (n + 1));
    get(in_col, in.col, sizeof(int32_t) * E);
    get(in_cost, in.cost, sizeof(double) * E);
    Arena extra;
    if (in_path || path_pts) {
      const size_t pts_bytes = path_pts ? sizeof(double) * E * (M + 1) * kD : 0;
      rc = extra.reserve(sizeof(int32_t) * E + pts_bytes + 16);
      if (rc) return rc;
      int32_t* ip = static_cast<int32_t*>(extra.ptr);
      double* pp = reinterpret_cast<double*>(static_cast<char*>(extra.ptr) + align16(sizeof(int32_t) * E));
      if (in_path) {
        in_path_kernel<<<std::max(1, std::min((n + 255) / 256, 1024)), 256, 0, s>>>(in.ptr, in.col, o.ptr,
                                                                               o.col, n, ip);
        GMT_CUDA(cudaGetLastError());
        ++ctx->launches;
        get(in_path, ip, sizeof(int32_t) * E);
      }
      if (path_pts) {
        kino_paths_kernel<Model><<<std::max(1, std::min(n, 4096)), 128, 0, s>>>(dc, o.ptr, o.col, o.tau, n,
                                                                               model, M, pp);
        GMT_CUDA(cudaGetLastError());
        ++ctx->launches;
        get(path_pts, pp, pts_bytes);
      }
      GMT_CUDA(cudaStreamSynchronize(s));
      extra.release();
    }
    GMT_CUDA(cudaStreamSynchronize(s));
  }
  om.release();
  im.release();
  cbuf.release();
  return GMT_OK;
}

}  // namespace

DiParams to_di(const gmt_di_params* p) {
  DiParams P;
  P.vmax = p->vmax;
  P.weight = p->weight;
  P.segments = p->segments;
  P.reserved = 0;
  return P;
}

QuadParams to_quad(const gmt_quad_params* p) {
  QuadParams P;
  P.g = p->g;
  P.vmax = p->vmax;
  P.amax = p->amax;
  P.ymax = p->ymax;
  P.wmax = p->wmax;
  P.weight = p->weight;
  P.segments = p->segments;
  P.reserved = 0;
  return P;
}

int validate_di(const gmt_di_params* p) {
  if (!p) return set_error(GMT_E_INVALID_INPUT, "double-integrator parameters are null");
  if (!(p->vmax > 0.0)) return set_error(GMT_E_INVALID_INPUT, "di.vmax must be positive");
  if (!(p->weight > 0.0)) return set_error(GMT_E_INVALID_INPUT, "di.weight must be positive");
  if (p->segments < 1 || p->segments > 64)
    return set_error(GMT_E_INVALID_INPUT, "di.segments must be in [1, 64]");
  return GMT_OK;
}

int validate_quad(const gmt_quad_params* p) {
  if (!p) return set_error(GMT_E_INVALID_INPUT, "quadrotor parameters are null");
  if (!(p->g > 0.0) || !(p->vmax > 0.0) || !(p->amax > 0.0) || !(p->ymax > 0.0) || !(p->wmax > 0.0) ||
      !(p->weight > 0.0))
    return set_error(GMT_E_INVALID_INPUT, "quad.g, vmax, amax, ymax, wmax, weight must be positive");
  if (p->segments < 1 || p->segments > 64)
    return set_error(GMT_E_INVALID_INPUT, "quad.segments must be in [1, 64]");
  return GMT_OK;
}

int build_di_graph_dev(gmt_ctx* ctx, const double* d_coords, int n, const gmt_di_params* p, double radius,
                       Arena& out_mem, DiRows* out, Arena& in_mem, DiRows* in) {
  return build_kino_graph_dev(ctx, d_coords, n, di_model(p, radius), radius, out_mem, out, in_mem, in);
}

int build_quad_graph_dev(gmt_ctx* ctx, const double* d_coords, int n, const gmt_quad_params* p,
                         double radius, Arena& out_mem, DiRows* out, Arena& in_mem, DiRows* in) {
  return build_kino_graph_dev(ctx, d_coords, n, quad_model(p, radius), radius, out_mem, out, in_mem, in);
}

DubinsParams to_dubins(const gmt_dubins_params* p, int pd) {
  DubinsParams P;
  P.rho = p->rho;
  P.step = p->discretization_step > 0.0 ? p->discretization_step : p->rho / 10.0;  // step()
  P.planar_cost_only = p->planar_cost_only != 0;
  P.dim = pd;
  return P;
}

int validate_dubins(const gmt_dubins_params* p, int pd) {
  if (!p) return set_error(GMT_E_INVALID_INPUT, "dubins parameters are null");
  if (pd != 2 && pd != 3) return set_error(GMT_E_INVALID_INPUT, "dubins steering needs 2 or 3 position coordinates");
  if (!(p->rho > 0.0)) return set_error(GMT_E_INVALID_INPUT, "dubins turning radius must be positive");
  return GMT_OK;
}

// Out-rows from a graph cache file (graph.cpp:322-341): costs as stored;
// in-rows = the transpose with sources ascending (g.in[e.other].push_back
// in u order); segment counts recomputed on the device.
int dubins_rows_from_host(gmt_ctx* ctx, const double* A, int n, int pd, const DubinsParams& P, const HostRows& h,
                          Arena& out_mem, DiRows* out, Arena& in_mem, DiRows* in) {
  const std::vector<int64_t>& hp = *h.ptr;
  const std::vector<int32_t>& hc = *h.col;
  const std::vector<double>& hw = *h.cost;
  const int64_t E = static_cast<int64_t>(hc.size());
  int rc = carve_rows(out_mem, n, E, out);
  if (rc == GMT_OK) rc = carve_rows(in_mem, n, E, in);
  if (rc) return rc;
  std::vector<int64_t> ip(static_cast<size_t>(n) + 1, 0);
  for (int64_t e = 0; e < E; ++e) ++ip[static_cast<size_t>(hc[e]) + 1];
  for (int v = 0; v < n; ++v) ip[v + 1] += ip[v];
  std::vector<int64_t> at(ip.begin(), ip.end() - 1);
  std::vector<int32_t> ic(static_cast<size_t>(E));
  std::vector<double> iw(static_cast<size_t>(E));
  for (int u = 0; u < n; ++u)
    for (int64_t e = hp[u]; e < hp[u + 1]; ++e) {
      const int64_t k = at[hc[e]]++;
      ic[k] = u;
      iw[k] = hw[e];
    }
  cudaStream_t s = ctx->stream;
  GMT_CUDA(cudaMemcpyAsync(out->ptr, hp.data(), sizeof(int64_t) * (n + 1), cudaMemcpyHostToDevice, s));
  GMT_CUDA(cudaMemcpyAsync(in->ptr, ip.data(), sizeof(int64_t) * (n + 1), cudaMemcpyHostToDevice, s));
  if (E) {
    GMT_CUDA(cudaMemcpyAsync(out->col, hc.data(), sizeof(int32_t) * E, cudaMemcpyHostToDevice, s));
    GMT_CUDA(cudaMemcpyAsync(out->cost, hw.data(), sizeof(double) * E, cudaMemcpyHostToDevice, s));
    GMT_CUDA(cudaMemcpyAsync(in->col, ic.data(), sizeof(int32_t) * E, cudaMemcpyHostToDevice, s));
    GMT_CUDA(cudaMemcpyAsync(in->cost, iw.data(), sizeof(double) * E, cudaMemcpyHostToDevice, s));
    GMT_CUDA(cudaMemsetAsync(in->tau, 0, sizeof(double) * E, s));
    const int nb = std::max(1, std::min(n, 4096));
    if (pd == 2)
      dubins_tau_kernel<2><<<nb, 128, 0, s>>>(A, out->ptr, out->col, n, P, out->tau);
    else
      dubins_tau_kernel<3><<<nb, 128, 0, s>>>(A, out->ptr, out->col, n, P, out->tau);
    GMT_CUDA(cudaGetLastError());
    ++ctx->launches;
  }
  GMT_CUDA(cudaStreamSynchronize(s));  // (the host vectors go out of scope)
  return GMT_OK;
}

// The directed Dubins graph of device samples (positions + headings):
// out-/in-rows as build_kino_graph_dev (or as a cache file gives them), plus
// every out-edge's path.
int build_dubins_graph_dev(gmt_ctx* ctx, const double* d_coords, const double* d_heading, int n, int pd,
                           const gmt_dubins_params* p, double radius, Arena& out_mem, DiRows* out,
                           Arena& in_mem, DiRows* in, Arena& path_mem, DubinsGraphPaths* paths,
                           const HostRows* cached) {
  int rc = validate_dubins(p, pd);
  if (rc) return rc;
  const DubinsParams P = to_dubins(p, pd);
  cudaStream_t s = ctx->stream;
  Arena aug;
  rc = aug.reserve(sizeof(double) * static_cast<size_t>(n) * (pd + 1));
  if (rc) return rc;
  augment_kernel<<<std::max(1, std::min((n + 255) / 256, 1024)), 256, 0, s>>>(d_coords, d_heading, n, pd,
                                                                            static_cast<double*>(aug.ptr));
  GMT_CUDA(cudaGetLastError());
  ++ctx->launches;
  const double* A = static_cast<const double*>(aug.ptr);
  if (cached) {
    rc = dubins_rows_from_host(ctx, A, n, pd, P, *cached, out_mem, out, in_mem, in);
  } else if (pd == 2) {
    DubinsModel<2> m{P, radius};
    rc = build_kino_graph_dev(ctx, A, n, m, radius, out_mem, out, in_mem, in);
  } else {
    DubinsModel<3> m{P, radius};
    rc = build_kino_graph_dev(ctx, A, n, m, radius, out_mem, out, in_mem, in);
  }
  if (rc) {
    aug.release();
    return rc;
  }
  const int64_t E = out->edges;
  Arena cnt;
  rc = cnt.reserve(sizeof(int64_t) * (E + 1));
  if (rc) {
    aug.release();
    return rc;
  }
  int64_t* counts = static_cast<int64_t*>(cnt.ptr);
  const int eb = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>((E + 255) / 256, 4096)));
  dubins_path_count_kernel<<<eb, 256, 0, s>>>(out->tau, E, counts);
  // path_ptr [E+1], in_path [E], out_path [E], then the points
  const size_t o_pp = 0;
  const size_t o_ip = align16(sizeof(int64_t) * (E + 1));
  const size_t o_op = o_ip + align16(sizeof(int32_t) * E);
  const size_t o_pts = o_op + align16(sizeof(int32_t) * E);
  Arena pp;
  rc = pp.reserve(sizeof(int64_t) * (E + 1));
  if (rc == GMT_OK) {
    scan_rows_kernel<<<1, 1024, 0, s>>>(counts, static_cast<int>(E), static_cast<int64_t*>(pp.ptr));
    GMT_CUDA(cudaGetLastError());
    ctx->launches += 2;
    int64_t total = 0;
    GMT_CUDA(cudaMemcpyAsync(&total, static_cast<int64_t*>(pp.ptr) + E, sizeof(total), cudaMemcpyDeviceToHost, s));
    GMT_CUDA(cudaStreamSynchronize(s));
    rc = path_mem.reserve(o_pts + sizeof(double) * static_cast<size_t>(total) * pd + 16);
    if (rc == GMT_OK) {
      char* b = static_cast<char*>(path_mem.ptr);
      paths->path_ptr = reinterpret_cast<int64_t*>(b + o_pp);
      paths->in_path = reinterpret_cast<int32_t*>(b + o_ip);
      paths->out_path = reinterpret_cast<int32_t*>(b + o_op);
      paths->pts = reinterpret_cast<double*>(b + o_pts);
      paths->num_points = total;
      GMT_CUDA(cudaMemcpyAsync(paths->path_ptr, pp.ptr, sizeof(int64_t) * (E + 1), cudaMemcpyDeviceToDevice, s));
      const int nb = std::max(1, std::min(n, 4096));
      if (pd == 2)
        dubins_path_fill_kernel<2><<<nb, 128, 0, s>>>(A, out->ptr, out->col, n, P, paths->path_ptr, paths->pts,
                                                      paths->out_path);
      else
        dubins_path_fill_kernel<3><<<nb, 128, 0, s>>>(A, out->ptr, out->col, n, P, paths->path_ptr, paths->pts,
                                                      paths->out_path);
      GMT_CUDA(cudaGetLastError());
      in_path_kernel<<<std::max(1, std::min((n + 255) / 256, 1024)), 256, 0, s>>>(in->ptr, in->col, out->ptr,
                                                                             out->col, n, paths->in_path);
      GMT_CUDA(cudaGetLastError());
      ctx->launches += 2;
      GMT_CUDA(cudaStreamSynchronize(s));
    }
  }
  pp.release();
  cnt.release();
  aug.release();
  return rc;
}

}  // namespace gmtb

using namespace gmtb;

extern "C" int gmt_di_costs(gmt_ctx* ctx, const double* x0s, const double* x1s, int64_t count,
                            const gmt_di_params* params, double* cost_out, double* tau_out) {
  gmtb::AllocScope alloc_scope_(ctx);
  int rc = validate_di(params);
  if (rc) return rc;
  return kino_costs(ctx, x0s, x1s, count, di_model(params, 1.0), cost_out, tau_out);
}

extern "C" int gmt_quad_costs(gmt_ctx* ctx, const double* x0s, const double* x1s, int64_t count,
                              const gmt_quad_params* params, double* cost_out, double* tau_out) {
  gmtb::AllocScope alloc_scope_(ctx);
  int rc = validate_quad(params);
  if (rc) return rc;
  return kino_costs(ctx, x0s, x1s, count, quad_model(params, 1.0), cost_out, tau_out);
}

extern "C" int gmt_build_di_graph(gmt_ctx* ctx, const double* coords, int32_t n,
                                  const gmt_di_params* params, double radius, int64_t* num_edges,
                                  int64_t* out_ptr, int32_t* out_col, double* out_cost,
                                  double* out_tau, int64_t* in_ptr, int32_t* in_col,
                                  double* in_cost, int32_t* in_path, double* path_pts) {
  gmtb::AllocScope alloc_scope_(ctx);
  int rc = validate_di(params);
  if (rc) return rc;
  return build_kino_graph_host(ctx, coords, n, di_model(params, radius), radius, num_edges, out_ptr,
                               out_col, out_cost, out_tau, in_ptr, in_col, in_cost, in_path, path_pts);
}

extern "C" int gmt_build_quad_graph(gmt_ctx* ctx, const double* coords, int32_t n,
                                    const gmt_quad_params* params, double radius, int64_t* num_edges,
                                    int64_t* out_ptr, int32_t* out_col, double* out_cost,
                                    double* out_tau, int64_t* in_ptr, int32_t* in_col,
                                    double* in_cost, int32_t* in_path, double* path_pts) {
  gmtb::AllocScope alloc_scope_(ctx);
  int rc = validate_quad(params);
  if (rc) return rc;
  return build_kino_graph_host(ctx, coords, n, quad_model(params, radius), radius, num_edges, out_ptr,
                               out_col, out_cost, out_tau, in_ptr, in_col, in_cost, in_path, path_pts);
}

extern "C" int gmt_dubins_costs(gmt_ctx* ctx, const double* x0s, const double* x1s, int64_t count, int32_t dim,
                                const gmt_dubins_params* params, double* cost_out, int32_t* segments_out) {
  gmtb::AllocScope alloc_scope_(ctx);
  int rc = validate_dubins(params, dim);
  if (rc) return rc;
  if (count <= 0) return GMT_OK;
  std::vector<double> segs(static_cast<size_t>(count));
  const DubinsParams P = to_dubins(params, dim);
  if (dim == 2)
    rc = kino_costs(ctx, x0s, x1s, count, DubinsModel<2>{P, 0.0}, cost_out, segs.data());
  else
    rc = kino_costs(ctx, x0s, x1s, count, DubinsModel<3>{P, 0.0}, cost_out, segs.data());
  if (rc) return rc;
  for (int64_t i = 0; i < count; ++i) segments_out[i] = static_cast<int32_t>(segs[i]);
  return GMT_OK;
}

