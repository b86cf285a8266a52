// graph.cu -- build_neighbor_graph (graph.cpp:117-188) for the Euclidean
// model as device kernels writing compressed rows.
//
// The reference buckets positions on a uniform grid and then applies the
// exact predicate euclidean_distance(u, v) <= r to every surviving pair; its
// result is provably the brute-force double loop (graph.hpp:57-59,
// test_graph.cpp:102-124).  Here every (u, v) pair is tested directly:
//   * warp per source row u, 32 consecutive targets per step read from a
//     structure-of-arrays copy of the coordinates (coalesced, L1-shared by
//     the warps of a CTA);
//   * the squared distance is summed in the reference's axis order with
//     correctly rounded ops; pairs with sq > r^2 (1 + 1e-12) are rejected
//     without a sqrt (a safe bound: sqrt_rn(sq) <= r implies
//     sq < r^2 (1 + 2^-51)), the rest take __dsqrt_rn and the inclusive
//     `c <= r` test of graph.cpp:159;
//   * ballot + popc give each accepted target its slot, so rows come out
//     sorted by target with no sort (graph.cpp:163-166);
//   * pass 1 counts, an exclusive scan makes the row offsets, pass 2 fills.
// Euclidean in-lists are the out-lists bit for bit (graph.cpp:184-186;
// (a-b)^2 == (b-a)^2 exactly), so one CSR serves both directions.
#include <cuda_runtime.h>

#include <cstdint>

#include "common.cuh"
#include "internal.cuh"
#include "offline.cuh"

namespace gmtb {

namespace {

constexpr uint32_t kFull = 0xffffffffu;
constexpr int kMaxDim = 16;

__global__ void to_soa_kernel(const double* __restrict__ coords, int n, int d,
                              double* __restrict__ soa) {
  const int64_t total = static_cast<int64_t>(n) * d;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t v = i / d, k = i - v * d;
    soa[k * n + v] = coords[i];
  }
}

// One warp per source row.  FILL = false: counts[u] = |out[u]|;
// FILL = true: writes col/cost at row_ptr[u].
template <int D, bool FILL>
__global__ void __launch_bounds__(256) rdisk_kernel(const double* __restrict__ soa, int n, int d_rt,
                                                    double r, double r2_hi,
                                                    int64_t* __restrict__ counts,
                                                    const int64_t* __restrict__ row_ptr,
                                                    int32_t* __restrict__ col,
                                                    double* __restrict__ cost) {
  const int d = D > 0 ? D : d_rt;
  const int lane = threadIdx.x & 31;
  const int warps = (blockDim.x >> 5) * gridDim.x;
  for (int u = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); u < n; u += warps) {
    double a[D > 0 ? D : kMaxDim];
#pragma unroll
    for (int k = 0; k < (D > 0 ? D : kMaxDim); ++k) {
      if (D > 0 || k < d) a[k] = __ldg(soa + static_cast<int64_t>(k) * n + u);
    }
    int64_t out = FILL ? row_ptr[u] : 0;
    for (int base = 0; base < n; base += 32) {
      const int v = base + lane;
      bool keep = false;
      double c = 0.0;
      if (v < n && v != u) {
        double sq = 0.0;
#pragma unroll
        for (int k = 0; k < (D > 0 ? D : kMaxDim); ++k) {
          if (D > 0 || k < d) {
            const double t = __dsub_rn(a[k], __ldg(soa + static_cast<int64_t>(k) * n + v));
            sq = __dadd_rn(sq, __dmul_rn(t, t));
          }
        }
        if (sq <= r2_hi) {
          c = __dsqrt_rn(sq);
          keep = c <= r;
        }
      }
      const uint32_t m = __ballot_sync(kFull, keep);
      if (FILL && keep) {
        const int64_t slot = out + __popc(m & ((1u << lane) - 1u));
        col[slot] = v;
        cost[slot] = c;
      }
      out += __popc(m);
    }
    if (!FILL && lane == 0) counts[u] = out;
  }
}

// Exclusive scan of counts[0..n) into row_ptr[0..n] by one CTA.
__global__ void __launch_bounds__(1024) scan_kernel(const int64_t* __restrict__ counts, int n,
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
      warp_sum[lane] = w;  // inclusive over warps
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

template <int D>
cudaError_t launch_rdisk(bool fill, const double* soa, int n, int d, double r, double r2_hi,
                         int64_t* counts, const int64_t* row_ptr, int32_t* col, double* cost,
                         int sm_count, cudaStream_t s) {
  const int threads = 256;
  const int warps_per_block = threads / 32;
  int blocks = (n + warps_per_block - 1) / warps_per_block;
  const int cap = sm_count * 8;
  if (blocks > cap) blocks = cap;
  if (blocks < 1) blocks = 1;
  if (fill) {
    rdisk_kernel<D, true><<<blocks, threads, 0, s>>>(soa, n, d, r, r2_hi, counts, row_ptr, col, cost);
  } else {
    rdisk_kernel<D, false><<<blocks, threads, 0, s>>>(soa, n, d, r, r2_hi, counts, row_ptr, col, cost);
  }
  return cudaGetLastError();
}

cudaError_t launch_rdisk_any(bool fill, const double* soa, int n, int d, double r, double r2_hi,
                             int64_t* counts, const int64_t* row_ptr, int32_t* col, double* cost,
                             int sm_count, cudaStream_t s) {
  switch (d) {
    case 2: return launch_rdisk<2>(fill, soa, n, d, r, r2_hi, counts, row_ptr, col, cost, sm_count, s);
    case 3: return launch_rdisk<3>(fill, soa, n, d, r, r2_hi, counts, row_ptr, col, cost, sm_count, s);
    case 4: return launch_rdisk<4>(fill, soa, n, d, r, r2_hi, counts, row_ptr, col, cost, sm_count, s);
    case 6: return launch_rdisk<6>(fill, soa, n, d, r, r2_hi, counts, row_ptr, col, cost, sm_count, s);
    case 12: return launch_rdisk<12>(fill, soa, n, d, r, r2_hi, counts, row_ptr, col, cost, sm_count, s);
    default: return launch_rdisk<0>(fill, soa, n, d, r, r2_hi, counts, row_ptr, col, cost, sm_count, s);
  }
}

}  // namespace

#define GMT_CUDA(call)                                   \
  do {                                                   \
    cudaError_t _e = (call);                             \
    if (_e != cudaSuccess) return cuda_error(_e, #call); \
  } while (0)

int build_graph_dev(gmt_ctx* ctx, const double* d_coords, int n, int d, double radius,
                    Arena& out, int64_t* num_edges, int64_t** row_ptr, int32_t** col,
                    double** cost) {
  if (!(radius > 0.0)) return set_error(GMT_E_INVALID_INPUT, "connection radius must be positive");
  if (n < 1) return set_error(GMT_E_INVALID_INPUT, "cannot build a graph over zero samples");
  if (d > kMaxDim) return set_error(GMT_E_INVALID_INPUT, "dimension above 16 is not supported");
  cudaStream_t s = ctx->stream;
  // scratch: soa coords + counts
  const size_t soa_bytes = align16(sizeof(double) * static_cast<size_t>(n) * d);
  const size_t cnt_bytes = align16(sizeof(int64_t) * static_cast<size_t>(n));
  Arena tmp;
  int rc = tmp.reserve(soa_bytes + cnt_bytes);
  if (rc) return rc;
  double* soa = static_cast<double*>(tmp.ptr);
  int64_t* counts = reinterpret_cast<int64_t*>(static_cast<char*>(tmp.ptr) + soa_bytes);
  const double r2_hi = radius * radius * (1.0 + 1e-12);
  int blocks = static_cast<int>((static_cast<int64_t>(n) * d + 255) / 256);
  if (blocks > 4096) blocks = 4096;
  to_soa_kernel<<<blocks, 256, 0, s>>>(d_coords, n, d, soa);
  GMT_CUDA(cudaGetLastError());
  ++ctx->launches;
  GMT_CUDA(launch_rdisk_any(false, soa, n, d, radius, r2_hi, counts, nullptr, nullptr, nullptr,
                            ctx->sm_count, s));
  ++ctx->launches;
  // row_ptr lives in the output arena; edges follow once E is known.
  Arena rp;
  rc = rp.reserve(sizeof(int64_t) * (n + 1));
  if (rc) {
    tmp.release();
    return rc;
  }
  scan_kernel<<<1, 1024, 0, s>>>(counts, n, static_cast<int64_t*>(rp.ptr));
  GMT_CUDA(cudaGetLastError());
  ++ctx->launches;
  int64_t E = 0;
  GMT_CUDA(cudaMemcpyAsync(&E, static_cast<int64_t*>(rp.ptr) + n, sizeof(int64_t),
                           cudaMemcpyDeviceToHost, s));
  GMT_CUDA(cudaStreamSynchronize(s));
  const size_t o_rp = 0;
  const size_t o_col = align16(sizeof(int64_t) * (n + 1));
  const size_t o_cost = o_col + align16(sizeof(int32_t) * static_cast<size_t>(E));
  const size_t total = o_cost + align16(sizeof(double) * static_cast<size_t>(E));
  rc = out.reserve(total);
  if (rc) {
    tmp.release();
    rp.release();
    return rc;
  }
  char* base = static_cast<char*>(out.ptr);
  *row_ptr = reinterpret_cast<int64_t*>(base + o_rp);
  *col = reinterpret_cast<int32_t*>(base + o_col);
  *cost = reinterpret_cast<double*>(base + o_cost);
  GMT_CUDA(cudaMemcpyAsync(*row_ptr, rp.ptr, sizeof(int64_t) * (n + 1), cudaMemcpyDeviceToDevice, s));
  GMT_CUDA(launch_rdisk_any(true, soa, n, d, radius, r2_hi, nullptr, *row_ptr, *col, *cost,
                            ctx->sm_count, s));
  ++ctx->launches;
  GMT_CUDA(cudaStreamSynchronize(s));
  tmp.release();
  rp.release();
  *num_edges = E;
  return GMT_OK;
}

}  // namespace gmtb

using namespace gmtb;

extern "C" int gmt_build_neighbor_graph(gmt_ctx* ctx, const double* coords, int32_t n, int32_t dim,
                                        double radius, int64_t* num_edges, int64_t* out_ptr,
                                        int32_t* out_col, double* out_cost) {
  gmtb::AllocScope alloc_scope_(ctx);
  if (n < 1) return set_error(GMT_E_INVALID_INPUT, "cannot build a graph over zero samples");
  if (dim < 1) return set_error(GMT_E_INVALID_INPUT, "dimension must be >= 1");
  Arena in;
  int rc = in.reserve(sizeof(double) * static_cast<size_t>(n) * dim);
  if (rc) return rc;
  GMT_CUDA(cudaMemcpyAsync(in.ptr, coords, sizeof(double) * static_cast<size_t>(n) * dim,
                           cudaMemcpyHostToDevice, ctx->stream));
  Arena g;
  int64_t E = 0, *rp = nullptr;
  int32_t* col = nullptr;
  double* cost = nullptr;
  rc = build_graph_dev(ctx, static_cast<const double*>(in.ptr), n, dim, radius, g, &E, &rp, &col, &cost);
  in.release();
  if (rc) return rc;
  *num_edges = E;
  if (out_ptr) {
    GMT_CUDA(cudaMemcpyAsync(out_ptr, rp, sizeof(int64_t) * (n + 1), cudaMemcpyDeviceToHost, ctx->stream));
    if (E > 0) {
      GMT_CUDA(cudaMemcpyAsync(out_col, col, sizeof(int32_t) * E, cudaMemcpyDeviceToHost, ctx->stream));
      GMT_CUDA(cudaMemcpyAsync(out_cost, cost, sizeof(double) * E, cudaMemcpyDeviceToHost, ctx->stream));
    }
    GMT_CUDA(cudaStreamSynchronize(ctx->stream));
  }
  g.release();
  return GMT_OK;
}
