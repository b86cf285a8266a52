// pool.cu -- batched double-integrator queries over one shared Halton sample
// pool (SURVEY.md §8(e), configs[4]).
//
// With Halton sampling every query's sample set is the first n free points
// of the SAME stream (sample_free, sampling.cpp:97-108), and a kinodynamic
// edge depends only on the two states and the cost threshold r.  So every
// query's graph is the induced subgraph of one pool graph, re-indexed by the
// monotone rank of the free points, plus two per-query rows:
//   * the goal-substituted sample n-1 (sampling.cpp:115-141), when no free
//     sample falls in the goal box, and
//   * the appended init, vertex n (append_init, sampling.cpp:144-154).
// Both are the largest indices, so they end every sorted out- and in-row
// (graph.cpp:163-166, 184-186) they appear in.
//
// The pool (Halton points + the directed graph over the first K of them,
// built by the same kinodynamic builder as every single instance) lives in
// the context and is reused across calls; K is the largest "cutoff" (the
// stream position of a query's n-th free point) seen so far.  Per call, for
// Q queries:
//   pool_free_kernel     free flag of every (query, candidate point)    Q x Kc
//   pool_select_kernel   rank of every free point, the first n kept     block / query
//   (host: the pool graph covers every cutoff, else it is regrown)
//   pool_subst_kernel    goal substitution (the reference's search)     block / query
//   pool_init_kernel     append_init (exact-duplicate check)            block / query
//   pool_special_cand_kernel / pool_special_kernel
//                        out-/in-rows of the substituted goal and init   warp / row
//   pool_layout_kernel   row capacities (pool degree + 2) -> row starts  block / query
//   (host: row regions sized from the per-query totals)
//   pool_rows_kernel     every derived row: the pool row filtered by
//                        rank (ballot compaction) + the special entries  warp / row
//   pool_desc_kernel     the DevInstance of every query
// Rows are padded by the two special entries each; DevInstance::in_end /
// out_end carry the row ends.  The derived instances are bit-identical to
// gmt_instance_build of each problem (tests/test_gpu_pool.py); queries off
// the fast path (an exact init duplicate, a long substitution search, a
// special row above kSpecCap) take gmt_instance_build.
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstring>
#include <string>
#include <vector>

#include "common.cuh"
#include "di.cuh"
#include "gmt_b200.h"
#include "internal.cuh"
#include "offline.cuh"
#include "sample_dev.cuh"
#include "solve.cuh"

namespace gmtb {

int plan_smem(gmt_ctx* ctx, int max_n, int max_d, int max_nb, int cluster, size_t* smem, int* obs_in_smem,
              size_t* gstate = nullptr);
int assign_gstate(Arena& arena, std::vector<SolveJob>& jobs, size_t bytes);
int carve_results(Arena& arena, int count, const int64_t* node_off, bool tree, bool stats,
                  std::vector<DevResult>& out, ResultScalars** scalars_base, int64_t* counters);

struct SamplePool {
  uint64_t start_index = 1;
  gmt_di_params gp{};
  double radius = 0.0;
  int Kp = 0;        // Halton points generated (candidates)
  Arena pts;         // Kp x 6
  int K = 0;         // the pool graph covers points [0, K)
  Arena out_mem, in_mem;
  DiRows out, in;
  Arena rec_mem;     // per in-edge check records (pool_rec_kernel), empty when GMT_POOL_REC=0
  int rec_len = 0;
  double build_ms = 0.0;      // last graph (re)build
  int last_fallbacks = 0;     // queries of the last call that took the single builder
  double stage_ms[8] = {};    // last call's stage times (GMT_POOL_TIMING=1)
};

void destroy_pool(SamplePool* p) {
  if (!p) return;
  p->pts.release();
  p->out_mem.release();
  p->in_mem.release();
  p->rec_mem.release();
  delete p;
}

namespace {

constexpr uint32_t kFull = 0xffffffffu;
constexpr int kD = kDiDim;
constexpr uint16_t kNoRank = 0xffffu;
constexpr int kSpecCap = 1024;   // entries of one special row (larger: the single builder)
constexpr int kCandCap = 4096;   // prefilter survivors of one special row (larger: the single builder)
constexpr int kSubstSearch = 1024;

#define GMT_CUDA(call)                                   \
  do {                                                   \
    cudaError_t _e = (call);                             \
    if (_e != cudaSuccess) return cuda_error(_e, #call); \
  } while (0)

struct Primes {
  uint32_t p[kD];
};

// Sequential carving of one allocation into 16-byte aligned sections.
struct Carver {
  size_t off = 0;
  template <typename T>
  size_t take(size_t count) {
    const size_t o = off;
    off = align16(off + sizeof(T) * count);
    return o;
  }
};

// Per-query parameters (host -> device) and outcome (device -> host).
struct PQ {
  int32_t n;
  int32_t nb;
  int32_t skip;  // not on the pool path: the single builder
  int32_t reserved;
  int64_t box_off;   // first box (rows of kD doubles)
  int64_t node_off;  // first node entry (n + 1 reserved)
  int64_t in_off;    // first slot of the query's in-row region
  int64_t out_off;   // first slot of the query's out-row region
};
struct PQOut {
  int32_t fallback;
  int32_t subst;
  int32_t goal_any;
  int32_t cutoff;       // stream position after the query's n-th free point
  int32_t spec_len[4];  // out(g), in(g), out(init), in(init)
  int64_t tot_in;       // row-region sizes (layout)
  int64_t tot_out;
};

__device__ __forceinline__ bool free_pt(const double* p, const double* lo, const double* hi, int nb) {
  if (!point_in_cube(p, kD)) return false;  // point_free (space.cpp:47-54)
  for (int b = 0; b < nb; ++b)
    if (box_contains(lo + b * kD, hi + b * kD, kD, p)) return false;
  return true;
}

// halton_point(start + p, 6) (sampling.cpp:46-51) for p in [from, to).
__global__ void pool_points_kernel(int from, int to, uint64_t start, Primes pr, double* __restrict__ out) {
  for (int i = from * kD + blockIdx.x * blockDim.x + threadIdx.x; i < to * kD; i += gridDim.x * blockDim.x) {
    const int p = i / kD, k = i - p * kD;
    out[i] = halton_dev(start + static_cast<uint64_t>(p), pr.p[k]);
  }
}

// flags[q][p] = point_free(candidate p, boxes of q); the query's boxes are
// staged in shared memory when they fit.
// (boxes <= kFreeSortMax: staged in ascending lo_x with the widest x
// extent w, so a point only tests the boxes whose lo_x lies in
// [x - w', x] (w' = w rounded up: every box containing the point is among
// them; Aabb::contains is exact and point_free's outcome does not depend on
// the box order).  Each block covers kFreePts points of one query.)
constexpr int kFreeSortMax = 256;
constexpr int kFreePts = 2048;
__global__ void __launch_bounds__(256) pool_free_kernel(const PQ* __restrict__ pq, const double* __restrict__ P,
                                                        int K, const double* __restrict__ box_lo,
                                                        const double* __restrict__ box_hi, int stage_cap,
                                                        uint8_t* __restrict__ flags) {
  extern __shared__ double bsm[];
  __shared__ unsigned long long wbits;
  const int q = blockIdx.y;
  const PQ Q = pq[q];
  if (Q.skip) return;
  const double* lo = box_lo + Q.box_off * kD;
  const double* hi = box_hi + Q.box_off * kD;
  const int nb = Q.nb;
  const int p0 = blockIdx.x * kFreePts;
  if (nb <= stage_cap && nb <= kFreeSortMax) {
    if (threadIdx.x == 0) wbits = 0ull;
    __syncthreads();
    for (int b = threadIdx.x; b < nb; b += blockDim.x) {
      const double x = lo[b * kD];
      int r = 0;
      for (int c = 0; c < nb; ++c) {
        const double y = lo[c * kD];
        r += (y < x || (y == x && c < b)) ? 1 : 0;
      }
      for (int k = 0; k < kD; ++k) {
        bsm[r * kD + k] = lo[b * kD + k];
        bsm[(nb + r) * kD + k] = hi[b * kD + k];
      }
      const double w = hi[b * kD] - x;
      if (w > 0.0) atomicMax(&wbits, static_cast<unsigned long long>(__double_as_longlong(w)));
    }
    __syncthreads();
    const double* slo = bsm;
    const double* shi = bsm + nb * kD;
    const double wx = __longlong_as_double(static_cast<long long>(wbits)) * (1.0 + 1e-12) + 1e-12;
    for (int p = p0 + threadIdx.x; p < K && p < p0 + kFreePts; p += blockDim.x) {
      double x[kD];
#pragma unroll
      for (int k = 0; k < kD; ++k) x[k] = __ldg(P + static_cast<int64_t>(p) * kD + k);
      bool free = point_in_cube(x, kD);
      if (free) {
        // first box with lo_x >= x - wx (binary search), then every box up
        // to lo_x > x
        const double t = x[0] - wx;
        int l = 0, h = nb;
        while (l < h) {
          const int m = (l + h) >> 1;
          if (slo[m * kD] < t) l = m + 1; else h = m;
        }
        for (int b = l; b < nb && !(slo[b * kD] > x[0]); ++b)
          if (box_contains(slo + b * kD, shi + b * kD, kD, x)) {
            free = false;
            break;
          }
      }
      flags[static_cast<int64_t>(q) * K + p] = free ? 1 : 0;
    }
    return;
  }
  if (nb <= stage_cap) {
    for (int i = threadIdx.x; i < nb * kD; i += blockDim.x) {
      bsm[i] = lo[i];
      bsm[nb * kD + i] = hi[i];
    }
    __syncthreads();
    // (the staged copy named directly: shared-space loads, not generic)
    for (int p = p0 + threadIdx.x; p < K && p < p0 + kFreePts; p += blockDim.x) {
      double x[kD];
#pragma unroll
      for (int k = 0; k < kD; ++k) x[k] = __ldg(P + static_cast<int64_t>(p) * kD + k);
      flags[static_cast<int64_t>(q) * K + p] = free_pt(x, bsm, bsm + nb * kD, nb) ? 1 : 0;
    }
    return;
  }
  for (int p = p0 + threadIdx.x; p < K && p < p0 + kFreePts; p += blockDim.x) {
    double x[kD];
#pragma unroll
    for (int k = 0; k < kD; ++k) x[k] = __ldg(P + static_cast<int64_t>(p) * kD + k);
    flags[static_cast<int64_t>(q) * K + p] = free_pt(x, lo, hi, nb) ? 1 : 0;
  }
}

// The first n free candidates in stream order are the query's samples
// 0..n-1 (sample_free's loop, sampling.cpp:97-108): ranks by a block scan.
__global__ void __launch_bounds__(1024) pool_select_kernel(const PQ* __restrict__ pq, const double* __restrict__ P,
                                                           int K, const uint8_t* __restrict__ flags,
                                                           const double* __restrict__ goal_lo,
                                                           const double* __restrict__ goal_hi,
                                                           uint16_t* __restrict__ rank_of, int32_t* __restrict__ sel,
                                                           double* __restrict__ qcoords, PQOut* __restrict__ out) {
  __shared__ int warp_sum[32];
  __shared__ int carry_s;
  const int q = blockIdx.x;
  const PQ Q = pq[q];
  if (Q.skip) return;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const double* glo = goal_lo + static_cast<int64_t>(q) * kD;
  const double* ghi = goal_hi + static_cast<int64_t>(q) * kD;
  if (tid == 0) carry_s = 0;
  __syncthreads();
  bool in_goal = false;
  for (int base = 0; base < K; base += blockDim.x) {
    const int p = base + tid;
    const int f = (p < K && flags[static_cast<int64_t>(q) * K + p]) ? 1 : 0;
    const uint32_t m = __ballot_sync(kFull, f);
    if (lane == 0) warp_sum[warp] = __popc(m);
    __syncthreads();
    if (warp == 0) {
      int w = lane < static_cast<int>(blockDim.x >> 5) ? warp_sum[lane] : 0;
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(kFull, w, o);
        if (lane >= o) w += y;
      }
      warp_sum[lane] = w;  // inclusive
    }
    __syncthreads();
    const int carry = carry_s;
    const int rank = carry + (warp > 0 ? warp_sum[warp - 1] : 0) + __popc(m & ((1u << lane) - 1u));
    const bool keep = f && rank < Q.n;
    if (p < K) rank_of[static_cast<int64_t>(q) * K + p] = keep ? static_cast<uint16_t>(rank) : kNoRank;
    if (keep) {
      sel[Q.node_off + rank] = p;
      double* c = qcoords + (Q.node_off + rank) * kD;
#pragma unroll
      for (int k = 0; k < kD; ++k) c[k] = P[static_cast<int64_t>(p) * kD + k];
      in_goal = in_goal || box_contains(glo, ghi, kD, c);  // goal.contains (sampling.cpp:110-112)
    }
    __syncthreads();
    if (tid == blockDim.x - 1) carry_s = carry + warp_sum[(blockDim.x >> 5) - 1];
    __syncthreads();
  }
  const int any = __syncthreads_or(in_goal ? 1 : 0);
  if (tid == 0) {
    PQOut o{};
    o.fallback = carry_s < Q.n ? 1 : 0;  // fewer than n free candidates (the host widens them)
    o.goal_any = any;
    o.cutoff = carry_s < Q.n ? K + 1 : sel[Q.node_off + Q.n - 1] + 1;
    out[q] = o;
  }
}

// Goal substitution (sampling.cpp:115-141): the first of the goal centre and
// the goal-box Halton points that is free and no exact duplicate of samples
// 0 .. n-2 replaces sample n-1 (whose pool point leaves the query).
__global__ void __launch_bounds__(256) pool_subst_kernel(const PQ* __restrict__ pq, int K,
                                                         const double* __restrict__ box_lo,
                                                         const double* __restrict__ box_hi,
                                                         const double* __restrict__ goal_lo,
                                                         const double* __restrict__ goal_hi, Primes pr,
                                                         uint16_t* __restrict__ rank_of, const int32_t* __restrict__ sel,
                                                         double* __restrict__ qcoords, PQOut* __restrict__ out) {
  __shared__ int best, dup;
  const int q = blockIdx.x;
  const PQ Q = pq[q];
  if (Q.skip || out[q].fallback || out[q].goal_any) return;
  const double* glo = goal_lo + static_cast<int64_t>(q) * kD;
  const double* ghi = goal_hi + static_cast<int64_t>(q) * kD;
  const double* lo = box_lo + Q.box_off * kD;
  const double* hi = box_hi + Q.box_off * kD;
  auto candidate = [&](int i, double* c) {
    if (i == 0) {  // Aabb::center (space.cpp:18-22)
      for (int k = 0; k < kD; ++k) c[k] = __dmul_rn(0.5, __dadd_rn(glo[k], ghi[k]));
    } else {  // lo + q * (hi - lo) (sampling.cpp:122-124)
      for (int k = 0; k < kD; ++k)
        c[k] = __dadd_rn(glo[k], __dmul_rn(halton_dev(static_cast<uint64_t>(i), pr.p[k]), __dsub_rn(ghi[k], glo[k])));
    }
  };
  int last = -1, found = -1;
  for (;;) {
    if (threadIdx.x == 0) {
      best = 0x7fffffff;
      dup = 0;
    }
    __syncthreads();
    // the smallest free candidate index above `last`: ascending chunks of
    // blockDim, stopping at the first chunk that holds one (usually the
    // goal's centre, i = 0)
    for (int base = last + 1; base < kSubstSearch; base += blockDim.x) {
      const int i = base + static_cast<int>(threadIdx.x);
      if (i < kSubstSearch) {
        double c[kD];
        candidate(i, c);
        if (free_pt(c, lo, hi, Q.nb)) atomicMin(&best, i);
      }
      __syncthreads();
      const bool done = best != 0x7fffffff;
      __syncthreads();  // (every thread has read best before the next chunk's atomicMin)
      if (done) break;
    }
    const int b = best;
    if (b == 0x7fffffff) break;
    double c[kD];
    candidate(b, c);
    for (int j = threadIdx.x; j < Q.n - 1; j += blockDim.x) {
      const double* s = qcoords + (Q.node_off + j) * kD;
      bool eq = true;
      for (int k = 0; k < kD; ++k) eq = eq && c[k] == s[k];
      if (eq) dup = 1;
    }
    __syncthreads();
    const int was_dup = dup;
    __syncthreads();
    if (!was_dup) {
      found = b;
      break;
    }
    last = b;
  }
  if (threadIdx.x == 0) {
    if (found < 0) {
      out[q].fallback = 1;  // a longer search: the single builder
    } else {
      candidate(found, qcoords + (Q.node_off + Q.n - 1) * kD);
      rank_of[static_cast<int64_t>(q) * K + sel[Q.node_off + Q.n - 1]] = kNoRank;
      out[q].subst = 1;
      out[q].goal_any = 1;
    }
  }
}

// append_init (sampling.cpp:144-154): an exact duplicate takes the single
// builder (it would reuse the sample's index); else the init is vertex n.
__global__ void __launch_bounds__(256) pool_init_kernel(const PQ* __restrict__ pq, const double* __restrict__ inits,
                                                        double* __restrict__ qcoords, PQOut* __restrict__ out) {
  __shared__ int dup;
  const int q = blockIdx.x;
  const PQ Q = pq[q];
  if (Q.skip || out[q].fallback) return;
  const double* init = inits + static_cast<int64_t>(q) * kD;
  if (threadIdx.x == 0) dup = 0;
  __syncthreads();
  for (int i = threadIdx.x; i < Q.n; i += blockDim.x) {
    const double* c = qcoords + (Q.node_off + i) * kD;
    bool eq = true;
    for (int k = 0; k < kD; ++k) eq = eq && c[k] == init[k];
    if (eq) dup = 1;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    if (dup) {
      out[q].fallback = 1;
    } else {
      for (int k = 0; k < kD; ++k) qcoords[(Q.node_off + Q.n) * kD + k] = init[k];
    }
  }
}

// The rows of the per-query vertices (list l: 0 out(g), 1 in(g), 2 out(init),
// 3 in(init); g = n-1 when substituted, init = n): every other vertex x
// with cost(s -> x) (or cost(x -> s)) <= r, ascending x -- kino_rows_kernel's
// predicate and order (di_graph.cu).  Two kernels: the exact-safe prefilters
// (few registers, many warps) compact the surviving columns in order, then
// the capped 2BVP solve runs lane-parallel over the survivors only.
// (One warp per special vertex testing both directions from one pass over
// the coordinates measured slower: 2.43 -> 2.89 ms per 4096 queries -- half
// the warps, and the two cost tests serialised.)
__global__ void __launch_bounds__(256) pool_special_cand_kernel(const PQ* __restrict__ pq, DiParams P, double bound,
                                                                double radius, const double* __restrict__ qcoords,
                                                                int32_t* __restrict__ cand, PQOut* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  const int gw = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);  // (query, list)
  const int q = gw >> 2, l = gw & 3;
  const PQ Q = pq[q];
  if (Q.skip || out[q].fallback) return;
  if (l < 2 && !out[q].subst) return;
  const int V = Q.n + 1;
  const int s = l < 2 ? Q.n - 1 : Q.n;
  const bool outgoing = (l & 1) == 0;
  const double* base = qcoords + Q.node_off * kD;
  double xs[kD];
#pragma unroll
  for (int k = 0; k < kD; ++k) xs[k] = base[static_cast<int64_t>(s) * kD + k];
  int32_t* cl = cand + (static_cast<int64_t>(q) * 4 + l) * kCandCap;
  // Two passes, so the rare pairs that need di_cost_exceeds' 12 parts do not
  // stall a whole warp iteration each (~6 % of the pairs at r = 1.6, i.e.
  // most 32-pair iterations hold one): (1) the position prefilter and the
  // whole-interval bound, the undecided columns compacted in order into cl;
  // (2) the parts over that dense list, compacted in place (write index <=
  // read index).  Same list as di_cost_exceeds per pair.
  int len = 0;
  for (int b0 = 0; b0 < V; b0 += 32) {
    const int x = b0 + lane;
    bool may = x < V && x != s;
    if (may) {
      double xx[kD];
#pragma unroll
      for (int k = 0; k < kD; ++k) xx[k] = base[static_cast<int64_t>(x) * kD + k];
      const double* from = outgoing ? xs : xx;
      const double* to = outgoing ? xx : xs;
      for (int k = 0; k < 3; ++k) {  // di_may_connect (di_graph.cu)
        const double D = to[k] - from[k];
        if (D > bound || -D > bound) may = false;
      }
      if (may) may = !di_cost_exceeds_whole(di_coef(from, to, P), radius);
    }
    const uint32_t m = __ballot_sync(kFull, may);
    const int slot = len + __popc(m & ((1u << lane) - 1u));
    if (may && slot < kCandCap) cl[slot] = x;
    len += __popc(m);
  }
  if (len <= kCandCap) {
    __syncwarp();
    const int undecided = len;
    len = 0;
    for (int b0 = 0; b0 < undecided; b0 += 32) {
      const int j = b0 + lane;
      const int x = j < undecided ? cl[j] : 0;
      bool may = j < undecided;
      if (may) {
        double xx[kD];
#pragma unroll
        for (int k = 0; k < kD; ++k) xx[k] = base[static_cast<int64_t>(x) * kD + k];
        may = !di_cost_exceeds_parts(outgoing ? di_coef(xs, xx, P) : di_coef(xx, xs, P), radius);
      }
      const uint32_t m = __ballot_sync(kFull, may);  // (every lane has read its entry)
      const int slot = len + __popc(m & ((1u << lane) - 1u));
      if (may) cl[slot] = x;
      len += __popc(m);
      __syncwarp();
    }
  }
  if (lane == 0) {
    out[q].spec_len[l] = len;  // (candidates here; the solve kernel overwrites it)
    if (len > kCandCap) out[q].fallback = 1;
  }
}

__global__ void __launch_bounds__(128) pool_special_kernel(const PQ* __restrict__ pq, DiParams P, double radius,
                                                           const double* __restrict__ qcoords,
                                                           const int32_t* __restrict__ cand,
                                                           int32_t* __restrict__ scol, double* __restrict__ scost,
                                                           double* __restrict__ stau, int32_t* __restrict__ sp_code,
                                                           uint16_t* __restrict__ sp_j, PQOut* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  const int gw = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int q = gw >> 2, l = gw & 3;
  const PQ Q = pq[q];
  if (Q.skip || out[q].fallback) return;
  if (l < 2 && !out[q].subst) return;
  const int s = l < 2 ? Q.n - 1 : Q.n;
  const bool outgoing = (l & 1) == 0;
  const double* base = qcoords + Q.node_off * kD;
  double xs[kD];
#pragma unroll
  for (int k = 0; k < kD; ++k) xs[k] = base[static_cast<int64_t>(s) * kD + k];
  const int32_t* cl = cand + (static_cast<int64_t>(q) * 4 + l) * kCandCap;
  const int nc = out[q].spec_len[l];
  const int64_t lb = (static_cast<int64_t>(q) * 4 + l) * kSpecCap;
  int len = 0;
  for (int b0 = 0; b0 < nc; b0 += 32) {
    const int j = b0 + lane;
    bool keep = false;
    double c = 0.0, t = 0.0;
    int x = 0;
    if (j < nc) {
      x = cl[j];
      double xx[kD];
#pragma unroll
      for (int k = 0; k < kD; ++k) xx[k] = base[static_cast<int64_t>(x) * kD + k];
      c = outgoing ? di_cost_tau(xs, xx, P, &t, radius) : di_cost_tau(xx, xs, P, &t, radius);
      keep = c <= radius;
    }
    const uint32_t m = __ballot_sync(kFull, keep);
    const int slot = len + __popc(m & ((1u << lane) - 1u));
    if (keep && slot < kSpecCap) {
      scol[lb + slot] = x;
      scost[lb + slot] = c;
      stau[lb + slot] = t;
      // per-vertex lookup for the rows kernel: bit l, and the entry of the
      // edges the vertex's in-row takes from g (l = 0) or init (l = 2)
      atomicOr(sp_code + Q.node_off + x, 1 << l);
      if (l == 0) sp_j[2 * (Q.node_off + x)] = static_cast<uint16_t>(slot);
      if (l == 2) sp_j[2 * (Q.node_off + x) + 1] = static_cast<uint16_t>(slot);
    }
    len += __popc(m);
  }
  __syncwarp();
  if (lane == 0) {
    out[q].spec_len[l] = len;
    if (len > kSpecCap) out[q].fallback = 1;
  }
}

// Row starts (relative to the query's regions): vertex x < n owns its pool
// point's degree + 2 slots (room for the two special entries), in rank
// order; the special rows follow (kSpecCap slots each).  A substituted
// vertex n-1 keeps its dropped pool point's (unused) slots.
__global__ void __launch_bounds__(1024) pool_layout_kernel(const PQ* __restrict__ pq, const int64_t* __restrict__ pin_ptr,
                                                           const int64_t* __restrict__ pout_ptr,
                                                           const int32_t* __restrict__ sel, int64_t* __restrict__ in_start,
                                                           int64_t* __restrict__ out_start, PQOut* __restrict__ out) {
  __shared__ int64_t ws_in[32], ws_out[32];
  __shared__ int64_t carry_in, carry_out;
  const int q = blockIdx.x;
  const PQ Q = pq[q];
  if (Q.skip || out[q].fallback) return;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
  if (tid == 0) {
    carry_in = 0;
    carry_out = 0;
  }
  __syncthreads();
  for (int base = 0; base < Q.n; base += blockDim.x) {
    const int x = base + tid;
    int64_t ci = 0, co = 0;
    if (x < Q.n) {
      const int p = sel[Q.node_off + x];
      ci = pin_ptr[p + 1] - pin_ptr[p] + 2;
      co = pout_ptr[p + 1] - pout_ptr[p] + 2;
    }
    int64_t si = ci, so = co;  // inclusive warp scans
    for (int o = 1; o < 32; o <<= 1) {
      const int64_t a = __shfl_up_sync(kFull, si, o), b = __shfl_up_sync(kFull, so, o);
      if (lane >= o) {
        si += a;
        so += b;
      }
    }
    if (lane == 31) {
      ws_in[warp] = si;
      ws_out[warp] = so;
    }
    __syncthreads();
    if (warp == 0) {
      int64_t a = lane < nw ? ws_in[lane] : 0, b = lane < nw ? ws_out[lane] : 0;
      for (int o = 1; o < 32; o <<= 1) {
        const int64_t ya = __shfl_up_sync(kFull, a, o), yb = __shfl_up_sync(kFull, b, o);
        if (lane >= o) {
          a += ya;
          b += yb;
        }
      }
      ws_in[lane] = a;
      ws_out[lane] = b;
    }
    __syncthreads();
    const int64_t bi = carry_in + (warp > 0 ? ws_in[warp - 1] : 0) + si - ci;
    const int64_t bo = carry_out + (warp > 0 ? ws_out[warp - 1] : 0) + so - co;
    if (x < Q.n) {
      in_start[Q.node_off + x] = bi;
      out_start[Q.node_off + x] = bo;
    }
    __syncthreads();
    if (tid == 0) {
      carry_in += ws_in[nw - 1];
      carry_out += ws_out[nw - 1];
    }
    __syncthreads();
  }
  if (tid == 0) {
    const PQOut& o = out[q];
    if (o.subst) {
      in_start[Q.node_off + Q.n - 1] = carry_in;
      out_start[Q.node_off + Q.n - 1] = carry_out;
    }
    in_start[Q.node_off + Q.n] = carry_in + kSpecCap;
    out_start[Q.node_off + Q.n] = carry_out + kSpecCap;
    out[q].tot_in = carry_in + 2 * kSpecCap;
    out[q].tot_out = carry_out + 2 * kSpecCap;
  }
}

// Every derived row: an 8-lane group per (query, vertex), four vertices per
// warp (their dependent load chains overlap).  A pool vertex's rows are its
// pool rows with non-member entries dropped (ballot compaction keeps their
// ascending order, ranks being monotone) and member sources/targets mapped to
// ranks, then the special vertices (n-1 before n) where the special rows hold
// the edge (sp_code / sp_j).  A special vertex copies its own rows.  The
// outputs are written with streaming stores: they are read by the solve,
// not here, and must not evict the pool graph from L2.
constexpr int kRowTile = 512;  // vertices per block
template <typename T>
__device__ __forceinline__ void row_store(T* p, T v, bool stream) {
  if (stream) {
    __stcs(p, v);
  } else {
    *p = v;
  }
}
// Check records of the pool's in-edges (common.cuh pool_rec_len), a warp per
// pool vertex x, a lane per in-edge y -> x: the waypoints are di_coord's,
// the very values of the cached polyline the reference's planner checks
// (graph.cpp edge_path; oracle_di_paths), and of the solve's own table.
__global__ void __launch_bounds__(256) pool_rec_kernel(const double* __restrict__ P, int K,
                                                       const int64_t* __restrict__ in_ptr,
                                                       const int32_t* __restrict__ in_col,
                                                       const double* __restrict__ in_tau, DiParams DP, int RL,
                                                       double* __restrict__ rec) {
  const int lane = threadIdx.x & 31;
  const int x = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (x >= K) return;
  const int M = DP.segments;
  const int64_t e1 = in_ptr[x + 1];
  const double* x1 = P + static_cast<int64_t>(x) * kD;
  for (int64_t e = in_ptr[x] + lane; e < e1; e += 32) {
    const double* x0 = P + static_cast<int64_t>(in_col[e]) * kD;
    const double tau = in_tau[e];
    double* r = rec + e * RL;
    double mn[3] = {kInf, kInf, kInf}, mx[3] = {-kInf, -kInf, -kInf};
    bool incube = true;
    for (int k = 0; k <= M; ++k) {
      for (int i = 0; i < kD; ++i) {
        const double v = di_coord(x0, x1, tau, k, i, DP);
        incube = incube && !(v < 0.0 || v > 1.0);
        if (i < 3) {
          r[kPoolRecHead + 3 * k + i] = v;
          mn[i] = v < mn[i] ? v : mn[i];
          mx[i] = mx[i] < v ? v : mx[i];
        }
      }
    }
    for (int i = 0; i < 3; ++i) {
      r[i] = mn[i];
      r[3 + i] = mx[i];
    }
    if (!incube) r[0] = __longlong_as_double(0x7ff8000000000000LL);  // NaN: the polyline leaves the cube
    for (int j = kPoolRecHead + 3 * (M + 1); j < RL; ++j) r[j] = 0.0;
  }
}

template <int kRowLanes, bool kStream>

__global__ void __launch_bounds__(256) pool_rows_kernel(
    const PQ* __restrict__ pq, const PQOut* __restrict__ po, int Kc, int stage_rank, const int64_t* __restrict__ pin_ptr,
    const int32_t* __restrict__ pin_col, const double* __restrict__ pin_cost, const double* __restrict__ pin_tau,
    const int64_t* __restrict__ pout_ptr, const int32_t* __restrict__ pout_col, const uint16_t* __restrict__ rank_of,
    const int32_t* __restrict__ sel, const int32_t* __restrict__ scol, const double* __restrict__ scost,
    const double* __restrict__ stau, const int32_t* __restrict__ sp_code, const uint16_t* __restrict__ sp_j,
    const int64_t* __restrict__ in_start, int64_t* __restrict__ in_end,
    const int64_t* __restrict__ out_start, int64_t* __restrict__ out_end, int32_t* __restrict__ in_col,
    double* __restrict__ in_cost, double* __restrict__ in_tau, int32_t* __restrict__ out_col,
    int32_t* __restrict__ in_pe) {
  extern __shared__ uint16_t rank_s[];
  const int q = blockIdx.y;
  const PQ Q = pq[q];
  if (Q.skip || po[q].fallback) return;
  // The query's rank map in shared memory (the in-/out-row gathers hit it
  // once per pool edge); the block then walks kRowTile of its vertices.
  const uint16_t* rk = rank_of + static_cast<int64_t>(q) * Kc;
  if (stage_rank) {
    for (int i = threadIdx.x; i < Kc; i += blockDim.x) rank_s[i] = rk[i];
    __syncthreads();
    rk = rank_s;
  }
  const int lane = threadIdx.x & 31;
  const int grp = lane / kRowLanes, gl = lane % kRowLanes;
  const uint32_t gshift = static_cast<uint32_t>(grp * kRowLanes);
  const int n = Q.n;
  const int rows_per_pass = (blockDim.x >> 5) * (32 / kRowLanes);
  for (int x0 = blockIdx.x * kRowTile; x0 < blockIdx.x * kRowTile + kRowTile && x0 <= n; x0 += rows_per_pass) {
  const int x = x0 + (threadIdx.x >> 5) * (32 / kRowLanes) + grp;
  const bool subst = po[q].subst != 0;
  int32_t* icol = in_col + Q.in_off;
  double* icost = in_cost + Q.in_off;
  double* itau = in_tau + Q.in_off;
  int32_t* ipe = in_pe ? in_pe + Q.in_off : nullptr;
  int32_t* ocol = out_col + Q.out_off;
  const int64_t lb = static_cast<int64_t>(q) * 4 * kSpecCap;
  const bool live = x <= n;
  const bool special = live && (x == n || (subst && x == n - 1));
  int64_t is = 0, os = 0, ie0 = 0, oe0 = 0;
  int li = 0, lo = 0, code = 0;
  if (live) {
    is = in_start[Q.node_off + x];
    os = out_start[Q.node_off + x];
    if (special) {
      const int l = x == n ? 2 : 0;
      li = po[q].spec_len[l + 1];
      lo = po[q].spec_len[l];
    } else {
      const int p = sel[Q.node_off + x];
      ie0 = pin_ptr[p];
      li = static_cast<int>(pin_ptr[p + 1] - ie0);
      oe0 = pout_ptr[p];
      lo = static_cast<int>(pout_ptr[p + 1] - oe0);
      code = sp_code[Q.node_off + x];
    }
  }
  if (special) {  // (the group copies the special row; group-uniform branch)
    const int l = x == n ? 2 : 0;
    for (int j = gl; j < li; j += kRowLanes) {
      row_store(icol + is + j, scol[lb + (l + 1) * kSpecCap + j], kStream);
      row_store(icost + is + j, scost[lb + (l + 1) * kSpecCap + j], kStream);
      row_store(itau + is + j, stau[lb + (l + 1) * kSpecCap + j], kStream);
      if (ipe) row_store(ipe + is + j, -1, kStream);
    }
    for (int j = gl; j < lo; j += kRowLanes) row_store(ocol + os + j, scol[lb + l * kSpecCap + j], kStream);
    li = lo = 0;  // (no pool rows to scan)
    if (gl == 0) {
      const int l2 = x == n ? 2 : 0;
      row_store(in_end + Q.node_off + x, is + po[q].spec_len[l2 + 1], kStream);
      row_store(out_end + Q.node_off + x, os + po[q].spec_len[l2], kStream);
    }
  }
  int lmax = li > lo ? li : lo;
  for (int o = kRowLanes; o < 32; o <<= 1) {  // the longest row of the warp
    const int t = __shfl_xor_sync(kFull, lmax, o);
    lmax = t > lmax ? t : lmax;
  }
  int wi = 0, wo = 0;
  const uint32_t below = (1u << gl) - 1u;
  for (int b0 = 0; b0 < lmax; b0 += kRowLanes) {
    const int j = b0 + gl;
    const int32_t ycol = j < li ? __ldg(pin_col + ie0 + j) : -1;
    const int32_t vcol = j < lo ? __ldg(pout_col + oe0 + j) : -1;
    // (pool points past the scan, y >= Kc, are no query's vertices: a pool
    // graph built for larger queries is longer than a later call's rank maps)
    const uint16_t ri = ycol >= 0 && ycol < Kc ? rk[ycol] : kNoRank;
    const uint16_t ro = vcol >= 0 && vcol < Kc ? rk[vcol] : kNoRank;
    constexpr uint32_t kGroupMask = kRowLanes == 32 ? 0xffffffffu : ((1u << kRowLanes) - 1u);
    const uint32_t mi = (__ballot_sync(kFull, ri != kNoRank) >> gshift) & kGroupMask;
    const uint32_t mo = (__ballot_sync(kFull, ro != kNoRank) >> gshift) & kGroupMask;
    if (ri != kNoRank) {
      const int64_t slot = is + wi + __popc(mi & below);
      row_store(icol + slot, static_cast<int32_t>(ri), kStream);
      row_store(icost + slot, __ldg(pin_cost + ie0 + j), kStream);
      row_store(itau + slot, __ldg(pin_tau + ie0 + j), kStream);
      if (ipe) row_store(ipe + slot, static_cast<int32_t>(ie0 + j), kStream);
    }
    if (ro != kNoRank) row_store(ocol + os + wo + __popc(mo & below), static_cast<int32_t>(ro), kStream);
    wi += __popc(mi);
    wo += __popc(mo);
  }
  if (live && !special && gl == 0) {
    int64_t w = is + wi;
    if (subst && (code & 1)) {  // g -> x (list 0), then init -> x (list 2)
      const int j = sp_j[2 * (Q.node_off + x)];
      row_store(icol + w, n - 1, kStream);
      row_store(icost + w, scost[lb + j], kStream);
      row_store(itau + w, stau[lb + j], kStream);
      if (ipe) row_store(ipe + w, -1, kStream);
      ++w;
    }
    if (code & 4) {
      const int j = sp_j[2 * (Q.node_off + x) + 1];
      row_store(icol + w, n, kStream);
      row_store(icost + w, scost[lb + 2 * kSpecCap + j], kStream);
      row_store(itau + w, stau[lb + 2 * kSpecCap + j], kStream);
      if (ipe) row_store(ipe + w, -1, kStream);
      ++w;
    }
    row_store(in_end + Q.node_off + x, w, kStream);
    int64_t v = os + wo;
    if (subst && (code & 2)) row_store(ocol + v++, n - 1, kStream);  // x -> g (list 1), then x -> init (list 3)
    if (code & 8) row_store(ocol + v++, n, kStream);
    row_store(out_end + Q.node_off + x, v, kStream);
  }
  }
}

__global__ void pool_desc_kernel(const PQ* __restrict__ pq, const PQOut* __restrict__ po, int count, double radius,
                                 DiParams P, const double* __restrict__ qcoords, const double* __restrict__ box_lo,
                                 const double* __restrict__ box_hi, const double* __restrict__ goal_lo,
                                 const double* __restrict__ goal_hi, const int64_t* __restrict__ in_start,
                                 const int64_t* __restrict__ in_end, const int64_t* __restrict__ out_start,
                                 const int64_t* __restrict__ out_end, const int32_t* __restrict__ in_col,
                                 const double* __restrict__ in_cost, const double* __restrict__ in_tau,
                                 const int32_t* __restrict__ out_col, DevInstance* __restrict__ descs,
                                 PoolView* __restrict__ views, PoolView shared_view, const int32_t* __restrict__ sel,
                                 const uint16_t* __restrict__ rank, const int32_t* __restrict__ sp_code,
                                 const uint16_t* __restrict__ sp_j, const int32_t* __restrict__ scol,
                                 const double* __restrict__ scost, const double* __restrict__ stau,
                                 const int32_t* __restrict__ in_pe, const double* __restrict__ prec, int prec_len) {
  const int q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= count) return;
  const PQ Q = pq[q];
  if (Q.skip || po[q].fallback) return;
  DevInstance D{};
  if (views) {  // the graph as a view of the pool (the default: no rows are materialised)
    PoolView v = shared_view;
    v.sel = sel + Q.node_off;
    v.rank = rank + static_cast<int64_t>(q) * shared_view.kc;
    v.code = sp_code + Q.node_off;
    v.spj = sp_j + 2 * Q.node_off;
    v.scol = scol + static_cast<int64_t>(q) * 4 * kSpecCap;
    v.scost = scost + static_cast<int64_t>(q) * 4 * kSpecCap;
    v.stau = stau + static_cast<int64_t>(q) * 4 * kSpecCap;
    for (int l = 0; l < 4; ++l) v.spec_len[l] = po[q].spec_len[l];
    v.subst = po[q].subst;
    views[q] = v;
    D.pool = views + q;
  }
  D.n = Q.n + 1;
  D.dim = kD;
  D.num_boxes = Q.nb;
  D.directed = 1;
  D.goal_count = po[q].goal_any;
  D.init_index = Q.n;
  D.radius = radius;
  D.num_edges = -1;  // (rows are padded; gmt_batch_graph counts them)
  D.coords = qcoords + Q.node_off * kD;
  D.box_lo = box_lo + Q.box_off * kD;
  D.box_hi = box_hi + Q.box_off * kD;
  D.goal_lo = goal_lo + static_cast<int64_t>(q) * kD;
  D.goal_hi = goal_hi + static_cast<int64_t>(q) * kD;
  if (!views) {  // materialised rows (GMT_POOL_ROWS=1)
    D.out_ptr = out_start + Q.node_off;
    D.out_end = out_end + Q.node_off;
    D.out_col = out_col + Q.out_off;
    D.out_cost = nullptr;  // (the solve reads out-row targets only)
    D.in_ptr = in_start + Q.node_off;
    D.in_end = in_end + Q.node_off;
    D.in_col = in_col + Q.in_off;
    D.in_cost = in_cost + Q.in_off;
    D.in_tau = in_tau + Q.in_off;
    if (in_pe && prec) {
      D.in_pe = in_pe + Q.in_off;
      D.pool_rec = prec;
      D.pool_rec_len = prec_len;
    }
  }
  D.steering = GMT_STEER_DOUBLE_INTEGRATOR;
  D.kin_segments = P.segments;
  D.kin_p[0] = P.vmax;
  D.kin_p[1] = P.weight;
  descs[q] = D;
}

__global__ void pool_gather_paths_kernel(const DevResult* __restrict__ rs, const DevInstance* const* __restrict__ insts,
                                         int count, int cap, int d, double* __restrict__ out) {
  const int q = blockIdx.x;
  if (q >= count) return;
  const DevResult R = rs[q];
  const ResultScalars sc = *R.scalars;
  const DevInstance* I = insts[q];
  const int len = sc.status != 0 ? 0 : (sc.path_len < cap ? sc.path_len : cap);
  for (int e = threadIdx.x; e < cap * d; e += blockDim.x) {
    const int k = e / d, i = e - k * d;
    out[static_cast<int64_t>(q) * cap * d + e] = k < len ? I->coords[static_cast<int64_t>(R.path[k]) * d + i] : 0.0;
  }
}

bool same_params(const gmt_di_params& a, const gmt_di_params& b) {
  return a.vmax == b.vmax && a.weight == b.weight && a.segments == b.segments;
}

// Problems that can take the shared pool of problems[0]'s sampling source.
bool pool_eligible(const gmt_problem& p, const gmt_problem& p0) {
  return p.steering == GMT_STEER_DOUBLE_INTEGRATOR && p.scene.dim == kD &&
         p.sampling.kind == GMT_SAMPLE_HALTON && p.sampling.start_index == p0.sampling.start_index &&
         p.radius_override > 0.0 && p.radius_override == p0.radius_override && same_params(p.di, p0.di) &&
         p.n >= 2 && p.n < static_cast<int>(kNoRank) && p.sampling.with_heading == 0;
}

// Candidates to scan for a problem: n over the free-volume estimate (boxes
// clipped to the unit cube), +5 % + 256 (as gmt_plan_problems sizes its
// candidates); a query that runs short widens the scan.
int pool_need(const gmt_problem& pr) {
  double blocked = 0.0;
  for (int b = 0; b < pr.scene.num_boxes; ++b) {
    double v = 1.0;
    for (int k = 0; k < kD; ++k) {
      const double lo = std::max(0.0, pr.scene.box_lo[static_cast<size_t>(b) * kD + k]);
      const double hi = std::min(1.0, pr.scene.box_hi[static_cast<size_t>(b) * kD + k]);
      v *= std::max(0.0, hi - lo);
    }
    blocked += v;
  }
  const double free_est = std::max(0.05, 1.0 - blocked);
  return static_cast<int>(std::ceil(std::min(4.0 * pr.n, pr.n / free_est * 1.05) + 256.0));
}

bool same_source(const SamplePool* p, const gmt_problem& p0) {
  return p && p->start_index == p0.sampling.start_index && p->radius == p0.radius_override &&
         same_params(p->gp, p0.di);
}

// The context's pool for problems like p0 with at least Kp candidate points.
int pool_points(gmt_ctx* ctx, const gmt_problem& p0, int Kp, SamplePool** out) {
  SamplePool* pool = ctx->pool;
  if (!same_source(pool, p0)) {
    destroy_pool(ctx->pool);
    ctx->pool = pool = new SamplePool;
    pool->start_index = p0.sampling.start_index;
    pool->gp = p0.di;
    pool->radius = p0.radius_override;
  }
  *out = pool;
  if (pool->Kp >= Kp) return GMT_OK;
  Kp = (std::max(Kp, pool->Kp + pool->Kp / 2) + 255) & ~255;
  Arena fresh;
  int rc = fresh.reserve(sizeof(double) * static_cast<size_t>(Kp) * kD);
  if (rc) return rc;
  if (pool->Kp)
    GMT_CUDA(cudaMemcpyAsync(fresh.ptr, pool->pts.ptr, sizeof(double) * static_cast<size_t>(pool->Kp) * kD,
                             cudaMemcpyDeviceToDevice, ctx->stream));
  Primes pr;
  for (int k = 0; k < kD; ++k) pr.p[k] = nth_prime_h(k + 1);
  pool_points_kernel<<<std::min(((Kp - pool->Kp) * kD + 255) / 256, 4096), 256, 0, ctx->stream>>>(
      pool->Kp, Kp, pool->start_index, pr, static_cast<double*>(fresh.ptr));
  GMT_CUDA(cudaGetLastError());
  ++ctx->launches;
  pool->pts.release();
  pool->pts = fresh;
  fresh.ptr = nullptr;
  fresh.cap = 0;
  pool->Kp = Kp;
  return GMT_OK;
}

// The pool graph over at least the first K points (rebuilt when it is shorter).
int pool_graph(gmt_ctx* ctx, SamplePool* pool, int K) {
  if (pool->K >= K) return GMT_OK;
  const auto t0 = std::chrono::steady_clock::now();
  K = std::min(pool->Kp, (std::max(K, pool->K + pool->K / 8) + 255) & ~255);
  pool->out_mem.release();
  pool->in_mem.release();
  pool->rec_mem.release();
  pool->rec_len = 0;
  pool->K = 0;
  int rc = build_di_graph_dev(ctx, static_cast<const double*>(pool->pts.ptr), K, &pool->gp, pool->radius,
                              pool->out_mem, &pool->out, pool->in_mem, &pool->in);
  if (rc) return rc;
  const char* rec_env = std::getenv("GMT_POOL_REC");  // 0: no check records (A/B)
  if (!(rec_env && rec_env[0] == '0') && pool->in.edges > 0) {
    const DiParams DP = to_di(&pool->gp);
    const int RL = pool_rec_len(DP.segments);
    rc = pool->rec_mem.reserve(sizeof(double) * static_cast<size_t>(pool->in.edges) * RL);
    if (rc) return rc;
    pool_rec_kernel<<<(K + 7) / 8, 256, 0, ctx->stream>>>(static_cast<const double*>(pool->pts.ptr), K, pool->in.ptr,
                                                        pool->in.col, pool->in.tau, DP, RL,
                                                        static_cast<double*>(pool->rec_mem.ptr));
    GMT_CUDA(cudaGetLastError());
    ++ctx->launches;
    pool->rec_len = RL;
  }
  GMT_CUDA(cudaStreamSynchronize(ctx->stream));
  pool->K = K;
  pool->build_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
  return GMT_OK;
}

struct StageTimer {
  bool on = false;
  cudaStream_t s = nullptr;
  std::vector<cudaEvent_t> ev;
  explicit StageTimer(cudaStream_t st) : s(st) {
    const char* e = std::getenv("GMT_POOL_TIMING");
    on = e && e[0] == '1';
  }
  void mark() {
    if (!on) return;
    cudaEvent_t e;
    cudaEventCreate(&e);
    cudaEventRecord(e, s);
    ev.push_back(e);
  }
  void report(SamplePool* pool) {
    if (!on) return;
    cudaEventSynchronize(ev.back());
    for (size_t i = 1; i < ev.size() && i <= 8; ++i) {
      float ms = 0.0f;
      cudaEventElapsedTime(&ms, ev[i - 1], ev[i]);
      pool->stage_ms[i - 1] = ms;
    }
    for (cudaEvent_t e : ev) cudaEventDestroy(e);
    ev.clear();
  }
};

}  // namespace

// Derive the instances of `count` problems into `meta` / `rows` (device).  On
// return inst[q] is the device descriptor of query q (a derived one, or one of
// the single-built instances appended to `owned`; null when the query's own
// build failed with status[q] = GMT_E_GOAL_BLOCKED / GMT_E_INFEASIBLE_SAMPLING),
// V[q] its vertex count, init[q] its init index, radius[q] its graph radius.
int pool_derive(gmt_ctx* ctx, const gmt_problem* problems, int count, Arena& meta, Arena& rows,
                std::vector<gmt_instance*>& owned, std::vector<const DevInstance*>& inst, std::vector<int>& V,
                std::vector<int>& init, std::vector<double>& radius, std::vector<int32_t>& status, int* max_V,
                int* max_nb, bool* viewed, bool prefer_rows) {
  cudaStream_t s = ctx->stream;
  *viewed = false;
  // Materialised rows cost a derivation pass (8 ms and ~15 GB of writes per
  // 4096 queries) and make each solve faster (37 vs 42 ms): batches built
  // once and launched many times take them (prefer_rows), one-shot
  // gmt_plan_problems reads the pool through each query's rank map.
  // GMT_POOL_ROWS=0/1 forces either (A/B checks).
  const char* mat_env = std::getenv("GMT_POOL_ROWS");
  bool materialise = mat_env && (mat_env[0] == '0' || mat_env[0] == '1') ? mat_env[0] == '1' : prefer_rows;
  const gmt_problem& p0 = problems[0];
  inst.assign(count, nullptr);
  V.assign(count, 0);
  init.assign(count, 0);
  radius.assign(count, 0.0);
  status.assign(count, GMT_OK);
  *max_V = 0;
  *max_nb = 0;
  std::vector<PQ> pq(count);
  // The scene arrays are packed straight into pinned memory (one async copy
  // each at full link speed); the call synchronises before it returns, so
  // the context's staging buffer is free again for the next call.
  int64_t all_boxes = 0;
  for (int q = 0; q < count; ++q) all_boxes += std::max(problems[q].scene.num_boxes, 0);
  const size_t nbox_d = static_cast<size_t>(std::max<int64_t>(all_boxes, 1)) * kD;
  const size_t nq_d = static_cast<size_t>(count) * kD;
  int rc0 = ctx->pool_pinned.reserve(sizeof(double) * (2 * nbox_d + 3 * nq_d));
  if (rc0) return rc0;
  double* h_blo = static_cast<double*>(ctx->pool_pinned.ptr);
  double* h_bhi = h_blo + nbox_d;
  double* h_glo = h_bhi + nbox_d;
  double* h_ghi = h_glo + nq_d;
  double* h_init = h_ghi + nq_d;
  int Kc = 0, eligible = 0, max_nbp = 0, max_n = 0;
  int64_t box_total = 0, node_total = 0;
  for (int q = 0; q < count; ++q) {
    const gmt_problem& pr = problems[q];
    int rc = validate_scene(&pr.scene);
    if (rc) return rc;
    if (!(pr.lambda > 0.0 && pr.lambda <= 1.0)) return set_error(GMT_E_INVALID_INPUT, "lambda must be in (0, 1]");
    PQ& Q = pq[q];
    std::memset(&Q, 0, sizeof(Q));
    Q.skip = pool_eligible(pr, p0) && validate_di(&pr.di) == GMT_OK ? 0 : 1;
    if (Q.skip) continue;
    ++eligible;
    Q.n = pr.n;
    Q.nb = pr.scene.num_boxes;
    Q.box_off = box_total;
    Q.node_off = node_total;
    Kc = std::max(Kc, pool_need(pr));
    max_nbp = std::max(max_nbp, Q.nb);
    max_n = std::max(max_n, pr.n);
    std::memcpy(h_blo + box_total * kD, pr.scene.box_lo, sizeof(double) * static_cast<size_t>(Q.nb) * kD);
    std::memcpy(h_bhi + box_total * kD, pr.scene.box_hi, sizeof(double) * static_cast<size_t>(Q.nb) * kD);
    std::memcpy(h_glo + static_cast<size_t>(q) * kD, pr.scene.goal_lo, sizeof(double) * kD);
    std::memcpy(h_ghi + static_cast<size_t>(q) * kD, pr.scene.goal_hi, sizeof(double) * kD);
    std::memcpy(h_init + static_cast<size_t>(q) * kD, pr.init, sizeof(double) * kD);
    box_total += Q.nb;
    node_total += Q.n + 1;
  }
  g_last_error.clear();
  {  // (views are read by the on-chip solve; larger queries get materialised rows)
    const SolveLayout L = solve_layout(max_n + 1, kD, max_nbp, true, false);
    if (L.total > ctx->smem_optin) materialise = true;
  }
  std::vector<PQOut> po(count);
  SamplePool* pool = nullptr;
  StageTimer timer(s);
  if (eligible) {
    // The candidate scan covers the pool graph (steady state: every query's
    // cutoff already lies inside it) or the free-volume estimate.
    if (same_source(ctx->pool, p0) && ctx->pool->K > 0) Kc = std::min(Kc, ctx->pool->K);
    Kc = std::min<int64_t>(Kc, 1000LL * max_n);
    for (;;) {
      int rc = pool_points(ctx, p0, Kc, &pool);
      if (rc) return rc;
      Carver c;
      const size_t o_pq = c.take<PQ>(count);
      const size_t o_po = c.take<PQOut>(count);
      const size_t o_blo = c.take<double>(std::max<int64_t>(box_total, 1) * kD);
      const size_t o_bhi = c.take<double>(std::max<int64_t>(box_total, 1) * kD);
      const size_t o_glo = c.take<double>(nq_d);
      const size_t o_ghi = c.take<double>(nq_d);
      const size_t o_init = c.take<double>(nq_d);
      const size_t o_flag = c.take<uint8_t>(static_cast<size_t>(count) * Kc);
      const size_t o_rank = c.take<uint16_t>(static_cast<size_t>(count) * Kc);
      const size_t o_sel = c.take<int32_t>(node_total);
      const size_t o_qc = c.take<double>(node_total * kD);
      const size_t o_scol = c.take<int32_t>(static_cast<size_t>(count) * 4 * kSpecCap);
      const size_t o_scost = c.take<double>(static_cast<size_t>(count) * 4 * kSpecCap);
      const size_t o_stau = c.take<double>(static_cast<size_t>(count) * 4 * kSpecCap);
      const size_t o_cand = c.take<int32_t>(static_cast<size_t>(count) * 4 * kCandCap);
      const size_t o_spc = c.take<int32_t>(node_total);
      const size_t o_spj = c.take<uint16_t>(2 * node_total);
      const size_t o_is = c.take<int64_t>(node_total);
      const size_t o_ie = c.take<int64_t>(node_total);
      const size_t o_os = c.take<int64_t>(node_total);
      const size_t o_oe = c.take<int64_t>(node_total);
      const size_t o_desc = c.take<DevInstance>(count);
      const size_t o_view = c.take<PoolView>(count);
      rc = meta.reserve(c.off);
      if (rc) return rc;
      char* B = static_cast<char*>(meta.ptr);
      auto* d_pq = reinterpret_cast<PQ*>(B + o_pq);
      auto* d_po = reinterpret_cast<PQOut*>(B + o_po);
      auto* d_blo = reinterpret_cast<double*>(B + o_blo);
      auto* d_bhi = reinterpret_cast<double*>(B + o_bhi);
      auto* d_glo = reinterpret_cast<double*>(B + o_glo);
      auto* d_ghi = reinterpret_cast<double*>(B + o_ghi);
      auto* d_init = reinterpret_cast<double*>(B + o_init);
      auto* d_flag = reinterpret_cast<uint8_t*>(B + o_flag);
      auto* d_rank = reinterpret_cast<uint16_t*>(B + o_rank);
      auto* d_sel = reinterpret_cast<int32_t*>(B + o_sel);
      auto* d_qc = reinterpret_cast<double*>(B + o_qc);
      auto* d_scol = reinterpret_cast<int32_t*>(B + o_scol);
      auto* d_scost = reinterpret_cast<double*>(B + o_scost);
      auto* d_stau = reinterpret_cast<double*>(B + o_stau);
      auto* d_cand = reinterpret_cast<int32_t*>(B + o_cand);
      auto* d_spc = reinterpret_cast<int32_t*>(B + o_spc);
      auto* d_spj = reinterpret_cast<uint16_t*>(B + o_spj);
      auto* d_is = reinterpret_cast<int64_t*>(B + o_is);
      auto* d_ie = reinterpret_cast<int64_t*>(B + o_ie);
      auto* d_os = reinterpret_cast<int64_t*>(B + o_os);
      auto* d_oe = reinterpret_cast<int64_t*>(B + o_oe);
      auto* d_desc = reinterpret_cast<DevInstance*>(B + o_desc);
      auto* d_view = reinterpret_cast<PoolView*>(B + o_view);
      auto put = [&](void* dst, const void* src, size_t bytes) -> int {
        if (bytes) GMT_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, s));
        return GMT_OK;
      };
      timer.mark();
      if ((rc = put(d_pq, pq.data(), sizeof(PQ) * count)) ||
          (rc = put(d_blo, h_blo, sizeof(double) * box_total * kD)) ||
          (rc = put(d_bhi, h_bhi, sizeof(double) * box_total * kD)) ||
          (rc = put(d_glo, h_glo, sizeof(double) * nq_d)) ||
          (rc = put(d_ghi, h_ghi, sizeof(double) * nq_d)) ||
          (rc = put(d_init, h_init, sizeof(double) * nq_d)))
        return rc;
      const double* P = static_cast<const double*>(pool->pts.ptr);
      const int stage_cap = 2048;  // boxes staged in shared memory up to 2048 * 96 B
      const int nb_st = std::min(max_nbp, stage_cap);
      const size_t fsm = sizeof(double) * 2 * kD * static_cast<size_t>(std::max(nb_st, 1));
      if (fsm > 48 * 1024)
        GMT_CUDA(cudaFuncSetAttribute(pool_free_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      static_cast<int>(fsm)));
      timer.mark();
      pool_free_kernel<<<dim3((Kc + kFreePts - 1) / kFreePts, count), 256, fsm, s>>>(d_pq, P, Kc, d_blo, d_bhi, nb_st,
                                                                                    d_flag);
      timer.mark();
      pool_select_kernel<<<count, 1024, 0, s>>>(d_pq, P, Kc, d_flag, d_glo, d_ghi, d_rank, d_sel, d_qc, d_po);
      GMT_CUDA(cudaGetLastError());
      ctx->launches += 2;
      GMT_CUDA(cudaMemcpyAsync(po.data(), d_po, sizeof(PQOut) * count, cudaMemcpyDeviceToHost, s));
      GMT_CUDA(cudaStreamSynchronize(s));
      int cutoff = 0, need = 0;
      for (int q = 0; q < count; ++q) {
        if (pq[q].skip) continue;
        if (po[q].fallback) need = std::max(need, Kc + Kc / 2);  // short: widen the scan
        else cutoff = std::max(cutoff, po[q].cutoff);
      }
      if (need > Kc && Kc < 1000LL * max_n) {
        Kc = static_cast<int>(std::min<int64_t>(need, 1000LL * max_n));
        continue;
      }
      rc = pool_graph(ctx, pool, cutoff);
      if (rc) return rc;
      const DiParams DP = to_di(&p0.di);
      Primes pr;
      for (int k = 0; k < kD; ++k) pr.p[k] = nth_prime_h(k + 1);
      timer.mark();
      pool_subst_kernel<<<count, 256, 0, s>>>(d_pq, Kc, d_blo, d_bhi, d_glo, d_ghi, pr, d_rank, d_sel, d_qc, d_po);
      pool_init_kernel<<<count, 256, 0, s>>>(d_pq, d_init, d_qc, d_po);
      timer.mark();
      GMT_CUDA(cudaMemsetAsync(d_spc, 0, sizeof(int32_t) * node_total, s));
      pool_special_cand_kernel<<<(4 * count + 7) / 8, 256, 0, s>>>(d_pq, DP, di_prefilter_bound(DP, pool->radius),
                                                                    pool->radius, d_qc, d_cand, d_po);
      pool_special_kernel<<<count, 128, 0, s>>>(d_pq, DP, pool->radius, d_qc, d_cand, d_scol, d_scost, d_stau, d_spc,
                                                d_spj, d_po);
      timer.mark();
      ctx->launches += 4;
      if (!materialise) {  // the graphs are views of the pool: no per-query rows
        PoolView sv{};
        sv.in_ptr = pool->in.ptr;
        sv.in_col = pool->in.col;
        sv.in_cost = pool->in.cost;
        sv.in_tau = pool->in.tau;
        sv.out_ptr = pool->out.ptr;
        sv.out_col = pool->out.col;
        sv.cap = kSpecCap;
        sv.kc = Kc;
        sv.k = pool->K;
        sv.rec = pool->rec_len ? static_cast<const double*>(pool->rec_mem.ptr) : nullptr;
        sv.rec_len = pool->rec_len;
        pool_desc_kernel<<<(count + 127) / 128, 128, 0, s>>>(
            d_pq, d_po, count, pool->radius, DP, d_qc, d_blo, d_bhi, d_glo, d_ghi, nullptr, nullptr, nullptr, nullptr,
            nullptr, nullptr, nullptr, nullptr, d_desc, d_view, sv, d_sel, d_rank, d_spc, d_spj, d_scol, d_scost,
            d_stau, nullptr, nullptr, 0);
        GMT_CUDA(cudaGetLastError());
        ++ctx->launches;
        GMT_CUDA(cudaMemcpyAsync(po.data(), d_po, sizeof(PQOut) * count, cudaMemcpyDeviceToHost, s));
        GMT_CUDA(cudaStreamSynchronize(s));
        timer.mark();
        for (int q = 0; q < count; ++q) {
          if (pq[q].skip || po[q].fallback) continue;
          inst[q] = d_desc + q;
          V[q] = pq[q].n + 1;
          init[q] = pq[q].n;
          radius[q] = pool->radius;
          *max_V = std::max(*max_V, V[q]);
          *max_nb = std::max(*max_nb, pq[q].nb);
          *viewed = true;
        }
        break;
      }
      pool_layout_kernel<<<count, 1024, 0, s>>>(d_pq, pool->in.ptr, pool->out.ptr, d_sel, d_is, d_os, d_po);
      GMT_CUDA(cudaGetLastError());
      ++ctx->launches;
      GMT_CUDA(cudaMemcpyAsync(po.data(), d_po, sizeof(PQOut) * count, cudaMemcpyDeviceToHost, s));
      GMT_CUDA(cudaStreamSynchronize(s));
      int64_t tin = 0, tout = 0;
      for (int q = 0; q < count; ++q) {
        if (pq[q].skip || po[q].fallback) continue;
        pq[q].in_off = tin;
        pq[q].out_off = tout;
        tin += po[q].tot_in;
        tout += po[q].tot_out;
      }
      Carver r;
      const size_t o_icol = r.take<int32_t>(tin);
      const size_t o_icost = r.take<double>(tin);
      const size_t o_itau = r.take<double>(tin);
      const size_t o_ocol = r.take<int32_t>(tout);
      const bool recs = pool->rec_len > 0;
      const size_t o_ipe = recs ? r.take<int32_t>(tin) : 0;
      rc = rows.reserve(r.off);
      if (rc) return rc;
      char* R = static_cast<char*>(rows.ptr);
      auto* d_icol = reinterpret_cast<int32_t*>(R + o_icol);
      auto* d_icost = reinterpret_cast<double*>(R + o_icost);
      auto* d_itau = reinterpret_cast<double*>(R + o_itau);
      auto* d_ocol = reinterpret_cast<int32_t*>(R + o_ocol);
      auto* d_ipe = recs ? reinterpret_cast<int32_t*>(R + o_ipe) : nullptr;
      if ((rc = put(d_pq, pq.data(), sizeof(PQ) * count))) return rc;
      timer.mark();
      const size_t rsm = sizeof(uint16_t) * static_cast<size_t>(Kc);
      const int stage_rank = rsm <= 96 * 1024 ? 1 : 0;
      // (a warp per vertex measured best: 8.2 ms vs 10.5 with 8-lane groups
      // for 4096 queries; streaming stores made no difference)
      auto rows_kern = pool_rows_kernel<32, false>;
      if (stage_rank && rsm > 48 * 1024)
        GMT_CUDA(cudaFuncSetAttribute(rows_kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      static_cast<int>(rsm)));
      rows_kern<<<dim3((max_n + 1 + kRowTile - 1) / kRowTile, count), 256, stage_rank ? rsm : 0, s>>>(
          d_pq, d_po, Kc, stage_rank, pool->in.ptr, pool->in.col, pool->in.cost, pool->in.tau, pool->out.ptr, pool->out.col,
          d_rank, d_sel, d_scol, d_scost, d_stau, d_spc, d_spj, d_is, d_ie, d_os, d_oe, d_icol, d_icost, d_itau,
          d_ocol, d_ipe);
      timer.mark();
      pool_desc_kernel<<<(count + 127) / 128, 128, 0, s>>>(d_pq, d_po, count, pool->radius, DP, d_qc, d_blo, d_bhi,
                                                           d_glo, d_ghi, d_is, d_ie, d_os, d_oe, d_icol, d_icost,
                                                           d_itau, d_ocol, d_desc, nullptr, PoolView{}, nullptr,
                                                           nullptr, nullptr, nullptr, nullptr, nullptr, nullptr,
                                                           d_ipe, static_cast<const double*>(pool->rec_mem.ptr),
                                                           pool->rec_len);
      GMT_CUDA(cudaGetLastError());
      timer.mark();
      ctx->launches += 2;
      for (int q = 0; q < count; ++q) {
        if (pq[q].skip || po[q].fallback) continue;
        inst[q] = d_desc + q;
        V[q] = pq[q].n + 1;
        init[q] = pq[q].n;
        radius[q] = pool->radius;
        *max_V = std::max(*max_V, V[q]);
        *max_nb = std::max(*max_nb, pq[q].nb);
      }
      break;
    }
    timer.report(pool);
  }
  // The rare paths and the problems off the pool: the single-instance builder.
  int fallbacks = 0;
  for (int q = 0; q < count; ++q) {
    if (!pq[q].skip && !po[q].fallback) continue;
    ++fallbacks;
    gmt_instance* one = nullptr;
    int rc = gmt_instance_build(ctx, &problems[q], &one);
    if (rc == GMT_E_GOAL_BLOCKED || rc == GMT_E_INFEASIBLE_SAMPLING) {
      status[q] = rc;  // the query's own build outcome (sampling.cpp:97-141)
      continue;
    }
    if (rc) return rc;
    owned.push_back(one);
    inst[q] = static_cast<const DevInstance*>(one->desc_mem.ptr);
    V[q] = one->desc.n;
    init[q] = one->desc.init_index;
    radius[q] = one->desc.radius;
    *max_V = std::max(*max_V, V[q]);
    *max_nb = std::max(*max_nb, one->desc.num_boxes);
  }
  if (pool) pool->last_fallbacks = fallbacks;
  return GMT_OK;
}

int pool_stats(const gmt_ctx* ctx, int32_t* K, int64_t* edges, double* build_ms, int32_t* fallbacks,
               double* stage_ms) {
  const SamplePool* p = ctx->pool;
  if (K) *K = p ? p->K : 0;
  if (edges) *edges = p ? p->out.edges : 0;
  if (build_ms) *build_ms = p ? p->build_ms : 0.0;
  if (fallbacks) *fallbacks = p ? p->last_fallbacks : 0;
  if (stage_ms)
    for (int i = 0; i < 8; ++i) stage_ms[i] = p ? p->stage_ms[i] : 0.0;
  return GMT_OK;
}

// Solve jobs for derived queries (status != OK entries are skipped).
static int batch_from_derived(gmt_ctx* ctx, gmt_batch* b, const gmt_problem* problems, int count,
                              const std::vector<const DevInstance*>& inst, const std::vector<int>& V,
                              const std::vector<int>& init, const std::vector<double>& radius, int max_V,
                              int max_nb, std::vector<int>& job_q, bool tree_stats) {
  b->ctx = ctx;
  b->node_off.assign(1, 0);
  job_q.clear();
  const int d = problems[0].scene.dim;
  bool kino = false;
  for (int q = 0; q < count; ++q) {
    if (problems[q].scene.dim != d) return set_error(GMT_E_INVALID_INPUT, "all problems of a batch share the dimension");
    kino = kino || problems[q].steering != GMT_STEER_EUCLIDEAN;
    if (!inst[q]) continue;
    SolveJob j{};
    j.inst = inst[q];
    j.init_index = init[q];
    j.mode = kModeGmt;
    j.lambda = problems[q].lambda;
    j.radius = radius[q];
    b->jobs.push_back(j);
    b->node_off.push_back(b->node_off.back() + V[q]);
    job_q.push_back(q);
  }
  const int J = static_cast<int>(b->jobs.size());
  if (J == 0) return GMT_OK;
  b->dim = d;
  // (the shape gmt_batch_create picks: 2-CTA clusters for a few kinodynamic
  // queries, one CTA each once they fill the SMs several times over)
  // Batched 6D double integrators: one 24-warp CTA per query (the shape
  // that measured best at every batch size: 4096 queries 34.4 ms vs 36.1 on
  // narrow CTAs, 512 queries 4.7 vs 5.8 ms; tools/scale_probe.py); other
  // kinodynamic queries: 2-CTA clusters while they fill the SMs less than
  // four times, single CTAs beyond.
  const bool di6 = kino && d == 6;
  b->cluster = ctx->batch_cluster ? ctx->batch_cluster : (di6 ? 1 : (kino && J < 4 * ctx->sm_count ? 2 : 1));
  if (b->pool) b->cluster = 1;  // (pool views are read by single-CTA solves)
  b->threads = ctx->batch_threads ? ctx->batch_threads : (b->cluster > 1 ? 512 : (di6 ? 768 : 256));
  if (b->threads == 768 && (b->cluster != 1 || d != 6)) b->threads = b->cluster > 1 ? 512 : 256;
  size_t gs = 0;
  int rc = plan_smem(ctx, max_V, d, max_nb, b->cluster, &b->smem, &b->obs, &gs);
  if (rc) return rc;
  if (!gs && solve_dyn_scratch(b->threads, d)) {  // (the 24-warp shape's scratch)
    const size_t total = align16(b->smem) + solve_dyn_scratch(b->threads, d);
    if (total <= ctx->smem_optin) {
      b->smem = total;
    } else {
      b->threads = 256;  // (too large for the 24-warp shape's scratch)
    }
  }

  if (gs) {  // too large for shared memory: global-memory wavefronts, one wide CTA each
    b->cluster = 1;
    b->threads = 512;
    rc = assign_gstate(b->gstate_mem, b->jobs, gs);
    if (rc) return rc;
  }
  rc = carve_results(b->res, J, b->node_off.data(), tree_stats, tree_stats, b->results, &b->scalars,
                     ctx->counting ? ctx->counters : nullptr);
  if (rc) return rc;
  for (int k = 0; k < J; ++k) b->jobs[k].res = b->results[k];
  rc = b->jobs_mem.reserve(sizeof(SolveJob) * J);
  if (rc) return rc;
  cudaError_t e = cudaMemcpyAsync(b->jobs_mem.ptr, b->jobs.data(), sizeof(SolveJob) * J, cudaMemcpyHostToDevice,
                                  ctx->stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(ctx->stream);
  if (e != cudaSuccess) return cuda_error(e, "batch jobs");
  return GMT_OK;
}

// gmt_plan_problems for double-integrator problems (batch_build.cu routes here).
int plan_problems_pool(gmt_ctx* ctx, const gmt_problem* problems, int32_t count, int32_t* status_out,
                       gmt_plan_summary* summaries, int32_t path_cap, double* path_states) {
  std::vector<gmt_instance*> owned;
  std::vector<const DevInstance*> inst;
  std::vector<int> V, init, job_q;
  std::vector<double> radius;
  std::vector<int32_t> status;
  int max_V = 0, max_nb = 0;
  bool viewed = false;
  int rc = pool_derive(ctx, problems, count, ctx->pool_work, ctx->pool_rows, owned, inst, V, init, radius, status,
                       &max_V, &max_nb, &viewed, false);
  gmt_batch b;
  b.pool = viewed;
  b.res = ctx->pool_res;  // (kept in the context across calls, like the derived instances)
  ctx->pool_res = Arena{};
  if (rc == GMT_OK)  // summaries (and paths) only: no trees, no per-pass stats
    rc = batch_from_derived(ctx, &b, problems, count, inst, V, init, radius, max_V, max_nb, job_q, false);
  const int J = static_cast<int>(b.jobs.size());
  cudaStream_t s = ctx->stream;
  if (rc == GMT_OK && J > 0) {
    rc = gmt_batch_launch(ctx, &b);
    std::vector<ResultScalars> hs(J);
    cudaError_t e = cudaSuccess;
    if (rc == GMT_OK) e = cudaMemcpyAsync(hs.data(), b.scalars, sizeof(ResultScalars) * J, cudaMemcpyDeviceToHost, s);
    Arena pg;
    if (rc == GMT_OK && e == cudaSuccess && path_states && path_cap > 0) {
      const size_t o_r = 0, o_i = align16(sizeof(DevResult) * J), o_o = o_i + align16(sizeof(void*) * J);
      rc = pg.reserve(o_o + sizeof(double) * static_cast<size_t>(J) * path_cap * kD);
      if (rc == GMT_OK) {
        std::vector<const DevInstance*> ip(J);
        for (int k = 0; k < J; ++k) ip[k] = b.jobs[k].inst;
        char* g = static_cast<char*>(pg.ptr);
        e = cudaMemcpyAsync(g + o_r, b.results.data(), sizeof(DevResult) * J, cudaMemcpyHostToDevice, s);
        if (e == cudaSuccess) e = cudaMemcpyAsync(g + o_i, ip.data(), sizeof(void*) * J, cudaMemcpyHostToDevice, s);
        if (e == cudaSuccess) {
          pool_gather_paths_kernel<<<J, 128, 0, s>>>(reinterpret_cast<const DevResult*>(g + o_r),
                                                     reinterpret_cast<const DevInstance* const*>(g + o_i), J,
                                                     path_cap, kD, reinterpret_cast<double*>(g + o_o));
          e = cudaGetLastError();
          ++ctx->launches;
        }
        std::vector<double> hp(static_cast<size_t>(J) * path_cap * kD);
        if (e == cudaSuccess)
          e = cudaMemcpyAsync(hp.data(), g + o_o, sizeof(double) * hp.size(), cudaMemcpyDeviceToHost, s);
        if (e == cudaSuccess) e = cudaStreamSynchronize(s);
        if (e == cudaSuccess)
          for (int k = 0; k < J; ++k)
            std::memcpy(path_states + static_cast<size_t>(job_q[k]) * path_cap * kD,
                        hp.data() + static_cast<size_t>(k) * path_cap * kD, sizeof(double) * path_cap * kD);
      }
    }
    if (rc == GMT_OK && e == cudaSuccess) e = cudaStreamSynchronize(s);
    pg.release();
    if (rc == GMT_OK && e != cudaSuccess) rc = cuda_error(e, "gmt_plan_problems results");
    if (rc == GMT_OK) {
      for (int k = 0; k < J; ++k) {
        gmt_plan_summary& o = summaries[job_q[k]];
        o.status = hs[k].status;
        o.goal_node = hs[k].goal_node;
        o.cost = hs[k].cost;
        o.iterations = hs[k].iterations;
        o.total_collision_checks = hs[k].total_checks;
        o.path_len = hs[k].path_len;
        o.num_stats = hs[k].num_stats;
      }
    }
  }
  if (rc == GMT_OK)
    for (int q = 0; q < count; ++q) status_out[q] = status[q];
  ctx->pool_res = b.res;
  b.res = Arena{};
  b.jobs_mem.release();
  for (gmt_instance* i : owned) gmt_instance_destroy(i);
  return rc;
}

}  // namespace gmtb

using namespace gmtb;

extern "C" int gmt_batch_create_problems(gmt_ctx* ctx, const gmt_problem* problems, int32_t count,
                                         int32_t* status_out, gmt_batch** out) {
  gmtb::AllocScope alloc_scope_(ctx);
  *out = nullptr;
  if (count < 1) return set_error(GMT_E_INVALID_INPUT, "batch needs at least one problem");
  auto* b = new gmt_batch;
  std::vector<const DevInstance*> inst;
  std::vector<int> V, init, job_q;
  std::vector<double> radius;
  std::vector<int32_t> status;
  int max_V = 0, max_nb = 0;
  bool viewed = false;
  int rc = pool_derive(ctx, problems, count, b->derived, b->derived_rows, b->owned, inst, V, init, radius, status,
                       &max_V, &max_nb, &viewed, true);
  b->pool = viewed;
  if (rc == GMT_OK)
    rc = batch_from_derived(ctx, b, problems, count, inst, V, init, radius, max_V, max_nb, job_q, true);
  if (rc == GMT_OK && b->jobs.empty()) rc = set_error(GMT_E_INVALID_INPUT, "no problem of the batch could be built");
  if (rc != GMT_OK) {
    delete b;
    return rc;
  }
  for (int q = 0; q < count; ++q) status_out[q] = status[q];
  *out = b;
  return GMT_OK;
}

extern "C" int gmt_ctx_pool_info(gmt_ctx* ctx, int32_t* pool_size, int64_t* num_edges, double* build_ms,
                                 int32_t* last_fallbacks, double* stage_ms) {
  if (!ctx) return set_error(GMT_E_INVALID_INPUT, "context is null");
  return pool_stats(ctx, pool_size, num_edges, build_ms, last_fallbacks, stage_ms);
}

// Rows of batch query q as compressed rows (host): the two-call pattern of
// the graph entry points (NULL in_ptr: sizes only).
extern "C" int gmt_batch_graph(gmt_ctx* ctx, gmt_batch* b, int32_t q, int32_t* n, int64_t* num_in, int64_t* num_out,
                               double* coords, int64_t* in_ptr, int32_t* in_col, double* in_cost, double* in_tau,
                               int64_t* out_ptr, int32_t* out_col) {
  gmtb::AllocScope alloc_scope_(ctx);
  if (!b || q < 0 || q >= static_cast<int32_t>(b->jobs.size()))
    return set_error(GMT_E_INVALID_INPUT, "query index out of range");
  cudaStream_t s = ctx->stream;
  DevInstance D;
  GMT_CUDA(cudaMemcpyAsync(&D, b->jobs[q].inst, sizeof(D), cudaMemcpyDeviceToHost, s));
  GMT_CUDA(cudaStreamSynchronize(s));
  const int V = D.n;
  if (D.pool) {  // a view of the shared pool: the rows the solve reads, rebuilt on the host
    PoolView pv;
    GMT_CUDA(cudaMemcpyAsync(&pv, D.pool, sizeof(pv), cudaMemcpyDeviceToHost, s));
    GMT_CUDA(cudaStreamSynchronize(s));
    const int K = pv.k, cap = pv.cap;
    std::vector<int64_t> pip(K + 1), pop(K + 1);
    GMT_CUDA(cudaMemcpyAsync(pip.data(), pv.in_ptr, sizeof(int64_t) * (K + 1), cudaMemcpyDeviceToHost, s));
    GMT_CUDA(cudaMemcpyAsync(pop.data(), pv.out_ptr, sizeof(int64_t) * (K + 1), cudaMemcpyDeviceToHost, s));
    GMT_CUDA(cudaStreamSynchronize(s));
    const int64_t Ei = pip[K], Eo = pop[K];
    std::vector<int32_t> pic(Ei), poc(Eo), sel(V), code(V), scol(4 * cap);
    std::vector<double> pics(Ei), pit(Ei), scost(4 * cap), stau(4 * cap);
    std::vector<uint16_t> rank(pv.kc), spj(2 * static_cast<size_t>(V));
    auto get = [&](void* dst, const void* src, size_t bytes) -> int {
      if (bytes) GMT_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, s));
      return GMT_OK;
    };
    int rc = GMT_OK;
    if ((rc = get(pic.data(), pv.in_col, 4 * Ei)) || (rc = get(pics.data(), pv.in_cost, 8 * Ei)) ||
        (rc = get(pit.data(), pv.in_tau, 8 * Ei)) || (rc = get(poc.data(), pv.out_col, 4 * Eo)) ||
        (rc = get(sel.data(), pv.sel, 4 * static_cast<size_t>(V - 1))) ||
        (rc = get(code.data(), pv.code, 4 * static_cast<size_t>(V))) ||
        (rc = get(spj.data(), pv.spj, 2 * 2 * static_cast<size_t>(V))) ||
        (rc = get(rank.data(), pv.rank, 2 * static_cast<size_t>(pv.kc))) ||
        (rc = get(scol.data(), pv.scol, 4 * 4 * static_cast<size_t>(cap))) ||
        (rc = get(scost.data(), pv.scost, 8 * 4 * static_cast<size_t>(cap))) ||
        (rc = get(stau.data(), pv.stau, 8 * 4 * static_cast<size_t>(cap))))
      return rc;
    GMT_CUDA(cudaStreamSynchronize(s));
    std::vector<int64_t> iptr(1, 0), optr(1, 0);
    std::vector<int32_t> icol, ocol;
    std::vector<double> icost, itau;
    const int init = V - 1, g = V - 2;
    for (int x = 0; x < V; ++x) {
      if (x == init || (pv.subst && x == g)) {
        const int l = x == init ? 2 : 0;
        for (int j = 0; j < pv.spec_len[l + 1]; ++j) {
          icol.push_back(scol[(l + 1) * cap + j]);
          icost.push_back(scost[(l + 1) * cap + j]);
          itau.push_back(stau[(l + 1) * cap + j]);
        }
        for (int j = 0; j < pv.spec_len[l]; ++j) ocol.push_back(scol[l * cap + j]);
      } else {
        const int p = sel[x];
        for (int64_t e = pip[p]; e < pip[p + 1]; ++e) {
          if (pic[e] >= pv.kc || rank[pic[e]] == kPoolNoRank) continue;
          icol.push_back(rank[pic[e]]);
          icost.push_back(pics[e]);
          itau.push_back(pit[e]);
        }
        if (pv.subst && (code[x] & 1)) {
          icol.push_back(g);
          icost.push_back(scost[spj[2 * x]]);
          itau.push_back(stau[spj[2 * x]]);
        }
        if (code[x] & 4) {
          icol.push_back(init);
          icost.push_back(scost[2 * cap + spj[2 * x + 1]]);
          itau.push_back(stau[2 * cap + spj[2 * x + 1]]);
        }
        for (int64_t e = pop[p]; e < pop[p + 1]; ++e)
          if (poc[e] < pv.kc && rank[poc[e]] != kPoolNoRank) ocol.push_back(rank[poc[e]]);
        if (pv.subst && (code[x] & 2)) ocol.push_back(g);
        if (code[x] & 8) ocol.push_back(init);
      }
      iptr.push_back(static_cast<int64_t>(icol.size()));
      optr.push_back(static_cast<int64_t>(ocol.size()));
    }
    *n = V;
    *num_in = static_cast<int64_t>(icol.size());
    *num_out = static_cast<int64_t>(ocol.size());
    if (!in_ptr) return GMT_OK;
    if (coords) GMT_CUDA(cudaMemcpyAsync(coords, D.coords, sizeof(double) * V * D.dim, cudaMemcpyDeviceToHost, s));
    std::copy(iptr.begin(), iptr.end(), in_ptr);
    std::copy(optr.begin(), optr.end(), out_ptr);
    std::copy(icol.begin(), icol.end(), in_col);
    if (in_cost) std::copy(icost.begin(), icost.end(), in_cost);
    if (in_tau) std::copy(itau.begin(), itau.end(), in_tau);
    if (out_col) std::copy(ocol.begin(), ocol.end(), out_col);
    GMT_CUDA(cudaStreamSynchronize(s));
    return GMT_OK;
  }
  std::vector<int64_t> is(V + 1), ie(V), os(V + 1), oe(V);
  GMT_CUDA(cudaMemcpyAsync(is.data(), D.in_ptr, sizeof(int64_t) * (D.in_end ? V : V + 1), cudaMemcpyDeviceToHost, s));
  GMT_CUDA(cudaMemcpyAsync(os.data(), D.out_ptr, sizeof(int64_t) * (D.out_end ? V : V + 1), cudaMemcpyDeviceToHost, s));
  if (D.in_end) GMT_CUDA(cudaMemcpyAsync(ie.data(), D.in_end, sizeof(int64_t) * V, cudaMemcpyDeviceToHost, s));
  if (D.out_end) GMT_CUDA(cudaMemcpyAsync(oe.data(), D.out_end, sizeof(int64_t) * V, cudaMemcpyDeviceToHost, s));
  GMT_CUDA(cudaStreamSynchronize(s));
  for (int x = 0; x < V; ++x) {
    if (!D.in_end) ie[x] = is[x + 1];
    if (!D.out_end) oe[x] = os[x + 1];
  }
  int64_t ni = 0, no = 0;
  for (int x = 0; x < V; ++x) {
    ni += ie[x] - is[x];
    no += oe[x] - os[x];
  }
  *n = V;
  *num_in = ni;
  *num_out = no;
  if (!in_ptr) return GMT_OK;
  if (coords) GMT_CUDA(cudaMemcpyAsync(coords, D.coords, sizeof(double) * V * D.dim, cudaMemcpyDeviceToHost, s));
  int64_t wi = 0, wo = 0;
  in_ptr[0] = 0;
  out_ptr[0] = 0;
  for (int x = 0; x < V; ++x) {
    const int64_t li = ie[x] - is[x], lo = oe[x] - os[x];
    if (li) {
      GMT_CUDA(cudaMemcpyAsync(in_col + wi, D.in_col + is[x], sizeof(int32_t) * li, cudaMemcpyDeviceToHost, s));
      if (in_cost && D.in_cost)
        GMT_CUDA(cudaMemcpyAsync(in_cost + wi, D.in_cost + is[x], sizeof(double) * li, cudaMemcpyDeviceToHost, s));
      if (in_tau && D.in_tau)
        GMT_CUDA(cudaMemcpyAsync(in_tau + wi, D.in_tau + is[x], sizeof(double) * li, cudaMemcpyDeviceToHost, s));
    }
    if (lo && out_col)
      GMT_CUDA(cudaMemcpyAsync(out_col + wo, D.out_col + os[x], sizeof(int32_t) * lo, cudaMemcpyDeviceToHost, s));
    wi += li;
    wo += lo;
    in_ptr[x + 1] = wi;
    out_ptr[x + 1] = wo;
  }
  GMT_CUDA(cudaStreamSynchronize(s));
  return GMT_OK;
}
