// sample.cu -- sample_free (sampling.cpp:81-142), append_init (:144-154) and
// build_instance (problem.cpp:336-363) on the device.
//
// The reference draws candidates one at a time and keeps the first n that
// are free and not exact duplicates.  Here the candidate stream is
// generated in parallel chunks -- Halton by index, PCG32 by O(log j)
// jump-ahead to draw j*dd -- with point_free evaluated per candidate, then
// an order-preserving compaction keeps stream order, so the kept set is
// the reference's set bit for bit.  Duplicates: Halton points are distinct
// whenever start_index + budget < 2^53 (coordinate 0 is the exact base-2
// radical inverse, injective on those indices), so only uniform streams run
// the exact-duplicate pass (each kept candidate against all earlier ones).
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "common.cuh"
#include "internal.cuh"
#include "di.cuh"
#include "offline.cuh"
#include "quad.cuh"
#include "sample_dev.cuh"
#include "solve.cuh"

namespace gmtb {

namespace {

constexpr uint32_t kFull = 0xffffffffu;
constexpr int kMaxDimS = 16;

#define GMT_CUDA(call)                                   \
  do {                                                   \
    cudaError_t _e = (call);                             \
    if (_e != cudaSuccess) return cuda_error(_e, #call); \
  } while (0)

struct GenParams {
  int kind;
  int with_heading;
  int d;
  int dd;  // draws per candidate (uniform)
  int nb;
  int count;
  uint64_t start_index;
  uint64_t s0;  // uniform: generator state before the first draw
  uint64_t j0;  // first attempt index of the chunk
  const double* box_lo;
  const double* box_hi;
  uint32_t primes[kMaxDimS + 1];
};

__device__ __forceinline__ bool point_free_serial(const double* p, int d, const double* lo,
                                                  const double* hi, int nb) {
  if (!point_in_cube(p, d)) return false;  // space.cpp:47-54
  for (int b = 0; b < nb; ++b)
    if (box_contains(lo + b * d, hi + b * d, d, p)) return false;
  return true;
}

// CandidateStream::draw (sampling.cpp:64-76) for attempts j0 .. j0+count.
__global__ void gen_kernel(GenParams P, double* __restrict__ cand, double* __restrict__ head,
                           uint8_t* __restrict__ flag) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= P.count) return;
  const uint64_t j = P.j0 + t;
  double c[kMaxDimS];
  double h = 0.0;
  const int d = P.d;
  if (P.kind == GMT_SAMPLE_HALTON) {
    const uint64_t idx = P.start_index + j;
    for (int k = 0; k < d; ++k) c[k] = halton_dev(idx, P.primes[k]);
    if (P.with_heading)
      h = __dmul_rn(__dmul_rn(halton_dev(idx, P.primes[d]), 2.0), 3.14159265358979323846);
  } else {
    uint64_t st = pcg_advance(P.s0, j * static_cast<uint64_t>(P.dd));
    for (int k = 0; k < d; ++k) {
      c[k] = static_cast<double>(pcg_out(st)) * 0x1p-32;  // next_double (rng.hpp:33)
      st = st * kPcgMult + kPcgInc;
    }
    if (P.with_heading)
      h = __dmul_rn(__dmul_rn(static_cast<double>(pcg_out(st)) * 0x1p-32, 2.0), 3.14159265358979323846);
  }
  for (int k = 0; k < d; ++k) cand[static_cast<int64_t>(t) * d + k] = c[k];
  head[t] = h;
  flag[t] = point_free_serial(c, d, P.box_lo, P.box_hi, P.nb) ? 1 : 0;
}

// Single-CTA ordered compaction: rows with flag set are appended, in order,
// at dst[*kept ...] (capacity `cap`); *kept is advanced by the total.
__global__ void __launch_bounds__(1024) compact_rows_kernel(
    const uint8_t* __restrict__ flag, int count, const double* __restrict__ src,
    const double* __restrict__ src_head, int d, double* __restrict__ dst,
    double* __restrict__ dst_head, int* kept, int cap) {
  __shared__ int warp_cnt[32];
  __shared__ int base_s;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
  if (tid == 0) base_s = *kept;
  __syncthreads();
  for (int b0 = 0; b0 < count; b0 += blockDim.x) {
    const int i = b0 + tid;
    const bool f = i < count && flag[i];
    const uint32_t m = __ballot_sync(kFull, f);
    if (lane == 0) warp_cnt[warp] = __popc(m);
    __syncthreads();
    int before = base_s;
    for (int w = 0; w < warp; ++w) before += warp_cnt[w];
    const int slot = before + __popc(m & ((1u << lane) - 1u));
    if (f && slot < cap) {
      for (int k = 0; k < d; ++k) dst[static_cast<int64_t>(slot) * d + k] = src[static_cast<int64_t>(i) * d + k];
      if (dst_head) dst_head[slot] = src_head[i];
    }
    __syncthreads();
    if (tid == 0) {
      int tot = 0;
      for (int w = 0; w < nw; ++w) tot += warp_cnt[w];
      base_s += tot;
    }
    __syncthreads();
  }
  if (tid == 0) *kept = base_s;
}

// Exact-duplicate marks: dup[i] = some j < i has identical coordinates
// (the std::set of sampling.cpp:92,106 holds every earlier kept sample).
__global__ void dup_kernel(const double* __restrict__ F, int from, int to, int d,
                           uint8_t* __restrict__ keep) {
  const int i = from + blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= to) return;
  const double* p = F + static_cast<int64_t>(i) * d;
  bool dup = false;
  for (int j = 0; j < i && !dup; ++j) {
    const double* q = F + static_cast<int64_t>(j) * d;
    bool eq = true;
    for (int k = 0; k < d; ++k) eq = eq && (p[k] == q[k]);
    dup = eq;
  }
  keep[i] = dup ? 0 : 1;
}

// Ordered index list of samples inside the goal box (sampling.cpp:110-112).
__global__ void __launch_bounds__(1024) goal_tag_kernel(const double* __restrict__ coords, int n,
                                                        int d, const double* __restrict__ glo,
                                                        const double* __restrict__ ghi,
                                                        int32_t* __restrict__ goal_idx,
                                                        int* __restrict__ goal_count) {
  __shared__ int warp_cnt[32];
  __shared__ int base_s;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
  if (tid == 0) base_s = 0;
  __syncthreads();
  for (int b0 = 0; b0 < n; b0 += blockDim.x) {
    const int i = b0 + tid;
    const bool f = i < n && box_contains(glo, ghi, d, coords + static_cast<int64_t>(i) * d);
    const uint32_t m = __ballot_sync(kFull, f);
    if (lane == 0) warp_cnt[warp] = __popc(m);
    __syncthreads();
    int before = base_s;
    for (int w = 0; w < warp; ++w) before += warp_cnt[w];
    if (f) goal_idx[before + __popc(m & ((1u << lane) - 1u))] = i;
    __syncthreads();
    if (tid == 0) {
      int tot = 0;
      for (int w = 0; w < nw; ++w) tot += warp_cnt[w];
      base_s += tot;
    }
    __syncthreads();
  }
  if (tid == 0) *goal_count = base_s;
}

struct SubstParams {
  int d;
  int nseen;  // samples 0 .. n-2 stay in `seen` (sampling.cpp:117)
  int nb;
  uint64_t i0;  // first Halton index of the chunk (0 = the goal centre)
  int count;
  const double* coords;
  const double* box_lo;
  const double* box_hi;
  const double* glo;
  const double* ghi;
  uint32_t primes[kMaxDimS];
};

__device__ __forceinline__ void subst_candidate(const SubstParams& P, uint64_t i, double* c) {
  if (i == 0) {  // Aabb::center (space.cpp:18-22)
    for (int k = 0; k < P.d; ++k) c[k] = __dmul_rn(0.5, __dadd_rn(P.glo[k], P.ghi[k]));
  } else {  // lo + q * (hi - lo) (sampling.cpp:122-124)
    for (int k = 0; k < P.d; ++k) {
      const double q = halton_dev(i, P.primes[k]);
      c[k] = __dadd_rn(P.glo[k], __dmul_rn(q, __dsub_rn(P.ghi[k], P.glo[k])));
    }
  }
}

// Goal substitution search (sampling.cpp:115-141): the smallest candidate
// index (0 = centre) that is free and not an exact duplicate of a kept
// sample.  subst_kernel finds the first free candidate of a chunk;
// subst_dup_kernel then checks that one candidate against the kept samples
// (a duplicate is rare: the host resumes the search after it).
__global__ void subst_kernel(SubstParams P, unsigned long long* best) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= P.count) return;
  const uint64_t i = P.i0 + t;
  double c[kMaxDimS];
  subst_candidate(P, i, c);
  if (point_free_serial(c, P.d, P.box_lo, P.box_hi, P.nb)) atomicMin(best, static_cast<unsigned long long>(i));
}

__global__ void subst_dup_kernel(SubstParams P, const unsigned long long* best, int* dup) {
  const unsigned long long i = *best;
  if (i == ~0ull) return;
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= P.nseen) return;
  double c[kMaxDimS];
  subst_candidate(P, i, c);
  const double* q = P.coords + static_cast<int64_t>(j) * P.d;
  bool eq = true;
  for (int k = 0; k < P.d; ++k) eq = eq && (c[k] == q[k]);
  if (eq) *dup = 1;
}

__global__ void subst_write_kernel(SubstParams P, uint64_t i, double* coords, double* head,
                                   int with_heading, uint32_t heading_prime, int slot) {
  double c[kMaxDimS];
  subst_candidate(P, i, c);
  for (int k = 0; k < P.d; ++k) coords[static_cast<int64_t>(slot) * P.d + k] = c[k];
  if (head) {
    head[slot] = (i == 0 || !with_heading)
                     ? 0.0
                     : __dmul_rn(__dmul_rn(halton_dev(i, heading_prime), 2.0), 3.14159265358979323846);
  }
}

// append_init (sampling.cpp:144-154): first exact duplicate, and whether
// the init lies in the goal box.
__global__ void find_init_kernel(const double* __restrict__ coords, const double* __restrict__ head,
                                 int n, int d, const double* __restrict__ init, int has_heading,
                                 double heading, const double* glo, const double* ghi, int* first,
                                 int* in_goal) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i == 0) *in_goal = box_contains(glo, ghi, d, init) ? 1 : 0;
  if (i >= n) return;
  bool eq = true;
  for (int k = 0; k < d; ++k) eq = eq && (coords[static_cast<int64_t>(i) * d + k] == init[k]);
  if (!eq) return;
  const bool same_heading = head ? (has_heading && head[i] == heading) : !has_heading;
  if (same_heading) atomicMin(first, i);
}

}  // namespace

int sample_free_dev(gmt_ctx* ctx, int32_t n, const gmt_scene* scene, const gmt_sample_source* src,
                    Arena& out, DevSamples* S) {
  if (n < 1) return set_error(GMT_E_INVALID_INPUT, "sample count must be >= 1");
  int rc = validate_scene(scene);
  if (rc) return rc;
  if (src->kind != GMT_SAMPLE_HALTON && src->kind != GMT_SAMPLE_UNIFORM)
    return set_error(GMT_E_INVALID_INPUT, "unknown sample kind");
  if (src->kind == GMT_SAMPLE_HALTON && src->start_index == 0)
    return set_error(GMT_E_INVALID_INPUT, "halton start_index is 1-based; got 0");
  const int d = scene->dim, nb = scene->num_boxes;
  if (d > kMaxDimS - 1) return set_error(GMT_E_INVALID_INPUT, "dimension above 15 is not supported");
  const bool heading = src->with_heading != 0;
  const uint64_t budget = 1000ULL * static_cast<uint64_t>(n);
  cudaStream_t s = ctx->stream;

  const int chunk = static_cast<int>(std::min<uint64_t>(std::max<uint64_t>(4ull * n, 8192ull), budget));
  const int cap = n + 1024;  // kept-candidate buffer (dups are rare)
  // device scratch: scene | chunk cand | chunk head | chunk flags | F | Fh | keep | counters
  const size_t o_scene = 0;
  const size_t o_cand = align16(o_scene + sizeof(double) * (2 * static_cast<size_t>(nb) * d + 2 * d));
  const size_t o_head = align16(o_cand + sizeof(double) * static_cast<size_t>(chunk) * d);
  const size_t o_flag = align16(o_head + sizeof(double) * chunk);
  const size_t o_F = align16(o_flag + chunk);
  const size_t o_Fh = align16(o_F + sizeof(double) * static_cast<size_t>(cap) * d);
  const size_t o_keep = align16(o_Fh + sizeof(double) * cap);
  const size_t o_cnt = align16(o_keep + cap);
  const size_t total = align16(o_cnt + 64);
  Arena tmp;
  rc = tmp.reserve(total);
  if (rc) return rc;
  char* base = static_cast<char*>(tmp.ptr);
  double* d_lo = reinterpret_cast<double*>(base + o_scene);
  double* d_hi = d_lo + static_cast<size_t>(nb) * d;
  double* d_glo = d_hi + static_cast<size_t>(nb) * d;
  double* d_ghi = d_glo + d;
  double* cand = reinterpret_cast<double*>(base + o_cand);
  double* chead = reinterpret_cast<double*>(base + o_head);
  uint8_t* flag = reinterpret_cast<uint8_t*>(base + o_flag);
  double* F = reinterpret_cast<double*>(base + o_F);
  double* Fh = reinterpret_cast<double*>(base + o_Fh);
  uint8_t* keep = reinterpret_cast<uint8_t*>(base + o_keep);
  int* d_kept = reinterpret_cast<int*>(base + o_cnt);
  // d_kept[1]: unused slot
  int* d_gcount = d_kept + 2;
  unsigned long long* d_best = reinterpret_cast<unsigned long long*>(base + o_cnt + 16);
  int* d_dup = reinterpret_cast<int*>(base + o_cnt + 24);

  auto fail = [&](int code) {
    tmp.release();
    return code;
  };
#define GMT_CUDA_T(call)                                                 \
  do {                                                                   \
    cudaError_t _e = (call);                                             \
    if (_e != cudaSuccess) return fail(cuda_error(_e, #call));           \
  } while (0)

  if (nb > 0) {
    GMT_CUDA_T(cudaMemcpyAsync(d_lo, scene->box_lo, sizeof(double) * nb * d, cudaMemcpyHostToDevice, s));
    GMT_CUDA_T(cudaMemcpyAsync(d_hi, scene->box_hi, sizeof(double) * nb * d, cudaMemcpyHostToDevice, s));
  }
  GMT_CUDA_T(cudaMemcpyAsync(d_glo, scene->goal_lo, sizeof(double) * d, cudaMemcpyHostToDevice, s));
  GMT_CUDA_T(cudaMemcpyAsync(d_ghi, scene->goal_hi, sizeof(double) * d, cudaMemcpyHostToDevice, s));
  GMT_CUDA_T(cudaMemsetAsync(d_kept, 0, 16, s));

  GenParams P{};
  P.kind = src->kind;
  P.with_heading = heading ? 1 : 0;
  P.d = d;
  P.dd = d + (heading ? 1 : 0);
  P.nb = nb;
  P.start_index = src->start_index;
  P.s0 = pcg_seed_state(src->seed);
  P.box_lo = d_lo;
  P.box_hi = d_hi;
  for (int k = 0; k <= d; ++k) P.primes[k] = nth_prime_h(k + 1);
  const bool need_dedup =
      src->kind == GMT_SAMPLE_UNIFORM || src->start_index + budget >= (1ULL << 53);

  uint64_t j0 = 0;
  int kept = 0, valid = 0, checked = 0;
  while (valid < n) {
    if (j0 >= budget || kept >= cap) {
      return fail(set_error(GMT_E_INFEASIBLE_SAMPLING,
                            "rejection budget of " + std::to_string(budget) +
                                " candidates exhausted after collecting " + std::to_string(valid) +
                                " samples"));
    }
    const int count = static_cast<int>(std::min<uint64_t>(chunk, budget - j0));
    P.j0 = j0;
    P.count = count;
    gen_kernel<<<(count + 255) / 256, 256, 0, s>>>(P, cand, chead, flag);
    GMT_CUDA_T(cudaGetLastError());
    compact_rows_kernel<<<1, 1024, 0, s>>>(flag, count, cand, chead, d, F, Fh, d_kept, cap);
    GMT_CUDA_T(cudaGetLastError());
    ctx->launches += 2;
    GMT_CUDA_T(cudaMemcpyAsync(&kept, d_kept, sizeof(int), cudaMemcpyDeviceToHost, s));
    GMT_CUDA_T(cudaStreamSynchronize(s));
    if (kept > cap) kept = cap;
    if (need_dedup && kept > checked) {
      dup_kernel<<<(kept - checked + 255) / 256, 256, 0, s>>>(F, checked, kept, d, keep);
      GMT_CUDA_T(cudaGetLastError());
      ++ctx->launches;
      std::vector<uint8_t> hk(kept - checked);
      GMT_CUDA_T(cudaMemcpyAsync(hk.data(), keep + checked, kept - checked, cudaMemcpyDeviceToHost, s));
      GMT_CUDA_T(cudaStreamSynchronize(s));
      for (uint8_t v : hk) valid += v;
    } else {
      valid += kept - checked;
    }
    checked = kept;
    j0 += count;
  }

  // Output: the first n valid rows (+1 row of room for append_init).
  const size_t o_oc = 0;
  const size_t o_oh = align16(sizeof(double) * static_cast<size_t>(n + 1) * d);
  const size_t o_og = align16(o_oh + sizeof(double) * (n + 1));
  const size_t out_total = align16(o_og + sizeof(int32_t) * (n + 2));
  rc = out.reserve(out_total);
  if (rc) return fail(rc);
  char* ob = static_cast<char*>(out.ptr);
  S->coords = reinterpret_cast<double*>(ob + o_oc);
  S->heading = heading ? reinterpret_cast<double*>(ob + o_oh) : nullptr;
  S->goal_idx = reinterpret_cast<int32_t*>(ob + o_og);
  S->n = n;
  if (need_dedup) {
    GMT_CUDA_T(cudaMemsetAsync(d_kept, 0, sizeof(int), s));
    compact_rows_kernel<<<1, 1024, 0, s>>>(keep, checked, F, Fh, d, S->coords,
                                           heading ? S->heading : nullptr, d_kept, n);
    GMT_CUDA_T(cudaGetLastError());
    ++ctx->launches;
  } else {
    GMT_CUDA_T(cudaMemcpyAsync(S->coords, F, sizeof(double) * static_cast<size_t>(n) * d,
                               cudaMemcpyDeviceToDevice, s));
    if (heading)
      GMT_CUDA_T(cudaMemcpyAsync(S->heading, Fh, sizeof(double) * n, cudaMemcpyDeviceToDevice, s));
  }
  goal_tag_kernel<<<1, 1024, 0, s>>>(S->coords, n, d, d_glo, d_ghi, S->goal_idx, d_gcount);
  GMT_CUDA_T(cudaGetLastError());
  ++ctx->launches;
  int gcount = 0;
  GMT_CUDA_T(cudaMemcpyAsync(&gcount, d_gcount, sizeof(int), cudaMemcpyDeviceToHost, s));
  GMT_CUDA_T(cudaStreamSynchronize(s));

  if (gcount == 0) {  // goal substitution (sampling.cpp:115-141)
    SubstParams Q{};
    Q.d = d;
    Q.nseen = n - 1;
    Q.nb = nb;
    Q.coords = S->coords;
    Q.box_lo = d_lo;
    Q.box_hi = d_hi;
    Q.glo = d_glo;
    Q.ghi = d_ghi;
    for (int k = 0; k < d; ++k) Q.primes[k] = nth_prime_h(k + 1);
    unsigned long long best = ~0ull;
    for (uint64_t i0 = 0; i0 <= budget && best == ~0ull;) {
      const int count = static_cast<int>(std::min<uint64_t>(4096, budget + 1 - i0));
      Q.i0 = i0;
      Q.count = count;
      GMT_CUDA_T(cudaMemsetAsync(d_best, 0xff, sizeof(unsigned long long), s));
      GMT_CUDA_T(cudaMemsetAsync(d_dup, 0, sizeof(int), s));
      subst_kernel<<<(count + 255) / 256, 256, 0, s>>>(Q, d_best);
      if (Q.nseen > 0) subst_dup_kernel<<<(Q.nseen + 255) / 256, 256, 0, s>>>(Q, d_best, d_dup);
      GMT_CUDA_T(cudaGetLastError());
      ctx->launches += 2;
      int dup = 0;
      GMT_CUDA_T(cudaMemcpyAsync(&best, d_best, sizeof(best), cudaMemcpyDeviceToHost, s));
      GMT_CUDA_T(cudaMemcpyAsync(&dup, d_dup, sizeof(int), cudaMemcpyDeviceToHost, s));
      GMT_CUDA_T(cudaStreamSynchronize(s));
      if (best != ~0ull && dup) {  // a duplicate: resume right after it
        i0 = best + 1;
        best = ~0ull;
      } else {
        i0 += count;
      }
    }
    if (best == ~0ull) {
      return fail(set_error(GMT_E_GOAL_BLOCKED,
                            "no free sample could be placed in the goal region within " +
                                std::to_string(budget) + " candidates"));
    }
    subst_write_kernel<<<1, 1, 0, s>>>(Q, best, S->coords, S->heading, heading ? 1 : 0,
                                       nth_prime_h(d + 1), n - 1);
    GMT_CUDA_T(cudaGetLastError());
    ++ctx->launches;
    const int32_t last = n - 1;
    GMT_CUDA_T(cudaMemcpyAsync(S->goal_idx, &last, sizeof(int32_t), cudaMemcpyHostToDevice, s));
    gcount = 1;
  }
  GMT_CUDA_T(cudaStreamSynchronize(s));
  S->goal_count = gcount;
  tmp.release();
  return GMT_OK;
#undef GMT_CUDA_T
}

int append_init_dev(gmt_ctx* ctx, int dim, DevSamples* S, const double* init, int has_heading,
                    double heading, const double* goal_lo, const double* goal_hi, int32_t* index) {
  cudaStream_t s = ctx->stream;
  Arena tmp;
  int rc = tmp.reserve(sizeof(double) * 3 * dim + 16);
  if (rc) return rc;
  double* d_init = static_cast<double*>(tmp.ptr);
  double* d_glo = d_init + dim;
  double* d_ghi = d_glo + dim;
  int* d_flags = reinterpret_cast<int*>(d_ghi + dim);
  auto fail = [&](int code) {
    tmp.release();
    return code;
  };
#define GMT_CUDA_T(call)                                       \
  do {                                                         \
    cudaError_t _e = (call);                                   \
    if (_e != cudaSuccess) return fail(cuda_error(_e, #call)); \
  } while (0)
  GMT_CUDA_T(cudaMemcpyAsync(d_init, init, sizeof(double) * dim, cudaMemcpyHostToDevice, s));
  GMT_CUDA_T(cudaMemcpyAsync(d_glo, goal_lo, sizeof(double) * dim, cudaMemcpyHostToDevice, s));
  GMT_CUDA_T(cudaMemcpyAsync(d_ghi, goal_hi, sizeof(double) * dim, cudaMemcpyHostToDevice, s));
  const int flags_init[2] = {0x7fffffff, 0};
  GMT_CUDA_T(cudaMemcpyAsync(d_flags, flags_init, sizeof(flags_init), cudaMemcpyHostToDevice, s));
  find_init_kernel<<<(S->n + 255) / 256 + 1, 256, 0, s>>>(S->coords, S->heading, S->n, dim, d_init,
                                                          has_heading, heading, d_glo, d_ghi,
                                                          d_flags, d_flags + 1);
  GMT_CUDA_T(cudaGetLastError());
  ++ctx->launches;
  int flags[2];
  GMT_CUDA_T(cudaMemcpyAsync(flags, d_flags, sizeof(flags), cudaMemcpyDeviceToHost, s));
  GMT_CUDA_T(cudaStreamSynchronize(s));
  if (flags[0] != 0x7fffffff) {
    *index = flags[0];
    tmp.release();
    return GMT_OK;
  }
  const int idx = S->n;
  GMT_CUDA_T(cudaMemcpyAsync(S->coords + static_cast<int64_t>(idx) * dim, d_init,
                             sizeof(double) * dim, cudaMemcpyDeviceToDevice, s));
  if (S->heading)
    GMT_CUDA_T(cudaMemcpyAsync(S->heading + idx, &heading, sizeof(double), cudaMemcpyHostToDevice, s));
  if (flags[1]) {
    GMT_CUDA_T(cudaMemcpyAsync(S->goal_idx + S->goal_count, &idx, sizeof(int32_t),
                               cudaMemcpyHostToDevice, s));
    S->goal_count += 1;
  }
  GMT_CUDA_T(cudaStreamSynchronize(s));
  S->n = idx + 1;
  *index = idx;
  tmp.release();
  return GMT_OK;
#undef GMT_CUDA_T
}

}  // namespace gmtb

using namespace gmtb;

extern "C" int gmt_sample_free(gmt_ctx* ctx, int32_t n, const gmt_scene* scene,
                               const gmt_sample_source* src, double* coords_out,
                               double* heading_out, int32_t* goal_idx_out,
                               int32_t* goal_count_out) {
  gmtb::AllocScope alloc_scope_(ctx);
  Arena out;
  DevSamples S;
  int rc = sample_free_dev(ctx, n, scene, src, out, &S);
  if (rc) return rc;
  const int d = scene->dim;
  cudaStream_t s = ctx->stream;
  GMT_CUDA(cudaMemcpyAsync(coords_out, S.coords, sizeof(double) * static_cast<size_t>(n) * d,
                           cudaMemcpyDeviceToHost, s));
  if (heading_out && S.heading)
    GMT_CUDA(cudaMemcpyAsync(heading_out, S.heading, sizeof(double) * n, cudaMemcpyDeviceToHost, s));
  GMT_CUDA(cudaMemcpyAsync(goal_idx_out, S.goal_idx, sizeof(int32_t) * S.goal_count,
                           cudaMemcpyDeviceToHost, s));
  GMT_CUDA(cudaStreamSynchronize(s));
  *goal_count_out = S.goal_count;
  out.release();
  return GMT_OK;
}

extern "C" int gmt_append_init(gmt_ctx* ctx, int32_t dim, double* coords, double* heading,
                               int32_t* n, const double* init, int32_t init_has_heading,
                               double init_heading, const double* goal_lo, const double* goal_hi,
                               int32_t* goal_idx, int32_t* goal_count, int32_t* index_out) {
  gmtb::AllocScope alloc_scope_(ctx);
  const int n0 = *n;
  Arena buf;
  int rc = buf.reserve(align16(sizeof(double) * (n0 + 1) * dim) + sizeof(double) * (n0 + 1) +
                       sizeof(int32_t) * (*goal_count + 2) + 64);
  if (rc) return rc;
  DevSamples S;
  char* b = static_cast<char*>(buf.ptr);
  S.coords = reinterpret_cast<double*>(b);
  b += align16(sizeof(double) * (n0 + 1) * dim);
  S.heading = heading ? reinterpret_cast<double*>(b) : nullptr;
  b += align16(sizeof(double) * (n0 + 1));
  S.goal_idx = reinterpret_cast<int32_t*>(b);
  S.n = n0;
  S.goal_count = *goal_count;
  cudaStream_t s = ctx->stream;
  GMT_CUDA(cudaMemcpyAsync(S.coords, coords, sizeof(double) * n0 * dim, cudaMemcpyHostToDevice, s));
  if (heading) GMT_CUDA(cudaMemcpyAsync(S.heading, heading, sizeof(double) * n0, cudaMemcpyHostToDevice, s));
  rc = append_init_dev(ctx, dim, &S, init, init_has_heading, init_heading, goal_lo, goal_hi, index_out);
  if (rc) {
    buf.release();
    return rc;
  }
  if (S.n > n0) {
    GMT_CUDA(cudaMemcpyAsync(coords + static_cast<int64_t>(n0) * dim, S.coords + static_cast<int64_t>(n0) * dim,
                             sizeof(double) * dim, cudaMemcpyDeviceToHost, s));
    if (heading) GMT_CUDA(cudaMemcpyAsync(heading + n0, S.heading + n0, sizeof(double), cudaMemcpyDeviceToHost, s));
    if (S.goal_count > *goal_count)
      GMT_CUDA(cudaMemcpyAsync(goal_idx + *goal_count, S.goal_idx + *goal_count, sizeof(int32_t),
                               cudaMemcpyDeviceToHost, s));
    GMT_CUDA(cudaStreamSynchronize(s));
  }
  *n = S.n;
  *goal_count = S.goal_count;
  buf.release();
  return GMT_OK;
}

// build_instance (problem.cpp:336-363): sample -> append init -> radius ->
// graph, every step on the device; the instance keeps its goal list.
static int instance_build(gmt_ctx* ctx, const gmt_problem* p, const char* cache_file,
                          gmt_instance** out, int32_t* cache_hit) {
  *out = nullptr;
  if (cache_hit) *cache_hit = 0;
  const gmt_scene* scene = &p->scene;
  const int d = scene->dim, nb = scene->num_boxes;
  int rc = validate_scene(scene);
  if (rc) return rc;
  const bool dubins = p->steering == GMT_STEER_DUBINS_AIRPLANE;
  // build_instance samples headings exactly for Dubins problems (problem.cpp:338-339).
  gmt_sample_source src = p->sampling;
  src.with_heading = dubins ? 1 : 0;
  if (dubins) {
    rc = validate_dubins(&p->dubins, d);
    if (rc) return rc;
  }
  Arena samples;
  DevSamples S;
  rc = sample_free_dev(ctx, p->n, scene, &src, samples, &S);
  if (rc) return rc;
  int32_t init_index = -1;
  rc = append_init_dev(ctx, d, &S, p->init, p->init_has_heading, p->init_heading, scene->goal_lo,
                       scene->goal_hi, &init_index);
  if (rc) {
    samples.release();
    return rc;
  }
  const bool quad = p->steering == GMT_STEER_QUADROTOR;
  const bool di = p->steering == GMT_STEER_DOUBLE_INTEGRATOR || quad;  // kinodynamic, directed
  if (p->steering != GMT_STEER_EUCLIDEAN && !di && !dubins) {
    samples.release();
    return set_error(GMT_E_INVALID_INPUT, "unsupported steering model");
  }
  double radius = p->radius_override;
  if (!(radius > 0.0)) {
    if (di) {  // the Theorem 1 radius assumes straight-line costs
      samples.release();
      return set_error(GMT_E_INVALID_INPUT,
                       "kinodynamic steering needs radius_override (a cost threshold)");
    }
    rc = gmt_connection_radius(d, p->n, p->eta, 1.0 /* free_measure_upper_bound, space.cpp:101-104 */,
                               &radius);
    if (rc) {
      samples.release();
      return rc;
    }
  }
  Arena g, g2, g3;
  DubinsGraphPaths dpaths;
  int64_t E = 0, *rp = nullptr;
  int32_t* col = nullptr;
  double* cost = nullptr;
  DiRows dout, din;
  // Graph cache (problem.cpp:354-360): a key / shape match supplies the graph.
  bool hit = false;
  uint64_t key = 0;
  std::vector<int64_t> hp;
  std::vector<int32_t> hc;
  std::vector<double> hw;
  if (cache_file) {
    if (di) {
      samples.release();
      return set_error(GMT_E_INVALID_INPUT,
                       "the graph cache covers the reference's steering models (Euclidean, Dubins airplane)");
    }
    rc = problem_key_of(p, &key);
    if (rc == GMT_OK) rc = cache_read(cache_file, key, S.n, radius, hp, hc, hw, &hit, cache_model_of(p));
    if (rc == GMT_OK && hit && !dubins) {  // (a Dubins hit: rows go through the Dubins builder below)
      E = static_cast<int64_t>(hc.size());
      const size_t o_col = align16(sizeof(int64_t) * (S.n + 1));
      const size_t o_cost = o_col + align16(sizeof(int32_t) * static_cast<size_t>(E));
      rc = g.reserve(o_cost + sizeof(double) * static_cast<size_t>(E) + 16);
      if (rc == GMT_OK) {
        char* b = static_cast<char*>(g.ptr);
        rp = reinterpret_cast<int64_t*>(b);
        col = reinterpret_cast<int32_t*>(b + o_col);
        cost = reinterpret_cast<double*>(b + o_cost);
        cudaStream_t s0 = ctx->stream;
        cudaError_t e = cudaMemcpyAsync(rp, hp.data(), sizeof(int64_t) * hp.size(), cudaMemcpyHostToDevice, s0);
        if (e == cudaSuccess && E)
          e = cudaMemcpyAsync(col, hc.data(), sizeof(int32_t) * E, cudaMemcpyHostToDevice, s0);
        if (e == cudaSuccess && E)
          e = cudaMemcpyAsync(cost, hw.data(), sizeof(double) * E, cudaMemcpyHostToDevice, s0);
        if (e == cudaSuccess) e = cudaStreamSynchronize(s0);
        if (e != cudaSuccess) rc = cuda_error(e, "graph cache upload");
      }
    }
    if (rc) {
      samples.release();
      g.release();
      return rc;
    }
  }
  if (hit && !dubins) {
    // graph supplied by the cache file
  } else if (dubins) {
    const HostRows cached{&hp, &hc, &hw};  // a cache hit: rows and costs from the file, paths recomputed
    rc = build_dubins_graph_dev(ctx, S.coords, S.heading, S.n, d, &p->dubins, radius, g, &dout, g2, &din, g3,
                                &dpaths, hit ? &cached : nullptr);
    E = dout.edges;
    rp = dout.ptr;
    col = dout.col;
    cost = dout.cost;
  } else if (di) {
    if (d != (quad ? kQuadDim : kDiDim)) {
      samples.release();
      return set_error(GMT_E_INVALID_INPUT, quad ? "the quadrotor needs dimension 12"
                                                 : "the double integrator needs dimension 6");
    }
    if (quad) {
      rc = validate_quad(&p->quad);
      if (rc == GMT_OK) rc = build_quad_graph_dev(ctx, S.coords, S.n, &p->quad, radius, g, &dout, g2, &din);
    } else {
      rc = validate_di(&p->di);
      if (rc == GMT_OK) rc = build_di_graph_dev(ctx, S.coords, S.n, &p->di, radius, g, &dout, g2, &din);
    }
    E = dout.edges;
    rp = dout.ptr;
    col = dout.col;
    cost = dout.cost;
  } else {
    rc = build_graph_dev(ctx, S.coords, S.n, d, radius, g, &E, &rp, &col, &cost);
  }
  if (rc) {
    samples.release();
    g.release();
    g2.release();
    g3.release();
    return rc;
  }
  auto* inst = new gmt_instance;
  const int n = S.n;
  const size_t o_coords = 0;
  const size_t o_lo = align16(o_coords + sizeof(double) * static_cast<size_t>(n) * d);
  const size_t o_hi = align16(o_lo + sizeof(double) * static_cast<size_t>(nb) * d);
  const size_t o_glo = align16(o_hi + sizeof(double) * static_cast<size_t>(nb) * d);
  const size_t o_ghi = align16(o_glo + sizeof(double) * d);
  const size_t o_gidx = align16(o_ghi + sizeof(double) * d);
  const size_t total = align16(o_gidx + sizeof(int32_t) * (S.goal_count + 1));
  rc = inst->aux.reserve(total);
  cudaStream_t s = ctx->stream;
  if (rc == GMT_OK) {
    char* b = static_cast<char*>(inst->aux.ptr);
    cudaError_t e = cudaMemcpyAsync(b + o_coords, S.coords, sizeof(double) * n * d, cudaMemcpyDeviceToDevice, s);
    if (e == cudaSuccess && nb > 0)
      e = cudaMemcpyAsync(b + o_lo, scene->box_lo, sizeof(double) * nb * d, cudaMemcpyHostToDevice, s);
    if (e == cudaSuccess && nb > 0)
      e = cudaMemcpyAsync(b + o_hi, scene->box_hi, sizeof(double) * nb * d, cudaMemcpyHostToDevice, s);
    if (e == cudaSuccess)
      e = cudaMemcpyAsync(b + o_glo, scene->goal_lo, sizeof(double) * d, cudaMemcpyHostToDevice, s);
    if (e == cudaSuccess)
      e = cudaMemcpyAsync(b + o_ghi, scene->goal_hi, sizeof(double) * d, cudaMemcpyHostToDevice, s);
    if (e == cudaSuccess)
      e = cudaMemcpyAsync(b + o_gidx, S.goal_idx, sizeof(int32_t) * S.goal_count, cudaMemcpyDeviceToDevice, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) rc = cuda_error(e, "instance assembly");
    DevInstance& D = inst->desc;
    D = DevInstance{};
    D.n = n;
    D.dim = d;
    D.num_boxes = nb;
    D.directed = 0;
    D.goal_count = S.goal_count;
    D.init_index = init_index;
    D.radius = radius;
    D.num_edges = E;
    D.coords = reinterpret_cast<const double*>(b + o_coords);
    D.box_lo = reinterpret_cast<const double*>(b + o_lo);
    D.box_hi = reinterpret_cast<const double*>(b + o_hi);
    D.goal_lo = reinterpret_cast<const double*>(b + o_glo);
    D.goal_hi = reinterpret_cast<const double*>(b + o_ghi);
    D.out_ptr = rp;
    D.out_col = col;
    D.out_cost = cost;
    D.in_ptr = rp;
    D.in_col = col;
    D.in_cost = cost;
    if (di) {
      D.directed = 1;
      D.in_ptr = din.ptr;
      D.in_col = din.col;
      D.in_cost = din.cost;
      D.in_tau = din.tau;
      D.out_tau = dout.tau;
      D.steering = p->steering;
      if (quad) {
        D.kin_segments = p->quad.segments;
        D.kin_p[0] = p->quad.g;
        D.kin_p[1] = p->quad.vmax;
        D.kin_p[2] = p->quad.amax;
        D.kin_p[3] = p->quad.ymax;
        D.kin_p[4] = p->quad.wmax;
        D.kin_p[5] = p->quad.weight;
      } else {
        D.kin_segments = p->di.segments;
        D.kin_p[0] = p->di.vmax;
        D.kin_p[1] = p->di.weight;
      }
      // The checks read build-time waypoint tables, as the reference's
      // planner reads the polyline cached with every edge (graph.cpp
      // edge_path): single solves 2.13 -> 0.63 ms (quadrotor n = 8000),
      // 0.198 -> 0.178 ms (double integrator n = 4000).  GMT_KINO_TABLES=0
      // regenerates every checked trajectory in the solve instead.
      const char* kt = std::getenv("GMT_KINO_TABLES");
      const bool tables = kt ? std::atoi(kt) != 0 : true;
      const int W = (D.kin_segments + 1) * d;
      if (rc == GMT_OK && tables && W <= 144 && din.edges > 0) {
        rc = inst->mem4.reserve(sizeof(double) * static_cast<size_t>(W) * din.edges);
        if (rc == GMT_OK) {
          double* wp = static_cast<double*>(inst->mem4.ptr);
          cudaError_t e = launch_kino_tables(D.coords, din.ptr, din.col, din.tau, n, p->steering, to_quad(&p->quad),
                                             to_di(&p->di), wp, ctx->sm_count, s);
          ++ctx->launches;
          if (e != cudaSuccess) rc = cuda_error(e, "kinodynamic waypoint tables");
          D.in_wp = wp;
        }
      }
    }
    if (dubins) {
      D.directed = 1;
      D.in_ptr = din.ptr;
      D.in_col = din.col;
      D.in_cost = din.cost;
      D.in_path = dpaths.in_path;
      D.out_path = dpaths.out_path;
      D.path_ptr = dpaths.path_ptr;
      D.path_pts = dpaths.pts;
      D.steering = GMT_STEER_DUBINS_AIRPLANE;
    }
    inst->goal_idx_dev = reinterpret_cast<const int32_t*>(b + o_gidx);
    inst->graph_n = n;
    inst->cache_model = cache_model_of(p);
  }
  samples.release();
  if (rc == GMT_OK) {
    inst->mem = g;  // the graph arenas now belong to the instance
    g.ptr = nullptr;
    inst->mem2 = g2;
    g2.ptr = nullptr;
    inst->mem3 = g3;
    g3.ptr = nullptr;
    rc = push_desc(ctx, inst);
    if (rc == GMT_OK) {
      cudaError_t e = cudaStreamSynchronize(s);
      if (e != cudaSuccess) rc = cuda_error(e, "instance build");
    }
  }
  if (rc != GMT_OK) {
    g.release();
    g2.release();
    g3.release();
    delete inst;
    return rc;
  }
  if (cache_file && !hit) {
    // save_graph_cache's result is ignored by build_instance (problem.cpp:361).
    if (gmt_instance_cache_save(ctx, inst, cache_file, key) != GMT_OK) g_last_error.clear();
  }
  if (cache_hit) *cache_hit = hit ? 1 : 0;
  *out = inst;
  return GMT_OK;
}

extern "C" int gmt_instance_build(gmt_ctx* ctx, const gmt_problem* p, gmt_instance** out) {
  gmtb::AllocScope alloc_scope_(ctx);
  return instance_build(ctx, p, nullptr, out, nullptr);
}

extern "C" int gmt_instance_build_cached(gmt_ctx* ctx, const gmt_problem* p, const char* cache_file,
                                         gmt_instance** out, int32_t* cache_hit) {
  gmtb::AllocScope alloc_scope_(ctx);
  if (!cache_file) return set_error(GMT_E_INVALID_INPUT, "gmt_instance_build_cached: null cache file");
  return instance_build(ctx, p, cache_file, out, cache_hit);
}
