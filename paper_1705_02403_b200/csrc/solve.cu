// solve.cu -- the GMT* online phase (gmt_plan, planner.cpp:94-198; fmt_plan,
// planner.cpp:200-262) as ONE persistent kernel launch per query (or per
// batch of queries).
//
// Execution model:
//   * A query is solved by a thread-block cluster of CS CTAs (CS = 1 for
//     batched solves, up to 16 for a single latency-critical query).
//   * Every CTA keeps a full replica of the wavefront in shared memory:
//     cost f64[V] plus open/closed/group bitmasks.  Phases P0-P3 of the
//     reference pass (min-open, fast-forward, group, goal test) therefore run
//     redundantly and locally in every CTA with no communication.
//   * Ownership is word-interleaved: node v belongs to CTA (v/32) mod CS.
//   * P4 (candidate gather): each CTA expands the group members it owns; the
//     lanes stream an out-row (sorted targets), OR the unexplored targets of
//     each 32-node word together with a segmented shuffle scan over the
//     sorted run, and one lane per word sets the bits in the owner's
//     candidate bitmask (a DSMEM atomic when the owner is another CTA).
//   * P5 (connect_candidate) runs warp-per-candidate on the owner CTA: the
//     lanes stream the candidate's in-row (col/cost, coalesced, 4 chunks in
//     flight per lane, next row's offsets prefetched), gather cost[y]/open(y)
//     from the local replica, reduce (cost, position) lexicographically with
//     three REDUX.MIN steps (== the reference's strict-< first-in-list rule),
//     then slab-test the single best edge: endpoints staged in shared memory,
//     boxes spread over the lanes, an exact-safe bounding-box separation test
//     in registers before the division-based clip.
//   * P6 (commit) writes the new cost into every replica (DSMEM stores) and
//     sets a `newopen` bit; labels only change at the next pass start, so
//     every candidate sees iteration-start labels exactly as in the
//     reference's parallel map + serial commit.
//   * Two cluster barriers per pass; no host round trip until the answer.
// The kernel is specialised on the dimension D (0 = any d <= 16) so the
// per-axis loops of the geometry unroll into registers.
#include <cooperative_groups.h>

#include <algorithm>
#include <cstdint>
#include <mutex>
#include <type_traits>

#include "common.cuh"
#include "di.cuh"
#include "quad.cuh"
#include "gmt_b200.h"
#include "solve.cuh"

namespace cg = cooperative_groups;

namespace gmtb {

namespace {

constexpr uint32_t kFull = 0xffffffffu;
constexpr int32_t kNone = 0x7fffffff;
// Row chunks in flight per lane: batched solves cover a typical in-row
// (~130 edges for C2) in one round with 16 lanes x 8; clusters use 32 lanes.
#ifndef GMT_UNROLL_BATCH
#define GMT_UNROLL_BATCH 8
#endif
#ifndef GMT_UNROLL_CLUSTER
#define GMT_UNROLL_CLUSTER 4
#endif
constexpr double kSepMargin = 1e-9;  // see segment_free_staged
#ifndef GMT_ROWS_PER_WARP
#define GMT_ROWS_PER_WARP 2
#endif
#ifndef GMT_ROWS_CLUSTER
#define GMT_ROWS_CLUSTER 1
#endif


// Longest of the rows the kRows lane groups of a warp are streaming.
template <int kRows>
__device__ __forceinline__ int rows_max(int len) {
  if constexpr (kRows == 1) {
    return len;
  } else if constexpr (kRows == 2) {
    const int other = __shfl_xor_sync(0xffffffffu, len, 16);
    return len > other ? len : other;
  } else {
    return static_cast<int>(__reduce_max_sync(0xffffffffu, static_cast<uint32_t>(len)));
  }
}

struct CtaShared {
  double red_min[32];
  double red_goal_c[32];
  int32_t red_goal_v[32];
  int32_t group_count;
  int32_t own_count;  // group members this CTA expands in P4
  int32_t cand_count;
  int32_t next_own;   // dynamic work distribution (clusters): next P4 row group
  int32_t next_cand;  // next P5 candidate group
  unsigned long long checks_acc;  // rank 0: cluster-wide checks of this pass
  int32_t added_acc;              // rank 0: cluster-wide additions of this pass
  int32_t feasible;
  int32_t vfull;  // D = 6: every box spans [0, 1] on the three velocity axes
  // (the 24-warp D = 6 shape) boxes staged in ascending lo_x order, and the
  // widest staged x extent him_x - lom_x rounded up: the edge cull scans
  // only the boxes whose lom_x lies in [pmn_x - wx, pmx_x]
  int32_t xsorted;
  double box_wx;
  const uint16_t* xfirst;  // x buckets of the sorted boxes (or null)
  // Loop state kept in shared memory rather than in every thread's
  // registers (the solve is register-bound): the threshold index i, the
  // pass number, the running check total (tid 0), per-warp check / commit
  // counts and the traffic counters.
  long long iter;
  long long total_checks;
  int32_t pass;
  int32_t wchecks[32];
  int32_t wadded[32];
  unsigned long long cnt_in, cnt_out;
};

// Boxes: box b, axis k at base[b*bs + k*as].  lom/him hold lo - m and
// hi + m (the separation bounds) when the boxes are staged in shared memory.
// idx (may be null): box i of this view is box idx[i] of the arrays (a
// per-edge list of the boxes that survive the polyline's bounding box).
// full (may be null): per box, the axes k with lo <= 0 and hi >= 1.  Once
// both endpoints are known to lie in the unit cube such an axis can neither
// separate a segment from the box nor narrow its slab interval: its clamped
// interval is [0, 1] (fl(lo - a) <= 0 <= a and fl(hi - a) >= fl(b - a) by
// monotone rounding), and dk == 0 leaves a inside [lo, hi].
struct Boxes {
  const double* lo;
  const double* hi;
  const double* lom;
  const double* him;
  const uint16_t* idx;
  const uint32_t* full;
  int bs;
  int as;
  int count;
};

template <int CS>
__device__ __forceinline__ void cluster_barrier() {
  if constexpr (CS > 1) {
    cg::this_cluster().sync();
  } else {
    __syncthreads();
  }
}

template <int CS, typename T>
__device__ __forceinline__ T* remote(T* p, int rank) {
  if constexpr (CS > 1) {
    return cg::this_cluster().map_shared_rank(p, rank);
  } else {
    return p;
  }
}

template <int D>
__device__ __forceinline__ int dims(int rt) {
  return D > 0 ? D : rt;
}

// Bulk prefetch of a byte range into L2 by the TMA engine
// (cp.async.bulk.prefetch.L2, sm_90+): one instruction per range, no
// registers, no completion to wait for.  The range is widened to 16-byte
// alignment as the instruction requires.
__device__ __forceinline__ void prefetch_l2(const void* p, size_t bytes) {
  if (bytes == 0) return;
  const uintptr_t a = reinterpret_cast<uintptr_t>(p) & ~static_cast<uintptr_t>(15);
  const uintptr_t e = (reinterpret_cast<uintptr_t>(p) + bytes + 15) & ~static_cast<uintptr_t>(15);
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(a),
               "r"(static_cast<uint32_t>(e - a))
               : "memory");
}


// x buckets of the sorted boxes (the 24-warp DI shape): xfirst[b] = the
// number of boxes whose lo_x - m lies below kXB0 + b * kXBW (b = 0: none,
// b = kXB: all), so a check's x window [lo_t, hi_t] maps to a conservative
// index range with two shared-memory loads (a bucket of slack either side
// absorbs the rounding of the bucket index).
constexpr int kXB = 256;
constexpr double kXB0 = -1.0, kXBW = 2.5 / kXB;
__device__ __forceinline__ int xbucket(double x) {
  double f = (x - kXB0) * (1.0 / kXBW);
  f = f < -4.0 ? -4.0 : (f > kXB + 4.0 ? kXB + 4.0 : f);
  return __double2int_rd(f);
}

// One 8-byte global -> shared copy that holds no register (LDGSTS), and the
// wait for this thread's copies.
__device__ __forceinline__ void cp_async8(void* smem_dst, const void* gsrc) {
  const uint32_t d = static_cast<uint32_t>(__cvta_generic_to_shared(smem_dst));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(d), "l"(gsrc) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

// A pointer into the dynamic shared memory rebased on the extern array, so
// the compiler sees its address space and loads through it are LDS (short
// scoreboard) instead of generic LD.  (The staged boxes' pointers are read
// back from the shared Boxes descriptor, which loses that information.)
extern __shared__ __align__(16) unsigned char gmt_dyn_smem[];
template <typename T>
__device__ __forceinline__ const T* shared_view(const T* p) {
  const uint32_t a = static_cast<uint32_t>(__cvta_generic_to_shared(p));
  const uint32_t b = static_cast<uint32_t>(__cvta_generic_to_shared(gmt_dyn_smem));
  return reinterpret_cast<const T*>(gmt_dyn_smem + static_cast<int32_t>(a - b));
}

// Closed box b contains p (Aabb::contains, space.cpp:11-16).
template <int D>
__device__ __forceinline__ bool box_has(const double* p, int d_rt, const Boxes& bx, int b) {
  const int d = dims<D>(d_rt);
  bool in = true;
#pragma unroll
  for (int k = 0; k < (D > 0 ? D : kMaxSolveDim); ++k) {
    if (D > 0 || k < d) {
      const double x = p[k];
      in = in && !(x < bx.lo[b * bx.bs + k * bx.as] || x > bx.hi[b * bx.bs + k * bx.as]);
    }
  }
  return in;
}

// Any box contains p (the loop of point_free, space.cpp:50-52), boxes spread
// over the lanes.  p is warp-uniform (shared memory).
template <int D>
__device__ __forceinline__ bool any_box_contains(const double* p, int d, const Boxes& bx, int lane) {
  bool in = false;
  for (int b = lane; b < bx.count && !in; b += kWarp) in = box_has<D>(p, d, bx, b);
  return __any_sync(kFull, in);
}

// segment_free (space.cpp:80-90) of the segment staged in the warp's `seg`
// scratch (a = seg[0..15], b = seg[16..31]).  Coordinate predicates run
// lane-per-axis, boxes lane-per-box.
//
// Exact-safe separation pre-test (no division): if on some axis both
// endpoints lie below lo - m or above hi + m (m = 1e-9), the reference's
// floating-point slab clip (space.cpp:60-78) reports a miss.  Proof sketch:
// a, b are in the unit cube here, so |dk| <= 1.  For b < a < lo - m or
// b > a > hi + m both rounded slab parameters are strictly negative; for
// a < b < lo - m or a > b > hi + m both exceed
// (1 + m)(1 - 2^-53)/(1 + 2^-53) > 1; either way tmin > tmax on that axis.
// The clip's outcome does not depend on the axis order (the running max/min
// of the slab ends are order-free and emptiness is monotone), and dk == 0
// is the clip's own early miss.  (fl(lo - m) differs from lo - m by at most
// 2^-53 |lo|, which only matters for |lo| > 1 where lo - b > 1 anyway.)
// Boxes that pass the pre-test go through the exact clip.
template <int D>
__device__ bool segment_free_ab(int d_rt, const Boxes& bx, int lane, const double* a, const double* b) {
  const int d = dims<D>(d_rt);
  bool eq = true, cube_a = true, cube_b = true;
  if (lane < d) {
    const double x = a[lane], y = b[lane];
    eq = x == y;
    cube_a = !(x < 0.0 || x > 1.0);
    cube_b = !(y < 0.0 || y > 1.0);
  }
  const bool same = __all_sync(kFull, eq);
  const bool in_a = __all_sync(kFull, cube_a);
  if (same) return in_a && !any_box_contains<D>(a, d, bx, lane);  // point_free(a)
  if (!in_a || !__all_sync(kFull, cube_b)) return false;
  // Segment bounding box: registers for a fixed small dimension, the staged
  // endpoints otherwise.
  constexpr int kReg = (D > 0 && D <= 6) ? D : 1;
  double mn[kReg], mx[kReg];
  if constexpr (D > 0 && D <= 6) {
#pragma unroll
    for (int k = 0; k < D; ++k) {
      const double x = a[k], y = b[k];
      mn[k] = x < y ? x : y;
      mx[k] = x < y ? y : x;
    }
  }
  // Boxes that survive the pre-test are clipped lane-parallel: lane
  // (slot, axis) computes one axis' slab interval of the slot-th surviving
  // box, and the d lanes of a slot combine max(0, t0_k) / min(1, t1_k) and
  // the dk == 0 misses.  The clip's result is a function of those order-free
  // max/min values, so this equals the reference's sequential axis loop.
  // (Running this scan on shared_view pointers when the boxes are staged --
  // LDS instead of generic loads -- made the 3D forest batch 2 % faster but,
  // as a second inlined copy, the configs[4] solves 1.5-7 % slower.)
  const int per = kWarp / d;
  const int slot = lane / d, axis = lane - slot * d;
  bool hit = false;
  for (int i0 = 0; i0 < bx.count && !hit; i0 += kWarp) {
    const int i = i0 + lane;
    bool sep = i >= bx.count;
    int ic = sep ? bx.count - 1 : i;  // idle lanes read a valid box
    if (bx.idx) ic = bx.idx[ic];
#pragma unroll
    for (int k = 0; k < (D > 0 ? D : kMaxSolveDim); ++k) {
      if (D == 0 && k >= d) break;
      double lo_k, hi_k;
      if (bx.lom) {
        lo_k = bx.lom[ic * bx.bs + k * bx.as];
        hi_k = bx.him[ic * bx.bs + k * bx.as];
      } else {
        lo_k = bx.lo[ic * bx.bs + k * bx.as] - kSepMargin;
        hi_k = bx.hi[ic * bx.bs + k * bx.as] + kSepMargin;
      }
      double smin, smax;
      if constexpr (D > 0 && D <= 6) {
        smin = mn[k];
        smax = mx[k];
      } else {
        const double x = a[k], y = b[k];
        smin = x < y ? x : y;
        smax = x < y ? y : x;
      }
      sep = sep || smax < lo_k || smin > hi_k;
    }
    uint32_t cm = __ballot_sync(kFull, !sep);
    while (cm) {
      const int nc = __popc(cm);
      const int take = nc < per ? nc : per;
      bool miss = false;
      double t0 = 0.0, t1 = 1.0;
      if (slot < take) {
        uint32_t mm = cm;  // the slot-th surviving box (slot < take, usually 0-2)
        for (int t = 0; t < slot; ++t) mm &= mm - 1u;
        int bi = i0 + __ffs(mm) - 1;
        if (bx.idx) bi = bx.idx[bi];
        const double ak = a[axis];
        const double dk = __dsub_rn(b[axis], ak);
        const double l = bx.lo[bi * bx.bs + axis * bx.as], h = bx.hi[bi * bx.bs + axis * bx.as];
        if (dk == 0.0) {
          miss = ak < l || ak > h;
        } else {
          t0 = __ddiv_rn(__dsub_rn(l, ak), dk);
          t1 = __ddiv_rn(__dsub_rn(h, ak), dk);
          if (t0 > t1) {
            const double t = t0;
            t0 = t1;
            t1 = t;
          }
          // The clip starts from tmin = 0, tmax = 1 (space.cpp:62-63):
          // clamp this axis' slab ends to the segment's own parameter range.
          t0 = (0.0 < t0) ? t0 : 0.0;  // std::max(0.0, t0)
          t1 = (t1 < 1.0) ? t1 : 1.0;  // std::min(1.0, t1)
        }
      }
      // Slot leaders (axis 0) fold in the other d - 1 axes' own values.
      double tmin = t0, tmax = t1;
      bool m = miss;
      const int mi = miss ? 1 : 0;
      for (int o = 1; o < d; ++o) {
        const double u0 = __shfl_down_sync(kFull, t0, o);
        const double u1 = __shfl_down_sync(kFull, t1, o);
        const int um = __shfl_down_sync(kFull, mi, o);
        tmin = (tmin < u0) ? u0 : tmin;
        tmax = (u1 < tmax) ? u1 : tmax;
        m = m || um != 0;
      }
      hit = __any_sync(kFull, axis == 0 && slot < take && !m && !(tmin > tmax));
      if (hit || take == nc) break;
      for (int t = 0; t < take; ++t) cm &= cm - 1u;  // drop the `take` boxes done
    }
  }
  return !hit;
}

template <int D>
__device__ __forceinline__ bool segment_free_staged(int d_rt, const Boxes& bx, int lane, const double* seg) {
  return segment_free_ab<D>(d_rt, bx, lane, seg, seg + 16);
}

template <int D>
__device__ bool segment_free_warp(const double* A, const double* B, int d, const Boxes& bx,
                                  int lane, double* seg) {
  __syncwarp();
  if (lane < d) seg[lane] = A[lane];
  if (lane >= 16 && lane - 16 < d) seg[lane] = B[lane - 16];
  __syncwarp();
  return segment_free_staged<D>(d, bx, lane, seg);
}

template <int D>
__device__ bool point_free_warp(const double* P, int d, const Boxes& bx, int lane, double* seg) {
  __syncwarp();
  if (lane < d) seg[lane] = P[lane];
  __syncwarp();
  bool cube = true;
  if (lane < d) cube = !(seg[lane] < 0.0 || seg[lane] > 1.0);
  if (!__all_sync(kFull, cube)) return false;
  return !any_box_contains<D>(seg, d, bx, lane);
}

// motion_free (planner.cpp:54-60) for a path edge: the cached polyline,
// every sub-segment through the exact test (polyline_free, space.cpp:92-99).
template <int D>
__device__ bool polyline_free_warp(const DevInstance& I, int d, const Boxes& bx, int32_t pid,
                                   int lane, double* seg) {
  const int64_t a = I.path_ptr[pid], b = I.path_ptr[pid + 1];
  const double* pts = I.path_pts + a * d;
  if (b - a == 1) return point_free_warp<D>(pts, d, bx, lane, seg);
  for (int64_t s = 0; s + 1 < b - a; ++s) {
    if (!segment_free_warp<D>(pts + s * d, pts + (s + 1) * d, d, bx, lane, seg)) return false;
  }
  return true;
}

// segment_hits_box (space.cpp:60-78) of one segment against one box on a
// single lane: the exact-safe separation pre-test of segment_free_ab, then
// the reference's sequential closed slab clip (tmin = 0, tmax = 1).
// POS3: every box spans [0, 1] on axes 3.. (the DI velocity axes when the
// solve's vfull holds): only the three position axes can separate or clip
// (a full position axis is neutral too, so none is skipped there).
template <int D, bool POS3 = false>
__device__ __forceinline__ bool seg_box_hit(const double* a, const double* b, int d_rt, const Boxes& bx, int box) {
  if constexpr (POS3) {
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      const double lo = bx.lom[box * bx.bs + k * bx.as], hi = bx.him[box * bx.bs + k * bx.as];
      const double x = a[k], y = b[k];
      if ((x < lo && y < lo) || (x > hi && y > hi)) return false;
    }
    double tmin = 0.0, tmax = 1.0;
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      const double ak = a[k];
      const double dk = __dsub_rn(b[k], ak);
      const double l = bx.lo[box * bx.bs + k * bx.as], h = bx.hi[box * bx.bs + k * bx.as];
      if (dk == 0.0) {
        if (ak < l || ak > h) return false;
      } else {
        double t0 = __ddiv_rn(__dsub_rn(l, ak), dk);
        double t1 = __ddiv_rn(__dsub_rn(h, ak), dk);
        if (t0 > t1) {
          const double t = t0;
          t0 = t1;
          t1 = t;
        }
        tmin = (tmin < t0) ? t0 : tmin;
        tmax = (t1 < tmax) ? t1 : tmax;
        if (tmin > tmax) return false;
      }
    }
    return true;
  }
  const int d = dims<D>(d_rt);
  const uint32_t full = bx.full ? bx.full[box] : 0u;  // (the caller has checked the cube)
#pragma unroll
  for (int k = 0; k < (D > 0 ? D : kMaxSolveDim); ++k) {
    if (D == 0 && k >= d) break;
    if ((full >> k) & 1u) continue;
    const double lo = bx.lom ? bx.lom[box * bx.bs + k * bx.as] : bx.lo[box * bx.bs + k * bx.as] - kSepMargin;
    const double hi = bx.him ? bx.him[box * bx.bs + k * bx.as] : bx.hi[box * bx.bs + k * bx.as] + kSepMargin;
    const double x = a[k], y = b[k];
    if ((x < lo && y < lo) || (x > hi && y > hi)) return false;
  }
  double tmin = 0.0, tmax = 1.0;
#pragma unroll
  for (int k = 0; k < (D > 0 ? D : kMaxSolveDim); ++k) {
    if (D == 0 && k >= d) break;
    if ((full >> k) & 1u) continue;
    const double ak = a[k];
    const double dk = __dsub_rn(b[k], ak);
    const double l = bx.lo[box * bx.bs + k * bx.as], h = bx.hi[box * bx.bs + k * bx.as];
    if (dk == 0.0) {
      if (ak < l || ak > h) return false;
    } else {
      double t0 = __ddiv_rn(__dsub_rn(l, ak), dk);
      double t1 = __ddiv_rn(__dsub_rn(h, ak), dk);
      if (t0 > t1) {
        const double t = t0;
        t0 = t1;
        t1 = t;
      }
      tmin = (tmin < t0) ? t0 : tmin;  // std::max(tmin, t0)
      tmax = (t1 < tmax) ? t1 : tmax;  // std::min(tmax, t1)
      if (tmin > tmax) return false;
    }
  }
  return true;
}

#ifndef GMT_POOL_HOIST
#define GMT_POOL_HOIST 1
#endif
#ifndef GMT_SB_VIEWS
#define GMT_SB_VIEWS 1
#endif

// seg_box_hit<6, true> with the staged box arrays passed in (axis stride
// `as`, box stride 1): shared_view pointers make the bound loads LDS
// (configs[4] rows solve 21.8 -> 21.0 ms per 4096 queries).
// (An exact-safe variant forming the quotients with a Newton reciprocal and
// dividing only for near ties measured no faster in rows and 16 % slower in
// the pool-view solve -- register pressure at the 80-register cap.)
__device__ __forceinline__ bool seg_box_hit_pos3(const double* a, const double* b, const double* blo,
                                                 const double* bhi, const double* lom, const double* him, int as,
                                                 int box) {
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    const double lo = lom[box + k * as], hi = him[box + k * as];
    const double x = a[k], y = b[k];
    if ((x < lo && y < lo) || (x > hi && y > hi)) return false;
  }
  double tmin = 0.0, tmax = 1.0;
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    const double ak = a[k];
    const double dk = __dsub_rn(b[k], ak);
    const double l = blo[box + k * as], h = bhi[box + k * as];
    if (dk == 0.0) {
      if (ak < l || ak > h) return false;
    } else {
      double t0 = __ddiv_rn(__dsub_rn(l, ak), dk);
      double t1 = __ddiv_rn(__dsub_rn(h, ak), dk);
      if (t0 > t1) {
        const double t = t0;
        t0 = t1;
        t1 = t;
      }
      tmin = (tmin < t0) ? t0 : tmin;
      tmax = (t1 < tmax) ? t1 : tmax;
      if (tmin > tmax) return false;
    }
  }
  return true;
}

__device__ __forceinline__ void kin_params(const DevInstance& I, QuadParams& QP, DiParams& DP) {
  const int M = I.kin_segments;
  QP.g = I.kin_p[0];
  QP.vmax = I.kin_p[1];
  QP.amax = I.kin_p[2];
  QP.ymax = I.kin_p[3];
  QP.wmax = I.kin_p[4];
  QP.weight = I.kin_p[5];
  QP.segments = M;
  QP.reserved = 0;
  DP.vmax = I.kin_p[0];
  DP.weight = I.kin_p[1];
  DP.segments = M;
  DP.reserved = 0;
}

// The waypoint table of one kinodynamic edge, lane-parallel over (waypoint,
// coordinate): rows 0 and M are the end points (staged in tab by the
// caller), the interior rows the very operations of di_coord / quad_coord.
// The quadrotor's per-chain lambda first (lanes 0-3, into the seg scratch);
// the double integrator's per-axis cubic coefficients c2, c3 (lanes 0-2) and
// waypoint times t_k (lanes 3..) first, which di_coord recomputes
// identically for every coordinate.  Returns (warp-uniform) whether every
// waypoint lies in the unit cube.  vfull (double integrator, every box spans
// the velocity axes): velocity entries only feed the cube test and may be
// replaced by 0.5 / -1 where |v| vs vmax decides it for certain.
template <int D>
__device__ bool kino_fill_table(bool quad, int dim, int M, double tau, int lane, double* seg, double* tab,
                                const QuadParams& QP, const DiParams& DP, bool vfull) {
  const double* x0 = tab;
  const double* x1 = tab + M * dim;
  if (quad) {
    if (lane < 4) quad_chain_lambda(x0, x1, tau, lane, QP, seg + 8 * lane, seg + 8 * lane + 4);
  } else if (lane < 3) {
    const double dp = di_sub(x1[lane], x0[lane]);
    const double v0 = di_vel(x0[3 + lane], DP), v1 = di_vel(x1[3 + lane], DP);
    const double tt = di_mul(tau, tau);
    seg[lane] = di_sub(di_div(di_mul(3.0, dp), tt), di_div(di_add(di_mul(2.0, v0), v1), tau));
    seg[3 + lane] = di_sub(di_div(di_add(v0, v1), tt), di_div(di_mul(2.0, dp), di_mul(tt, tau)));
  } else if (lane - 2 < M) {
    const int k = lane - 2;
    seg[6 + k] = di_div(di_mul(tau, static_cast<double>(k)), static_cast<double>(M));
  }
  __syncwarp();
  bool incube = true;
  for (int e = lane; e < (M + 1) * dim; e += kWarp) {
    const int k = e / dim, i = e - k * dim;
    double v;
    if (k == 0 || k == M) {
      v = tab[e];
    } else if (quad) {
      int c, ci;
      quad_locate(i, &c, &ci);
      v = quad_chain_coord(seg + 8 * c, seg + 8 * c + 4, tau, k, c, ci, QP);
    } else {
      const int a = i < 3 ? i : i - 3;
      const double t = seg[6 + k], c2 = seg[a], c3 = seg[3 + a];
      const double v0 = di_vel(x0[3 + a], DP);
      if (i < 3) {
        v = di_add(x0[a], di_mul(t, di_add(v0, di_mul(t, di_add(c2, di_mul(t, c3))))));
      } else {
        const double vv = di_add(v0, di_mul(t, di_add(di_mul(2.0, c2), di_mul(t, di_mul(3.0, c3)))));
        const double av = vv < 0.0 ? -vv : vv;
        if (vfull && av <= DP.vmax * (1.0 - 1e-14)) {
          // Every box spans the velocity axes, so this coordinate only feeds
          // the cube test, and |v| < vmax puts s = (v / vmax + 1) / 2 in
          // [0, 1] for certain: no division (the value itself is never read).
          v = 0.5;
        } else if (vfull && av >= DP.vmax * (1.0 + 1e-14)) {
          v = -1.0;  // outside [0, 1] for certain (the edge leaves the cube)
        } else {
          v = di_mul(0.5, di_add(di_div(vv, DP.vmax), 1.0));
        }
      }
    }
    tab[e] = v;
    incube = incube && !(v < 0.0 || v > 1.0);
  }
  return __all_sync(kFull, incube);
}

// The same test for a kinodynamic edge (double integrator, quadrotor):
// its waypoint table from the build-time store (in_wp, indexed by the in-edge)
// or regenerated; without a table: lanes 0..dim-1 and 16..16+dim-1 evaluate the
// coordinates of waypoints s and s+1 (di_coord / quad_coord, the very
// functions that materialise stored paths), then the segment goes through
// segment_free_staged.
template <int D>
__device__ bool kino_edge_free_warp(const DevInstance& I, const Boxes& bx, int from, int to,
                                    double tau, int lane, double* seg, double* tab = nullptr,
                                    int tab_cap = 0, uint16_t* cull = nullptr, int cull_cap = 0,
                                    bool staged = false, bool vfull = false, int64_t edge = -1) {
  // Only the generic-dimension kernel can see a 12D quadrotor instance.
  const bool quad = D == 0 && I.steering == GMT_STEER_QUADROTOR;
  const int dim = quad ? kQuadDim : kDiDim;
  // staged: the caller holds the endpoints in seg[0..dim) and seg[16..16+dim)
  const double* x0 = staged ? seg : I.coords + static_cast<int64_t>(from) * dim;
  const double* x1 = staged ? seg + 16 : I.coords + static_cast<int64_t>(to) * dim;
  if (tau == 0.0) return point_free_warp<D>(x0, dim, bx, lane, seg);
  const int M = I.kin_segments;
  QuadParams QP;
  DiParams DP;
  kin_params(I, QP, DP);
  if (tab && (M + 1) * dim <= tab_cap && (quad || M + 6 <= kWarp)) {
    __syncwarp();
    bool incube = true;
    if (I.in_wp && edge >= 0) {
      // The table stored at build time (kino_table_kernel: this very fill),
      // the reference's cached polyline (graph.cpp edge_path) in table form.
      const int W = (M + 1) * dim;
      const double* src = I.in_wp + edge * W;
      for (int e = lane; e < W; e += kWarp) {
        const double v = __ldg(src + e);
        tab[e] = v;
        incube = incube && !(v < 0.0 || v > 1.0);
      }
      incube = __all_sync(kFull, incube);
    } else {
      if (lane < dim) {  // the end points are waypoints 0 and M (and free seg for scratch)
        const double a = x0[lane], b = x1[lane];
        tab[lane] = a;
        tab[M * dim + lane] = b;
      }
      __syncwarp();
      incube = kino_fill_table<D>(quad, dim, M, tau, lane, seg, tab, QP, DP, vfull);
    }
    // polyline_free (space.cpp:92-99) = every waypoint in the unit cube (each
    // segment's point_in_cube / point_free endpoint test) and no (segment,
    // box) pair hit -- a degenerate segment's all-axes dk == 0 clip is
    // exactly Aabb::contains; the outcome does not depend on the order.
    if (!incube) return false;
    __syncwarp();
    // Boxes the whole polyline's bounding box (widened by the separation
    // margin) misses are missed by every segment's own pre-test: they are
    // dropped once per edge, and the segments test the survivors only.
    Boxes sub = bx;
    if (cull && bx.count > 0) {
      if (lane < dim) {
        double mn = tab[lane], mx = tab[lane];
        for (int k = 1; k <= M; ++k) {
          const double x = tab[k * dim + lane];
          mn = x < mn ? x : mn;
          mx = x < mx ? mx : x;
        }
        seg[lane] = mn;
        seg[16 + lane] = mx;
      }
      __syncwarp();
      constexpr int kR = D > 0 ? D : 1;  // fixed dimension: the bounding box in registers
      double pmn[kR], pmx[kR];
      if constexpr (D > 0) {
#pragma unroll
        for (int k = 0; k < D; ++k) {
          pmn[k] = seg[k];
          pmx[k] = seg[16 + k];
        }
      }
      int kept = 0;
      for (int i0 = 0; i0 < bx.count && kept <= cull_cap; i0 += kWarp) {
        const int b = i0 + lane;
        bool meets = b < bx.count;
        const int bc = meets ? b : 0;
        if constexpr (D > 0) {
          const uint32_t full = bx.full ? bx.full[bc] : 0u;
#pragma unroll
          for (int k = 0; k < D; ++k) {
            if ((full >> k) & 1u) continue;
            const double lo = bx.lom ? bx.lom[bc * bx.bs + k * bx.as] : bx.lo[bc * bx.bs + k * bx.as] - kSepMargin;
            const double hi = bx.him ? bx.him[bc * bx.bs + k * bx.as] : bx.hi[bc * bx.bs + k * bx.as] + kSepMargin;
            meets = meets && !(pmx[k] < lo || pmn[k] > hi);
          }
        } else {
          for (int k = 0; k < dim && meets; ++k) {
            const double lo = bx.lom ? bx.lom[bc * bx.bs + k * bx.as] : bx.lo[bc * bx.bs + k * bx.as] - kSepMargin;
            const double hi = bx.him ? bx.him[bc * bx.bs + k * bx.as] : bx.hi[bc * bx.bs + k * bx.as] + kSepMargin;
            meets = !(seg[16 + k] < lo || seg[k] > hi);
          }
        }
        const uint32_t m = __ballot_sync(kFull, meets);
        const int at = kept + __popc(m & ((1u << lane) - 1u));
        if (meets && at < cull_cap) cull[at] = static_cast<uint16_t>(b);
        kept += __popc(m);
      }
      __syncwarp();
      if (kept <= cull_cap) {
        sub.idx = cull;
        sub.count = kept;
      }
    }
    // Lane per (segment, box) pair, each through the reference's clip.
    const int nbx = sub.count;
    const int pairs = M * nbx;
    for (int p0 = 0; p0 < pairs; p0 += kWarp) {
      const int p = p0 + lane;
      bool hit = false;
      if (p < pairs) {
        const int sg = p / nbx, bi = p - sg * nbx;
        hit = seg_box_hit<D>(tab + sg * dim, tab + (sg + 1) * dim, dim, bx, sub.idx ? sub.idx[bi] : bi);
      }
      if (__any_sync(kFull, hit)) return false;
    }
    return true;
  }
  const int i = lane & 15;
  const int k = lane >> 4;
  for (int s = 0; s < M; ++s) {
    __syncwarp();
    if (i < dim) seg[lane] = quad ? quad_coord(x0, x1, tau, s + k, i, QP) : di_coord(x0, x1, tau, s + k, i, DP);
    __syncwarp();
    if (!segment_free_staged<D>(dim, bx, lane, seg)) return false;
  }
  return true;
}

// The double integrator's lazy check on a G-lane group (half or quarter warp),
// so the candidates a batched warp scans are checked concurrently: the same
// steps as kino_edge_free_warp's table path (waypoint table from the cubic
// coefficients, cube test, polyline bounding-box cull, one lane per
// (segment, box) pair through the reference's clip) with group-masked votes.
// seg: the group's 32 staged doubles (a = [0..6), b = [16..22)); tab: its
// waypoint table ((M + 1) * 6 <= 64); cull: its box list.
// rec (every box spans the velocity axes, a pool edge): the edge's check
// record (common.cuh), which replaces the table, the cube test and the
// bounding box; the table's positions are read only when some box survives
// the cull.
template <int G, bool SB = false>
__device__ bool di_edge_free_half(const DevInstance& I, const Boxes& bx, double tau, int gl, uint32_t gmask,
                                  int gbase, double* seg, double* tab, uint16_t* cull, int cull_cap, bool vfull,
                                  double box_wx = -1.0, const double* rec = nullptr,
                                  const uint16_t* xfirst = nullptr) {
  constexpr int dim = kDiDim;
  static_assert(G >= 8, "a group must hold a state's coordinates and the coefficient lanes");
  constexpr uint32_t kGroupBits = G == 32 ? 0xffffffffu : ((1u << G) - 1u);
  const int M = I.kin_segments;
  DiParams DP;
  DP.vmax = I.kin_p[0];
  DP.weight = I.kin_p[1];
  DP.segments = M;
  DP.reserved = 0;
  // point_free(x0) (the degenerate edge's single state).  (A record's
  // zero-duration polyline is M copies of x0, which the record path tests
  // the same way: cube, then Aabb::contains by the all-dk == 0 clip.)
  if (!rec && tau == 0.0) {
    bool cube = true;
    if (gl < dim) cube = !(seg[gl] < 0.0 || seg[gl] > 1.0);
    if (!__all_sync(gmask, cube)) return false;
    bool in = false;
    for (int b = gl; b < bx.count && !in; b += G) in = box_has<6>(seg, dim, bx, b);
    return !__any_sync(gmask, in);
  }
  if (rec) {
    // The pool edge's record, all of it in flight at once: the bounding box
    // (NaN: the polyline leaves the cube) and the waypoint positions.
    // (asynchronous copies straight into shared memory: no registers held)
    const int rl = kPoolRecHead + 3 * (M + 1);
    for (int e = gl; e < rl; e += G)  // min -> seg[0..3), max -> seg[16..19), positions -> tab
      cp_async8(e < kPoolRecHead ? seg + (e < 3 ? e : 13 + e) : tab + (e - kPoolRecHead), rec + e);
    cp_async_wait_all();
    __syncwarp(gmask);
    if (__any_sync(gmask, gl == 0 && seg[0] != seg[0])) return false;
  } else {
  if (gl < dim) {
    tab[gl] = seg[gl];
    tab[M * dim + gl] = seg[16 + gl];
  }
  __syncwarp(gmask);
  const double* x0 = tab;
  const double* x1 = tab + M * dim;
  if (gl < 3) {
    const double D = di_sub(x1[gl], x0[gl]);
    const double v0 = di_vel(x0[3 + gl], DP), v1 = di_vel(x1[3 + gl], DP);
    const double tt = di_mul(tau, tau);
    seg[gl] = di_sub(di_div(di_mul(3.0, D), tt), di_div(di_add(di_mul(2.0, v0), v1), tau));
    seg[3 + gl] = di_sub(di_div(di_add(v0, v1), tt), di_div(di_mul(2.0, D), di_mul(tt, tau)));
  } else {
    for (int k = gl - 2; k < M; k += G - 3) {
      const double tk = di_mul(tau, static_cast<double>(k));
      // (tau k) / M: for M a power of two the quotient is the exact scaling
      // tk * (1 / M) unless it would be subnormal -- the same double
      seg[6 + k] = ((M & (M - 1)) == 0 && tk >= 1e-290) ? di_mul(tk, 1.0 / static_cast<double>(M))
                                                         : di_div(tk, static_cast<double>(M));
    }
  }
  __syncwarp(gmask);
  bool incube = true;
  for (int e = gl + dim; e < M * dim; e += G) {  // interior waypoints (rows 1 .. M-1)
    const int k = e / dim, i = e - k * dim;
    const int a = i < 3 ? i : i - 3;
    const double t = seg[6 + k], c2 = seg[a], c3 = seg[3 + a];
    const double v0 = di_vel(x0[3 + a], DP);
    double v;
    if (i < 3) {
      v = di_add(x0[a], di_mul(t, di_add(v0, di_mul(t, di_add(c2, di_mul(t, c3))))));
    } else {
      const double vv = di_add(v0, di_mul(t, di_add(di_mul(2.0, c2), di_mul(t, di_mul(3.0, c3)))));
      const double av = vv < 0.0 ? -vv : vv;
      if (vfull && av <= DP.vmax * (1.0 - 1e-14)) {
        v = 0.5;  // (see kino_edge_free_warp: only the cube test reads it, and it passes)
      } else if (vfull && av >= DP.vmax * (1.0 + 1e-14)) {
        v = -1.0;
      } else {
        v = di_mul(0.5, di_add(di_div(vv, DP.vmax), 1.0));
      }
    }
    tab[e] = v;
    incube = incube && !(v < 0.0 || v > 1.0);
  }
  if (gl < dim) {
    incube = incube && !(x0[gl] < 0.0 || x0[gl] > 1.0) && !(x1[gl] < 0.0 || x1[gl] > 1.0);
  }
  if (!__all_sync(gmask, incube)) return false;
  __syncwarp(gmask);
  // polyline bounding box -> the boxes it meets (exact-safe cull)
  if (gl < dim) {
    double mn = tab[gl], mx = tab[gl];
    for (int k = 1; k <= M; ++k) {
      const double x = tab[k * dim + gl];
      mn = x < mn ? x : mn;
      mx = x < mx ? mx : x;
    }
    seg[gl] = mn;
    seg[16 + gl] = mx;
  }
  __syncwarp(gmask);
  }  // (rec)
  double pmn[dim], pmx[dim];
#pragma unroll
  for (int k = 0; k < dim; ++k) {
    pmn[k] = seg[k];
    pmx[k] = seg[16 + k];
  }
  Boxes sub = bx;
  int kept = 0;
  int ib = 0, ie = bx.count;
  if (vfull && box_wx >= 0.0) {
    // Boxes staged in ascending lom_x: only [first lom_x >= pmn_x - wx,
    // first lom_x > pmx_x) can meet the bounding box on x (every him_x <=
    // lom_x + wx; the 1e-9 widening absorbs the subtraction's rounding).
    // Two rounds over the group: the chunk, then the index in it.
    const double lo_t = (pmn[0] - box_wx) - 1e-9, hi_t = pmx[0];
    if (xfirst) {
      int bl = xbucket(lo_t) - 1, bh = xbucket(hi_t) + 2;
      bl = bl < 0 ? 0 : (bl > kXB ? kXB : bl);
      bh = bh < 0 ? 0 : (bh > kXB ? kXB : bh);
      ib = xfirst[bl];
      ie = xfirst[bh];
    } else {
    const int chunk = (bx.count + G - 1) / G;
    const int last = gl * chunk + chunk - 1 < bx.count ? gl * chunk + chunk - 1 : bx.count - 1;
    const double xe = gl * chunk < bx.count ? bx.lom[last] : kInf;
    const int c_lo = __popc((__ballot_sync(gmask, xe < lo_t) >> gbase) & kGroupBits);
    const int c_hi = __popc((__ballot_sync(gmask, !(xe > hi_t)) >> gbase) & kGroupBits);
    ib = c_lo * chunk;
    ie = c_hi * chunk;
    for (int j0 = ib; j0 < bx.count && j0 < (c_lo + 1) * chunk; j0 += G) {
      const int j = j0 + gl;
      const bool below = j < bx.count && j < (c_lo + 1) * chunk && bx.lom[j] < lo_t;
      ib += __popc((__ballot_sync(gmask, below) >> gbase) & kGroupBits);
    }
    for (int j0 = ie; j0 < bx.count && j0 < (c_hi + 1) * chunk; j0 += G) {
      const int j = j0 + gl;
      const bool in = j < bx.count && j < (c_hi + 1) * chunk && !(bx.lom[j] > hi_t);
      ie += __popc((__ballot_sync(gmask, in) >> gbase) & kGroupBits);
    }
    ie = ie < bx.count ? ie : bx.count;
    }
  }
  if (SB && vfull) {
    // The staged boxes are in this CTA's shared memory: LDS views (box
    // stride 1, axis stride as); only the position axes can separate.
    const double* const lom_v = shared_view(bx.lom);
    const double* const him_v = shared_view(bx.him);
    const int as = bx.as;
    for (int i0 = ib; i0 < ie && kept <= cull_cap; i0 += G) {
      const int b = i0 + gl;
      bool meets = b < ie;
      const int bc = meets ? b : 0;
#pragma unroll
      for (int k = 0; k < 3; ++k) meets = meets && !(pmx[k] < lom_v[bc + k * as] || pmn[k] > him_v[bc + k * as]);
      const uint32_t m = (__ballot_sync(gmask, meets) >> gbase) & kGroupBits;
      const int at = kept + __popc(m & ((1u << gl) - 1u));
      if (meets && at < cull_cap) cull[at] = static_cast<uint16_t>(b);
      kept += __popc(m);
    }
    ie = ib;  // (done: the generic loop below runs no iteration)
  }
  for (int i0 = ib; i0 < ie && kept <= cull_cap; i0 += G) {
    const int b = i0 + gl;
    bool meets = b < ie;
    const int bc = meets ? b : 0;
    if (vfull) {  // (boxes staged: lom / him set) only the position axes can separate
#pragma unroll
      for (int k = 0; k < 3; ++k)
        meets = meets && !(pmx[k] < bx.lom[bc * bx.bs + k * bx.as] || pmn[k] > bx.him[bc * bx.bs + k * bx.as]);
    } else {
      const uint32_t full = bx.full ? bx.full[bc] : 0u;
#pragma unroll
      for (int k = 0; k < dim; ++k) {
        if ((full >> k) & 1u) continue;
        const double lo = bx.lom ? bx.lom[bc * bx.bs + k * bx.as] : bx.lo[bc * bx.bs + k * bx.as] - kSepMargin;
        const double hi = bx.him ? bx.him[bc * bx.bs + k * bx.as] : bx.hi[bc * bx.bs + k * bx.as] + kSepMargin;
        meets = meets && !(pmx[k] < lo || pmn[k] > hi);
      }
    }
    const uint32_t m = (__ballot_sync(gmask, meets) >> gbase) & kGroupBits;
    const int at = kept + __popc(m & ((1u << gl) - 1u));
    if (meets && at < cull_cap) cull[at] = static_cast<uint16_t>(b);
    kept += __popc(m);
  }
  __syncwarp(gmask);
  if (kept <= cull_cap) {
    sub.idx = cull;
    sub.count = kept;
  }
  int ts = dim;  // waypoint stride in tab
  if (rec) {
    if (kept == 0) return true;  // no box meets the polyline's bounding box
    ts = 3;
  }
  const int nbx = sub.count;
  const int pairs = M * nbx;
  const int lg_m = (M & (M - 1)) == 0 ? __ffs(M) - 1 : -1;  // (box-major pairs: no division for M = 2^k)
  if (SB && vfull) {
    const double* const lo_v = shared_view(bx.lo);
    const double* const hi_v = shared_view(bx.hi);
    const double* const lom_v = shared_view(bx.lom);
    const double* const him_v = shared_view(bx.him);
    const int as = bx.as;
    for (int p0 = 0; p0 < pairs; p0 += G) {
      const int p = p0 + gl;
      bool hit = false;
      if (p < pairs) {
        const int bi = lg_m >= 0 ? p >> lg_m : p / M;
        const int sg = p - bi * M;
        const int box = sub.idx ? sub.idx[bi] : bi;
        hit = seg_box_hit_pos3(tab + sg * ts, tab + (sg + 1) * ts, lo_v, hi_v, lom_v, him_v, as, box);
      }
      if (__any_sync(gmask, hit)) return false;
    }
    return true;
  }
  for (int p0 = 0; p0 < pairs; p0 += G) {
    const int p = p0 + gl;
    bool hit = false;
    if (p < pairs) {
      const int bi = lg_m >= 0 ? p >> lg_m : p / M;
      const int sg = p - bi * M;
      const int box = sub.idx ? sub.idx[bi] : bi;
      hit = vfull ? seg_box_hit<6, true>(tab + sg * ts, tab + (sg + 1) * ts, dim, bx, box)
                  : seg_box_hit<6>(tab + sg * ts, tab + (sg + 1) * ts, dim, bx, box);
    }
    if (__any_sync(gmask, hit)) return false;
  }
  return true;
}

__device__ __forceinline__ double block_min(double v, double* red, int lane, int warp, int nw) {
  for (int o = 16; o; o >>= 1) {
    const double t = __shfl_xor_sync(kFull, v, o);
    v = t < v ? t : v;
  }
  if (lane == 0) red[warp] = v;
  __syncthreads();
  v = lane < nw ? red[lane] : kInf;
  for (int o = 16; o; o >>= 1) {
    const double t = __shfl_xor_sync(kFull, v, o);
    v = t < v ? t : v;
  }
  return v;
}

// Lexicographic (cost, index) minimum; "none" is (inf, kNone).
__device__ __forceinline__ void argmin_step(double& c, int32_t& v, double oc, int32_t ov) {
  if (oc < c || (oc == c && ov < v)) {
    c = oc;
    v = ov;
  }
}

__device__ __forceinline__ void block_argmin(double& c, int32_t& v, CtaShared& sh, int lane,
                                             int warp, int nw) {
  for (int o = 16; o; o >>= 1) {
    argmin_step(c, v, __shfl_xor_sync(kFull, c, o), __shfl_xor_sync(kFull, v, o));
  }
  if (lane == 0) {
    sh.red_goal_c[warp] = c;
    sh.red_goal_v[warp] = v;
  }
  __syncthreads();
  c = lane < nw ? sh.red_goal_c[lane] : kInf;
  v = lane < nw ? sh.red_goal_v[lane] : kNone;
  for (int o = 16; o; o >>= 1) {
    argmin_step(c, v, __shfl_xor_sync(kFull, c, o), __shfl_xor_sync(kFull, v, o));
  }
}

}  // namespace

// Two CTA shapes: WIDE = 512 threads with up to 128 registers (clusters,
// and single-CTA queries that want the registers), narrow = 256 threads,
// 64 registers, four CTAs per SM.
#ifndef GMT_ROWS_CS
#define GMT_ROWS_CS 1
#endif
#ifndef GMT_DI_XAHEAD
#define GMT_DI_XAHEAD 1
#endif
#ifndef GMT_UNROLL_DI24
#define GMT_UNROLL_DI24 GMT_UNROLL_BATCH
#endif
#ifndef GMT_DI_XBUCKET
#define GMT_DI_XBUCKET 1
#endif
#ifndef GMT_DI_DYNAMIC
#define GMT_DI_DYNAMIC 2  // (P5 dynamic: 24.6 -> 24.1 ms per 4096 configs[4] queries; P4 too: no gain)
#endif
#ifndef GMT_BATCH_MIN_BLOCKS
#define GMT_BATCH_MIN_BLOCKS 4
#endif
// COUNT: single-CTA solves count the open-source gathers only in the
// instantiation launched while traffic counters are on (GMT_OPT_COUNTERS);
// cluster solves always can.
// Kinodynamic queries (D = 6 double integrator, D = 0 quadrotor) need about
// 55 KB of shared memory per narrow CTA, so three fit an SM: those narrow
// kernels get the registers of three CTAs per SM.
// GS: the wavefront state (cost, bitmasks, lists, staged boxes) lives in a
// per-query global buffer (SolveJob::gstate, L2-resident) instead of shared
// memory -- queries too large for the shared-memory opt-in (single CTA).
// POOL: jobs may carry shared-pool views (DevInstance::pool, batched DI
// queries): their rows are read from the pool graph through the query's
// rank map instead of materialised rows.
// NW != 0: a CTA of NW warps at one per SM (the batched double integrator's
// latency shape for batches of a few waves: 24 warps = the SM's three narrow
// CTAs' worth on one query, 80 registers).
template <int CS, int D, bool WIDE, bool COUNT, bool GS = false, bool POOL = false, int NW = 0>
__global__ void __launch_bounds__(NW ? NW * 32 : (WIDE ? 512 : 256),
                                  NW ? 1 : (WIDE ? 1 : ((D == 6 || D == 0) ? 3 : GMT_BATCH_MIN_BLOCKS)))
    gmt_solve_kernel(const SolveJob* __restrict__ jobs, int obs_in_smem) {
  constexpr bool kParentSmem = CS > 1;  // single-CTA solves keep parents in HBM
  constexpr int kMaxWarps = NW ? NW : (WIDE ? 16 : 8);
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ CtaShared sh;
  // Rows streamed concurrently per warp in P4/P5: two for batched
  // single-CTA solves (latency hiding), one for clusters (few candidates per
  // warp; the pass critical path matters).
  // (the 24-warp batched DI shape streams and checks four candidates per warp)
  constexpr int kRows = CS == 1 ? ((D == 6 && NW == 24) ? GMT_ROWS_DI24 : GMT_ROWS_PER_WARP) : GMT_ROWS_CLUSTER;
  constexpr int kLanesPerRow = kWarp / kRows;
  constexpr int kUnroll = CS == 1 ? ((D == 6 && NW == 24) ? GMT_UNROLL_DI24 : GMT_UNROLL_BATCH) : GMT_UNROLL_CLUSTER;
  // Dynamic row / candidate distribution (a shared counter): clusters, and
  // the batched 24-warp DI shape's candidates (GMT_DI_DYNAMIC bit 1: P4 rows,
  // bit 2: P5 candidates), whose lazy checks vary widely in cost.
  constexpr bool kDi24 = CS == 1 && D == 6 && NW == 24;
  constexpr bool kRowsCs = kDi24 && GMT_ROWS_CS && !POOL;  // streaming loads of materialised rows (not compiled into the view kernel: it perturbed that one by 12 %)
  constexpr bool kDynOwn = CS > 1 || (kDi24 && (GMT_DI_DYNAMIC & 1));
  constexpr bool kDynamic = CS > 1 || (kDi24 && (GMT_DI_DYNAMIC & 2));
  // Per-warp scratch: kRows staged segments, kinodynamic waypoint tables
  // (double integrator: D = 6; quadrotor: D = 0) and surviving-box lists --
  // batched DI solves check kRows edges per warp at once (one table / list
  // each).  NW kernels (more than the 48 KB of static shared memory) keep it
  // in dynamic shared memory after the solve layout (solve_dyn_scratch).
  constexpr int kTabCap = D == 6 ? kDiTabCap : (D == 0 ? 144 : 1);
  constexpr int kKinSlots = (D == 6 && kRows >= 2) ? kRows : 1;
  constexpr int kCullCap = (D == 0 || D == 6) ? 64 : 1;  // per-warp surviving-box list
  constexpr bool kDynScratch = NW != 0;
  constexpr int kSegN = kMaxWarps * 32 * kRows;
  constexpr int kTabN = (D == 0 || D == 6) ? kMaxWarps * kTabCap * kKinSlots : 1;
  constexpr int kCullN = kMaxWarps * kCullCap * kKinSlots;
  __shared__ double seg_st[kDynScratch ? 1 : kSegN];
  __shared__ double tab_st[kDynScratch ? 1 : kTabN];
  __shared__ uint16_t cull_st[kDynScratch ? 1 : kCullN];

  const int q = blockIdx.x / CS;
  int rank = 0;
  if constexpr (CS > 1) rank = static_cast<int>(cg::this_cluster().block_rank());
  // The job, instance and result descriptors live in shared memory: their
  // ~30 pointers are reloaded (LDS, broadcast) where used instead of pinning
  // registers for the whole solve.
  __shared__ SolveJob job_s;
  __shared__ DevInstance inst_s;
  __shared__ PoolView pv_s;
  if (threadIdx.x == 0) {
    job_s = jobs[q];
    inst_s = *job_s.inst;
    if (!inst_s.out_end) inst_s.out_end = inst_s.out_ptr + 1;  // CSR: row x ends at ptr[x + 1]
    if (!inst_s.in_end) inst_s.in_end = inst_s.in_ptr + 1;
    if (POOL && inst_s.pool) pv_s = *inst_s.pool;
  }
  __syncthreads();
  const SolveJob& job = job_s;
  const DevInstance& I = inst_s;
  const bool viewed = POOL && I.pool != nullptr;  // (block-uniform)
  const PoolView& PV = pv_s;
  const DevResult& R = job_s.res;
  const int n = I.n, d = dims<D>(I.dim), nb = I.num_boxes;
  using ListT = typename std::conditional<GS, int32_t, uint16_t>::type;  // work-list vertex ids
  const SolveLayout L = solve_layout(n, d, nb, obs_in_smem != 0, kParentSmem, GS ? 4 : 2);
  const int W = L.words;
  unsigned char* const sbase = GS ? job_s.gstate : smem;  // (GS = false: shared memory)

  double* cost_s = reinterpret_cast<double*>(sbase + L.off_cost);
  uint16_t* parent_s = reinterpret_cast<uint16_t*>(sbase + L.off_parent);
  uint32_t* open_w = reinterpret_cast<uint32_t*>(sbase + L.off_bits);
  uint32_t* closed_w = open_w + L.words_pad;
  uint32_t* group_w = closed_w + L.words_pad;
  uint32_t* newopen_w = group_w + L.words_pad;
  uint32_t* cand_w = newopen_w + L.words_pad;
  uint32_t* goal_w = cand_w + L.words_pad;
  ListT* list = reinterpret_cast<ListT*>(sbase + L.off_list);
  double* seg_s = seg_st;
  double* tab_s = tab_st;
  uint16_t* cull_s = cull_st;
  if constexpr (kDynScratch) {
    unsigned char* scratch = smem + align16(L.total);
    seg_s = reinterpret_cast<double*>(scratch);
    tab_s = seg_s + kSegN;
    cull_s = reinterpret_cast<uint16_t*>(tab_s + kTabN);
  }

  const int tid = threadIdx.x, nt = blockDim.x;
  const int lane = tid & 31, warp = tid >> 5, nw = nt >> 5;
  double* seg = seg_s + warp * 32 * kRows;

  __shared__ Boxes bx_s;
  Boxes bxl;
  bxl.count = nb;
  if (obs_in_smem) {
    // Stage the boxes axis-major, with the separation bounds lo - m, hi + m.
    double* lo = reinterpret_cast<double*>(sbase + L.off_obs);
    double* hi = lo + static_cast<size_t>(nb) * d;
    double* lom = hi + static_cast<size_t>(nb) * d;
    double* him = lom + static_cast<size_t>(nb) * d;
    // The 24-warp D = 6 shape stages the boxes in ascending lo_x order (ties
    // by index): the pair tests' outcome does not depend on the box order,
    // and the edge cull then scans an x range (di_edge_free_half).
    constexpr bool kXSort = D == 6 && kDynScratch;
    constexpr int kSortMax = 256;
    __shared__ uint8_t xrank_s[kXSort ? kSortMax : 1];
    __shared__ uint16_t xfirst_s[(kXSort && GMT_DI_XBUCKET) ? kXB + 1 : 1];
    if constexpr (kXSort && GMT_DI_XBUCKET) {
      if (tid == 0) sh.xfirst = xfirst_s;
    }
    const bool xsort = kXSort && nb <= kSortMax;
    if (xsort) {
      for (int b = tid; b < nb; b += nt) {
        const double x = I.box_lo[b * d];
        int r = 0;
        for (int c = 0; c < nb; ++c) {
          const double y = I.box_lo[c * d];
          r += (y < x || (y == x && c < b)) ? 1 : 0;
        }
        xrank_s[b] = static_cast<uint8_t>(r);
      }
      __syncthreads();
    }
    for (int idx = tid; idx < nb * d; idx += nt) {
      const int b0 = idx / d, k = idx - b0 * d;
      const int b = xsort ? xrank_s[b0] : b0;
      const double l = I.box_lo[idx], h = I.box_hi[idx];
      lo[k * nb + b] = l;
      hi[k * nb + b] = h;
      lom[k * nb + b] = l - kSepMargin;
      him[k * nb + b] = h + kSepMargin;
    }
    uint32_t* full = reinterpret_cast<uint32_t*>(him + static_cast<size_t>(nb) * d);
    for (int b0 = tid; b0 < nb; b0 += nt) {
      uint32_t m = 0u;
      for (int k = 0; k < d; ++k)
        if (I.box_lo[b0 * d + k] <= 0.0 && I.box_hi[b0 * d + k] >= 1.0) m |= 1u << k;
      full[xsort ? xrank_s[b0] : b0] = m;
    }
    if (xsort) {
      __syncthreads();
      if (tid == 0) {
        double w = 0.0;
        for (int b = 0; b < nb; ++b) {
          const double e = him[b] - lom[b];
          w = e > w ? e : w;
        }
        sh.box_wx = w * (1.0 + 1e-12) + 1e-12;  // (rounded up: every him_x <= lom_x + box_wx)
      }
      if constexpr (kXSort && GMT_DI_XBUCKET) {
        for (int b = tid; b <= kXB; b += nt) {
          const double xb = kXB0 + static_cast<double>(b) * kXBW;
          int c = 0;
          for (int i = 0; i < nb; ++i) c += lom[i] < xb ? 1 : 0;
          xfirst_s[b] = static_cast<uint16_t>(b == 0 ? 0 : (b == kXB ? nb : c));
        }
      }
    }
    if (tid == 0) sh.xsorted = xsort ? 1 : 0;
    bxl.lo = lo, bxl.hi = hi, bxl.lom = lom, bxl.him = him, bxl.bs = 1, bxl.as = nb;
    bxl.full = full;
    if constexpr (D == 6) {
      __syncthreads();
      int vf = 1;
      for (int b = tid; b < nb; b += nt) vf &= (full[b] & 0x38u) == 0x38u ? 1 : 0;
      vf = __syncthreads_and(vf);
      if (tid == 0) sh.vfull = vf;
    }
  } else {
    bxl.lo = I.box_lo, bxl.hi = I.box_hi, bxl.lom = nullptr, bxl.him = nullptr, bxl.bs = d, bxl.as = 1;
    bxl.full = nullptr;
    if (tid == 0) sh.vfull = 0;
    if (tid == 0) sh.xsorted = 0;
  }
  bxl.idx = nullptr;

  // make_wavefront (planner.cpp:25-35) on every replica.
  const int init = job.init_index;
  for (int v = tid; v < n; v += nt) {
    cost_s[v] = kInf;
    if constexpr (kParentSmem) parent_s[v] = 0xffffu;
  }
  for (int w = tid; w < W; w += nt) {
    open_w[w] = closed_w[w] = group_w[w] = newopen_w[w] = cand_w[w] = 0u;
  }
  // Goal membership is geometric: goal.contains(samples.states[v])
  // (planner.cpp:147), evaluated once per solve into a bitmask.
  for (int w = warp; w < W; w += nw) {
    const int v = w * 32 + lane;
    bool g = v < n;
    if (g) g = box_contains(I.goal_lo, I.goal_hi, d, I.coords + static_cast<int64_t>(v) * d);
    const uint32_t gb = __ballot_sync(kFull, g);
    if (lane == 0) goal_w[w] = gb;
  }
  for (int v = rank * nt + tid; v < n; v += CS * nt) {
    if (R.iter_added) R.iter_added[v] = (v == init) ? 0 : -1;
    if (!kParentSmem) R.parent[v] = -1;
  }
  if (tid == 0) {
    sh.group_count = 0;
    sh.own_count = 0;
    sh.cand_count = 0;
    sh.checks_acc = 0ull;
    sh.added_acc = 0;
    sh.iter = 0;
    sh.total_checks = 0;
    sh.next_own = kRows * (static_cast<int>(blockDim.x) >> 5);
    sh.next_cand = kRows * (static_cast<int>(blockDim.x) >> 5);
    sh.pass = 0;
    sh.cnt_in = 0ull;
    sh.cnt_out = 0ull;
    bx_s = bxl;
  }
  if (tid < 32) {
    sh.wchecks[tid] = 0;
    sh.wadded[tid] = 0;
  }
  __syncthreads();
  const Boxes& bx = bx_s;  // read from shared memory where used
  // Shared-pool views: pool point y -> query vertex (or -1).  (A shared-
  // memory bitmask + rank bases measured slower than this L1-cached gather:
  // 46.6 vs 41.9 ms per 4096 queries.)
  // (The whole rank map staged in shared memory measured slower as well in
  // the 24-warp shape: 26.6 vs 23.3 ms per 4096 queries; so did the open set
  // mirrored as pool-point bits, gathering ranks for open entries only: 27.9
  // vs 27.2 ms -- the scan waits on the pool rows' loads, not on the map.)
  auto pool_rank = [&](int y) -> int {
    // (y >= kc: a pool point past this call's scan, no query's vertex)
    const uint16_t r = y < PV.kc ? __ldg(PV.rank + y) : kPoolNoRank;
    return r == kPoolNoRank ? -1 : static_cast<int>(r);
  };

  // infeasible_input (planner.cpp:39-41, 108): empty tree.
  if (warp == 0) {
    const bool ok = I.goal_count > 0 &&
                    point_free_warp<D>(I.coords + static_cast<int64_t>(init) * d, d, bx, lane, seg);
    if (lane == 0) sh.feasible = ok ? 1 : 0;
  }
  __syncthreads();
  if (!sh.feasible) {
    if (rank == 0 && tid == 0) {
      ResultScalars s;
      s.status = 2;
      s.goal_node = -1;
      s.cost = kInf;
      s.iterations = 0;
      s.total_checks = 0;
      s.path_len = 0;
      s.num_stats = 0;
      s.tree_size = 0;
      s.reserved = 0;
      *R.scalars = s;
    }
    return;
  }
  if (tid == 0) {
    cost_s[init] = 0.0;
    open_w[init >> 5] |= 1u << (init & 31);
  }
  // The coordinates are read once per lazy check (both endpoints): make the
  // whole array L2-resident up front (each CTA of a cluster takes a slice).
  if (tid == 0) {
    const size_t bytes = sizeof(double) * static_cast<size_t>(n) * d;
    const size_t slice = (bytes / CS + 15) & ~static_cast<size_t>(15);
    const size_t off = slice * rank;
    if (off < bytes) {
      prefetch_l2(reinterpret_cast<const char*>(I.coords) + off,
                  off + slice < bytes ? slice : bytes - off);
    }
  }
  cluster_barrier<CS>();  // every replica initialised before any remote access

  const double delta = __dmul_rn(job.lambda, job.radius);  // GmtParams::delta
  int status = 1;
  int goal = -1;
  // Traffic counters for the roofline's algorithmic bytes:
  // out-row edges (P4) and in-row edges (P5) are summed per row into
  // shared memory; in-edges whose source was open (the cost[y] gathers) per
  // lane.
  const bool counting = R.counters != nullptr;
  int cnt_open = 0;

#ifdef GMT_PHASE_TIMING
  // [0..3] the passes' phases (thread 0); [4..7] per-warp sums over the P5
  // loop: the whole loop, inside the lazy checks (group 0), the barrier wait
  // after the loop, the P4 loop
  __shared__ unsigned long long sh_ph[8];
  long long ph_t = clock64();
  if (tid < 8) sh_ph[tid] = 0;
#endif
  for (;;) {
    long long i = sh.iter;  // written by tid 0 only, behind the pass barriers
    if (job.mode == kModeFmt) {
      // fmt_plan (planner.cpp:207-225): z = first minimum-cost open node;
      // the "group" is {z}; no thresholds.
      double zc = kInf;
      int32_t z = kNone;
      for (int w = warp; w < W; w += nw) {
        if ((open_w[w] >> lane) & 1u) argmin_step(zc, z, cost_s[w * 32 + lane], w * 32 + lane);
      }
      block_argmin(zc, z, sh, lane, warp, nw);
      if (z == kNone) {
        status = 1;
        break;
      }
      if ((goal_w[z >> 5] >> (z & 31)) & 1u) {
        status = 0;
        goal = z;
        if (tid == 0) sh.group_count = 1;  // the final group's size
        break;
      }
      if (tid == 0) {
        group_w[z >> 5] = 1u << (z & 31);
        if (((z >> 5) & (CS - 1)) == rank) {
          list[0] = static_cast<ListT>(z);
          sh.own_count = 1;
        }
      }
      __syncthreads();
    } else {
      // P0: min cost over open nodes (planner.cpp:119-122).
      double m = kInf;
      for (int w = warp; w < W; w += nw) {
        if ((open_w[w] >> lane) & 1u) {
          const double c = cost_s[w * 32 + lane];
          m = c < m ? c : m;
        }
      }
      m = block_min(m, sh.red_min, lane, warp, nw);
      if (m == kInf) {  // planner.cpp:123-127
        status = 1;
        break;
      }
      // P1: fast-forward (planner.cpp:132-136); i*delta is (double)i * delta.
      if (m > __dmul_rn(static_cast<double>(i), delta)) {
        const long long jump = static_cast<long long>(ceil(__ddiv_rn(m, delta)));
        i = jump > i + 1 ? jump : i + 1;
        while (m > __dmul_rn(static_cast<double>(i), delta)) ++i;
      }
      const double thr = __dmul_rn(static_cast<double>(i), delta);
      if (tid == 0) sh.iter = i;  // every thread read sh.iter before block_min's barrier

      // P2 + P3: group bitmask/list and min-cost goal member (planner.cpp:137-149).
      double gc = kInf;
      int32_t gv = kNone;
      for (int w = warp; w < W; w += nw) {
        const uint32_t ow = open_w[w];
        const int v = w * 32 + lane;
        const bool g = ((ow >> lane) & 1u) && cost_s[v] <= thr;
        const uint32_t gb = __ballot_sync(kFull, g);
        if (gb) {
          // Every CTA sees the whole group; the members of words it owns go
          // to its P4 work list (list order is arbitrary, ownership is not).
          int base = 0;
          const bool own = (w & (CS - 1)) == rank;
          if (lane == 0) {
            group_w[w] = gb;
            atomicAdd(&sh.group_count, __popc(gb));
            if (own) base = atomicAdd(&sh.own_count, __popc(gb));
          }
          base = __shfl_sync(kFull, base, 0);
          if (g) {
            if (own) list[base + __popc(gb & ((1u << lane) - 1u))] = static_cast<ListT>(v);
            if ((goal_w[w] >> lane) & 1u) argmin_step(gc, gv, cost_s[v], v);
          }
        }
      }
      block_argmin(gc, gv, sh, lane, warp, nw);
      if (gv != kNone) {  // planner.cpp:150-156
        status = 0;
        goal = gv;
        break;
      }
    }

#ifdef GMT_PHASE_TIMING
    if (tid == 0) { const long long t_ = clock64(); sh_ph[0] += static_cast<unsigned long long>(t_ - ph_t); ph_t = t_; }
    const long long w_p4 = clock64();
#endif
    // Rows are processed kRows at a time per warp: lane group h (lanes
    // kLanesPerRow*h ...) streams row k + h, so kRows rows' loads are in
    // flight together.
    const int h = lane / kLanesPerRow, hl = lane % kLanesPerRow;

    // P4: mark unexplored out-neighbours of the owned group members
    // (planner.cpp:159-166).
    {
      const int own = sh.own_count;
      int k = kRows * warp;
      int64_t e0 = 0;
      int len = 0;
      // Shared-pool views: a vertex's out-row is its pool row mapped through
      // the rank map (ext = the row's edges into g / init, code bits 1 / 3),
      // or g's / init's own list (rowp, already in query ids).
      const int32_t* rowp = nullptr;
      int ext = 0;
      auto pool_out_row = [&](int g, int64_t* pe0, int* plen, const int32_t** prow, int* pext) {
        const int nv = I.n - 1;  // init = n (the vertex count is n + 1)
        if (g == nv || (PV.subst && g == nv - 1)) {
          const int l = g == nv ? 2 : 0;
          *prow = PV.scol + static_cast<int64_t>(l) * PV.cap;
          *pe0 = 0;
          *plen = PV.spec_len[l];
          *pext = 0;
        } else {
          const int p = __ldg(PV.sel + g);
          *pe0 = __ldg(PV.out_ptr + p);
          *plen = static_cast<int>(__ldg(PV.out_ptr + p + 1) - *pe0);
          *prow = nullptr;
          *pext = __ldg(PV.code + g);
        }
      };
      if (k + h < own) {
        const int g = list[k + h];
        if (viewed) {
          pool_out_row(g, &e0, &len, &rowp, &ext);
        } else {
          e0 = __ldg(I.out_ptr + g);
          len = static_cast<int>(__ldg(I.out_end + g) - e0);
        }
      }
      while (k < own) {
        // Clusters take the next row pair from a shared counter (their few,
        // uneven rows balance better); batched CTAs stride statically.
        int kn = k + kRows * nw;
        if constexpr (kDynOwn) {
          if (lane == 0) kn = atomicAdd(&sh.next_own, kRows);
          kn = __shfl_sync(kFull, kn, 0);
        }
        int64_t n0 = 0;
        int nlen = 0;
        const int32_t* nrowp = nullptr;
        int next_ext = 0;
        if (kn + h < own) {  // next rows' offsets in flight during these rows
          const int gn = list[kn + h];
          if (viewed) {
            pool_out_row(gn, &n0, &nlen, &nrowp, &next_ext);
          } else {
            n0 = __ldg(I.out_ptr + gn);
            nlen = static_cast<int>(__ldg(I.out_end + gn) - n0);
          }
        }
        const int lmax = rows_max<kRows>(len);
        if (counting && hl == 0 && len > 0) atomicAdd(&sh.cnt_out, static_cast<unsigned long long>(len));
        const bool mapped = viewed && rowp == nullptr;  // pool row: entries are pool points
        const int32_t* ocol = (viewed ? (rowp ? rowp : PV.out_col + e0) : I.out_col + e0) + hl;
        const int lim = len - hl;
#if GMT_POOL_HOIST
        const uint16_t* const pv_rank = PV.rank;
        const int pv_kc = PV.kc;
#endif
        if (viewed && hl == 0 && ext) {  // the row's edges into g (n - 1) and init (n)
          if (PV.subst && (ext & 2)) atomicOr(cand_w + ((I.n - 2) >> 5), 1u << ((I.n - 2) & 31));
          if (ext & 8) atomicOr(cand_w + ((I.n - 1) >> 5), 1u << ((I.n - 1) & 31));
        }
        for (int off = 0; off < lmax; off += kLanesPerRow * kUnroll) {
          int xs[kUnroll];
#pragma unroll
          for (int u = 0; u < kUnroll; ++u)
            xs[u] = off + u * kLanesPerRow < lim
                        ? ((kRowsCs && !viewed) ? __ldcs(ocol + off + u * kLanesPerRow) : __ldg(ocol + off + u * kLanesPerRow))
                        : -1;
          if (mapped) {
#if GMT_POOL_HOIST
#pragma unroll
            for (int u = 0; u < kUnroll; ++u) {
              const int y = xs[u];
              const uint16_t r = (y >= 0 && y < pv_kc) ? __ldg(pv_rank + y) : kPoolNoRank;
              xs[u] = r == kPoolNoRank ? -1 : static_cast<int>(r);
            }
#else
#pragma unroll
            for (int u = 0; u < kUnroll; ++u)
              if (xs[u] >= 0) xs[u] = pool_rank(xs[u]);
#endif
          }
#pragma unroll
          for (int u = 0; u < kUnroll; ++u) {
            if (off + u * kLanesPerRow >= lmax) break;  // warp-uniform
            const int x = xs[u];
            const bool valid = x >= 0;
            if constexpr (CS == 1) {
              // One CTA: a shared-memory atomic per edge; explored targets
              // are masked out when the candidate list is built.
              if (valid) atomicOr(cand_w + (x >> 5), 1u << (x & 31));
              continue;
            }
            const int w = valid ? (x >> 5) : (-1 - lane);
            uint32_t bit = 0u;
            if (valid && !(((open_w[w] | closed_w[w]) >> (x & 31)) & 1u)) bit = 1u << (x & 31);
            // Each half's row is sorted, so equal words form runs: suffix-OR
            // each run into its first lane, which sets the word once (an
            // equal word in the other half only adds more of its own bits).
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
              const uint32_t ob = __shfl_down_sync(kFull, bit, o);
              const int ow = __shfl_down_sync(kFull, w, o);
              if (lane + o < 32 && ow == w) bit |= ob;
            }
            const int pw = __shfl_up_sync(kFull, w, 1);
            if ((lane == 0 || pw != w) && bit) {
              atomicOr(remote<CS>(cand_w, w & (CS - 1)) + w, bit);
            }
          }
        }
        k = kn;
        e0 = n0;
        len = nlen;
        rowp = nrowp;
        ext = next_ext;
      }
    }
#ifdef GMT_PHASE_TIMING
    if (lane == 0) atomicAdd(&sh_ph[7], static_cast<unsigned long long>(clock64() - w_p4));
#endif
    cluster_barrier<CS>();  // [1] candidate marks complete
#ifdef GMT_PHASE_TIMING
    if (tid == 0) { const long long t_ = clock64(); sh_ph[1] += static_cast<unsigned long long>(t_ - ph_t); ph_t = t_; }
#endif

    // Own candidates (words w = rank mod CS) -> list.
    for (int w = rank + CS * tid; w < W; w += CS * nt) {
      uint32_t bits = cand_w[w];
      if (bits) {
        cand_w[w] = 0u;
        if constexpr (CS == 1) bits &= ~(open_w[w] | closed_w[w]);
        int base = atomicAdd(&sh.cand_count, __popc(bits));
        while (bits) {
          const int b = __ffs(bits) - 1;
          bits &= bits - 1u;
          list[base++] = static_cast<ListT>(w * 32 + b);
        }
      }
    }
    __syncthreads();
    const int ccount = sh.cand_count;
#ifdef GMT_PHASE_TIMING
    if (tid == 0) { const long long t_ = clock64(); sh_ph[2] += static_cast<unsigned long long>(t_ - ph_t); ph_t = t_; }
#endif

    // P5 + P6: connect_candidate (planner.cpp:62-90) and commit (178-189).
    // Half h scans candidate k + h's in-row and reduces its (cost, position)
    // argmin; then the whole warp lazily checks the two chosen edges in turn.
#ifdef GMT_PHASE_TIMING
    long long w_bar = 0;
#endif
    {
#ifdef GMT_PHASE_TIMING
      const long long w_p5 = clock64();
      unsigned long long w_chk = 0;
#endif
      double* segh = seg + 32 * h;  // group h's segment: a = [0..15], b = [16..31]
      int k = kRows * warp;
      int x = -1;
      int64_t e0 = 0;
      int len = 0;
      // Shared-pool views: the candidate's in-row is its pool row (mapped,
      // then its edges from g / init, code bits 0 / 2, at positions len,
      // len + 1) or, for g, its own in-list.  (init is open from the start,
      // so it is never a candidate.)
      int ext = 0;
      bool spec_row = false;
      auto pool_in_row = [&](int xv, int64_t* pe0, int* plen, bool* pspec, int* pext) {
        if (PV.subst && xv == I.n - 2) {
          *pspec = true;
          *pe0 = 0;
          *plen = PV.spec_len[1];
          *pext = 0;
        } else {
          const int p = __ldg(PV.sel + xv);
          *pspec = false;
          *pe0 = __ldg(PV.in_ptr + p);
          *plen = static_cast<int>(__ldg(PV.in_ptr + p + 1) - *pe0);
          *pext = __ldg(PV.code + xv);
        }
      };
      if (k + h < ccount) {
        x = list[k + h];
        if (viewed) {
          pool_in_row(x, &e0, &len, &spec_row, &ext);
        } else {
          e0 = __ldg(I.in_ptr + x);
          len = static_cast<int>(__ldg(I.in_end + x) - e0);
        }
      }
      // (Staging each group's next in-row into shared memory with cp.async
      // while the current candidate is checked measured slower: 21.0 -> 24.6
      // ms rows, 27.2 -> 35.2 ms views per 4096 configs[4] queries with 64
      // entries per group -- the L1 carve-out it takes and the registers.)
      // (batched DI) the candidate's coordinates are loaded one iteration
      // ahead, with the next row's offsets
      constexpr bool kXAhead = GMT_DI_XAHEAD && D == 6 && kRows >= 2 && kLanesPerRow >= 6;
      double xcrd = 0.0;
      if constexpr (kXAhead) {
        if (x >= 0 && hl < 6) xcrd = __ldg(I.coords + static_cast<int64_t>(x) * 6 + hl);
      }
      while (k < ccount) {
        int kn = k + kRows * nw;
        if constexpr (kDynamic) {
          if (lane == 0) kn = atomicAdd(&sh.next_cand, kRows);
          kn = __shfl_sync(kFull, kn, 0);
        }
        int xn = -1;
        int64_t n0 = 0;
        int nlen = 0;
        int next_ext = 0;
        bool next_spec = false;
        if (kn + h < ccount && viewed) {
          xn = list[kn + h];
          pool_in_row(xn, &n0, &nlen, &next_spec, &next_ext);
        } else if (kn + h < ccount) {
          xn = list[kn + h];
          n0 = __ldg(I.in_ptr + xn);
          nlen = static_cast<int>(__ldg(I.in_end + xn) - n0);
          if constexpr (D == 6 && kRows >= 2) {
            // (DI: a lazy check outlasts a row fetch -- the next rows are
            // pulled into L2 by the TMA engine meanwhile; an evict-first
            // cache policy on these prefetches measured 20.79 -> 20.84 ms)
            // (not in_tau: one duration per row is read, after the argmin)
            if (hl == 0 && I.in_tau && nlen > 0) {
              prefetch_l2(I.in_col + n0, sizeof(int32_t) * nlen);
              prefetch_l2(I.in_cost + n0, sizeof(double) * nlen);
              if (I.in_pe) prefetch_l2(I.in_pe + n0, sizeof(int32_t) * nlen);
            }
          }
        }
        double nxcrd = 0.0;
        if constexpr (kXAhead) {
          if (xn >= 0 && hl < 6) nxcrd = __ldg(I.coords + static_cast<int64_t>(xn) * 6 + hl);
        }
        // The segment's B endpoint (the candidate) is staged while the row
        // streams in; the A endpoint (the chosen parent) after the argmin.
        __syncwarp();
        if constexpr (kXAhead) {
          if (x >= 0 && hl < 6) segh[16 + hl] = xcrd;
        } else if constexpr (kLanesPerRow >= kMaxSolveDim) {
          if (x >= 0 && hl < d) segh[16 + hl] = __ldg(I.coords + static_cast<int64_t>(x) * d + hl);
        } else {
          for (int t = hl; x >= 0 && t < d; t += kLanesPerRow)
            segh[16 + t] = __ldg(I.coords + static_cast<int64_t>(x) * d + t);
        }
        double bv = kInf;
        int bo = -1;  // position of the lane's best edge within the row
        int by = -1;
        const int lmax = rows_max<kRows>(len);
        if (counting && hl == 0 && len > 0) atomicAdd(&sh.cnt_in, static_cast<unsigned long long>(len));
        // Lane base pointers, formed once per row: the chunk loads below are
        // then immediate offsets from them (no per-element address math).
        const bool mapped = viewed && !spec_row;
        const int32_t* rcol =
            (viewed ? (spec_row ? PV.scol + PV.cap : PV.in_col + e0) : I.in_col + e0) + hl;
        const double* rcost =
            (viewed ? (spec_row ? PV.scost + PV.cap : PV.in_cost + e0) : I.in_cost + e0) + hl;
        const int lim = len - hl;  // element u of chunk `off` exists iff off + u * kLanesPerRow < lim
#if GMT_POOL_HOIST
        const uint16_t* const pv_rank = PV.rank;
        const int pv_kc = PV.kc;
#endif
        for (int off = 0; off < lmax; off += kLanesPerRow * kUnroll) {
          int ys[kUnroll];
          double cs[kUnroll];
          if (kRowsCs && !viewed) {
            // (materialised rows are read once per launch: evict-first in
            // L2, so the pool check records and row offsets stay resident)
#pragma unroll
            for (int u = 0; u < kUnroll; ++u) {
              const bool in = off + u * kLanesPerRow < lim;
              ys[u] = in ? __ldcs(rcol + off + u * kLanesPerRow) : -1;
              cs[u] = in ? __ldcs(rcost + off + u * kLanesPerRow) : 0.0;
            }
          } else {
#pragma unroll
            for (int u = 0; u < kUnroll; ++u) {
              const bool in = off + u * kLanesPerRow < lim;
              ys[u] = in ? __ldg(rcol + off + u * kLanesPerRow) : -1;
              cs[u] = in ? __ldg(rcost + off + u * kLanesPerRow) : 0.0;
            }
          }
          if (mapped) {
#if GMT_POOL_HOIST
            // (the map's base and length from registers: pool_rank reloads
            // them from the shared descriptor for every element)
#pragma unroll
            for (int u = 0; u < kUnroll; ++u) {
              const int y = ys[u];
              const uint16_t r = (y >= 0 && y < pv_kc) ? __ldg(pv_rank + y) : kPoolNoRank;
              ys[u] = r == kPoolNoRank ? -1 : static_cast<int>(r);
            }
#else
#pragma unroll
            for (int u = 0; u < kUnroll; ++u)
              if (ys[u] >= 0) ys[u] = pool_rank(ys[u]);
#endif
          }
#pragma unroll
          for (int u = 0; u < kUnroll; ++u) {
            // Branch-free: the open bit and the (always in-bounds) cost
            // gather are formed for every element, the min update predicated.
            const int y = ys[u];
            const int ys0 = y >= 0 ? y : 0;
            const bool op = y >= 0 && ((open_w[ys0 >> 5] >> (ys0 & 31)) & 1u);
            if constexpr (COUNT || CS > 1) cnt_open += op ? 1 : 0;
            const double c = __dadd_rn(cost_s[ys0], cs[u]);
            if (op && c < bv) {
              bv = c;
              bo = off + u * kLanesPerRow + hl;
              by = y;
            }
          }
        }
        if (viewed && hl == 0 && x >= 0 && ext) {
          // the in-edges from g (n - 1) and init (n): positions after the row
          int pos = len;
          for (int t = 0; t < 2; ++t) {
            const bool has = t == 0 ? (PV.subst && (ext & 1)) : ((ext & 4) != 0);
            if (!has) continue;
            const int y = t == 0 ? I.n - 2 : I.n - 1;
            const int l = t == 0 ? 0 : 2;
            const int j = __ldg(PV.spj + 2 * x + t);
            const bool op = (open_w[y >> 5] >> (y & 31)) & 1u;
            if constexpr (COUNT || CS > 1) cnt_open += op ? 1 : 0;
            const double c = __dadd_rn(cost_s[y], __ldg(PV.scost + static_cast<int64_t>(l) * PV.cap + j));
            if (op && c < bv) {
              bv = c;
              bo = pos;
              by = y;
            }
            ++pos;
          }
        }
        // Group argmin of (cost, position) == the reference's strict-<
        // first-in-list rule; every lane of the group ends with the result.
        if constexpr (kRows == 1) {
          // Whole warp: costs are >= 0, so their IEEE bit patterns order
          // like the values; three REDUX.MIN steps pick the smallest cost,
          // then the earliest position among exact ties.
          const unsigned long long key =
              bo >= 0 ? static_cast<unsigned long long>(__double_as_longlong(bv)) : ~0ull;
          const uint32_t khi = static_cast<uint32_t>(key >> 32), klo = static_cast<uint32_t>(key);
          const uint32_t mhi = __reduce_min_sync(kFull, khi);
          const uint32_t mlo = __reduce_min_sync(kFull, khi == mhi ? klo : 0xffffffffu);
          const bool tie = khi == mhi && klo == mlo;
          const uint32_t mbo = __reduce_min_sync(kFull, tie ? static_cast<uint32_t>(bo) : 0xffffffffu);
          if (mhi != 0xffffffffu || mlo != 0xffffffffu) {
            const int src = __ffs(__ballot_sync(kFull, tie && static_cast<uint32_t>(bo) == mbo)) - 1;
            bv = __shfl_sync(kFull, bv, src);
            by = __shfl_sync(kFull, by, src);
            bo = static_cast<int>(mbo);
          } else {
            bo = -1;
          }
        } else {
#pragma unroll
          for (int o = kLanesPerRow / 2; o; o >>= 1) {
            const double ov = __shfl_xor_sync(kFull, bv, o);
            const int oo = __shfl_xor_sync(kFull, bo, o);
            const int oy = __shfl_xor_sync(kFull, by, o);
            if (oo >= 0 && (bo < 0 || ov < bv || (ov == bv && oo < bo))) {
              bv = ov;
              bo = oo;
              by = oy;
            }
          }
        }
        // The chosen in-edge's duration (kinodynamic graphs) and both chosen
        // parents' coordinates in flight together.
        // A pool edge's check record (batched DI over the shared pool, every
        // box spanning the velocity axes): the edge's own pool in-edge.  The record
        // holds everything the check reads (the duration and the end points
        // are not loaded), so its copy starts right after the argmin.
        const double* rec_b = nullptr;
        if constexpr (D == 6 && kRows >= 2) {
          if (bo >= 0 && sh.vfull) {
            if (viewed) {
              if (PV.rec && !spec_row && bo < len) rec_b = PV.rec + (e0 + bo) * PV.rec_len;
            } else if (I.in_pe) {
              // (loading it for every best update during the scan measured
              // slower: 23.8 vs 22.0 ms, register pressure in the scan loop)
              const int32_t pe = __ldg(I.in_pe + e0 + bo);
              if (pe >= 0) rec_b = I.pool_rec + static_cast<int64_t>(pe) * I.pool_rec_len;
            }
          }
        }
        double tau_b = 0.0;
        if ((D == 0 || D == 6) && bo >= 0 && !rec_b && I.in_tau) tau_b = __ldg(I.in_tau + e0 + bo);
        if (viewed && bo >= 0 && !rec_b) {
          if (spec_row) {
            tau_b = __ldg(PV.stau + PV.cap + bo);
          } else if (bo < len) {
            tau_b = __ldg(PV.in_tau + e0 + bo);
          } else {  // an edge from g or init (at len: g when present, else init)
            const int t = (bo == len && PV.subst && (ext & 1)) ? 0 : 1;
            const int j = __ldg(PV.spj + 2 * x + t);
            tau_b = __ldg(PV.stau + static_cast<int64_t>(t == 0 ? 0 : 2) * PV.cap + j);
          }
        }
        if constexpr (kLanesPerRow >= kMaxSolveDim) {
          if (bo >= 0 && hl < d) segh[hl] = __ldg(I.coords + static_cast<int64_t>(by) * d + hl);
        } else {
          for (int t = hl; bo >= 0 && !rec_b && t < d; t += kLanesPerRow)
            segh[t] = __ldg(I.coords + static_cast<int64_t>(by) * d + t);
        }
        __syncwarp();
        // Batched double-integrator solves: the two candidates are checked
        // concurrently, one per half warp (their row scans and argmins
        // already are); the values of half h are its own lanes'.
        if constexpr (D == 6 && kRows >= 2) {
          if ((I.in_tau || viewed) && (I.kin_segments + 1) * 6 <= kTabCap && I.kin_segments <= 14) {
            constexpr uint32_t kGroup = kLanesPerRow == 32 ? 0xffffffffu : ((1u << kLanesPerRow) - 1u);
            const uint32_t gmask = kGroup << (kLanesPerRow * h);
            if (bo >= 0) {
              if (hl == 0) atomicAdd(&sh.wchecks[warp], 1);
#ifdef GMT_PHASE_TIMING
              const long long w_c0 = clock64();
#endif
              const bool ok = di_edge_free_half<kLanesPerRow, !GS && GMT_SB_VIEWS>(
                  I, bx_s, tau_b, hl, gmask, kLanesPerRow * h, segh, tab_s + (warp * kRows + h) * kTabCap,
                  cull_s + (warp * kRows + h) * kCullCap, kCullCap, sh.vfull,
                  (kDynScratch && sh.xsorted) ? sh.box_wx : -1.0, rec_b,
                  (kDynScratch && sh.xsorted && GMT_DI_XBUCKET) ? sh.xfirst : nullptr);
#ifdef GMT_PHASE_TIMING
              if (lane == 0) w_chk += clock64() - w_c0;
#endif
              if (ok && hl == 0) {
                atomicAdd(&sh.wadded[warp], 1);
                cost_s[x] = bv;
                atomicOr(newopen_w + (x >> 5), 1u << (x & 31));
                R.parent[x] = by;
                if (R.iter_added) R.iter_added[x] = sh.iter;
              }
            }
            __syncwarp();
            k = kn;
            x = xn;
            xcrd = nxcrd;
            e0 = n0;
            len = nlen;
            ext = next_ext;
            spec_row = next_spec;
            continue;
          }
        }
#pragma unroll 1
        for (int c = 0; c < kRows; ++c) {
          const int src = kLanesPerRow * c;
          // (one row per warp: the values are already warp-uniform)
          const int boc = kRows == 1 ? bo : __shfl_sync(kFull, bo, src);
          if (boc < 0) continue;  // no open in-neighbour (or no candidate): not checked
          const int xc = kRows == 1 ? x : __shfl_sync(kFull, x, src);
          const int byc = kRows == 1 ? by : __shfl_sync(kFull, by, src);
          const double bvc = kRows == 1 ? bv : __shfl_sync(kFull, bv, src);
          const int64_t bec = (kRows == 1 ? e0 : __shfl_sync(kFull, e0, src)) + boc;
          double* sc = seg + 32 * c;
          if (lane == 0) ++sh.wchecks[warp];
          const int32_t pid = I.in_path ? __ldg(I.in_path + bec) : -1;
          auto edge_free = [&](const Boxes& B) -> bool {
            if ((D == 0 || D == 6) && I.in_tau) {  // kinodynamic: regenerated polyline (di.cuh, quad.cuh)
              const double tc = kRows == 1 ? tau_b : __shfl_sync(kFull, tau_b, src);
              // the endpoints are staged in sc when a lane group can hold them
              return kino_edge_free_warp<D>(I, B, byc, xc, tc, lane, sc,
                                            tab_s + ((D == 0 || D == 6) ? warp * kTabCap * kKinSlots : 0), kTabCap,
                                            cull_s + warp * kCullCap * kKinSlots, kCullCap, true, D == 6 && sh.vfull,
                                            bec);
            }
            if (pid < 0) return segment_free_staged<D>(d, B, lane, sc);  // segment_free (planner.cpp:59)
            return polyline_free_warp<D>(I, d, B, pid, lane, sc);       // polyline_free (planner.cpp:56-58)
          };
          bool ok;
          if constexpr (WIDE) {  // registers to spare: the descriptor off the check's critical path
            const Boxes breg = bx_s;
            ok = edge_free(breg);
          } else {
            ok = edge_free(bx_s);
          }
          if (ok) {
            if (lane == 0) ++sh.wadded[warp];
            if (lane < CS) {
              remote<CS>(cost_s, lane)[xc] = bvc;
              atomicOr(remote<CS>(newopen_w, lane) + (xc >> 5), 1u << (xc & 31));
            }
            if (lane == 0) {
              if constexpr (kParentSmem) {
                remote<CS>(parent_s, 0)[xc] = static_cast<uint16_t>(byc);
              } else {
                R.parent[xc] = byc;
              }
              if (R.iter_added) R.iter_added[xc] = sh.iter;
            }
          }
        }
        k = kn;
        x = xn;
        xcrd = nxcrd;
        e0 = n0;
        len = nlen;
        ext = next_ext;
        spec_row = next_spec;
      }
#ifdef GMT_PHASE_TIMING
      if (lane == 0) {
        atomicAdd(&sh_ph[4], static_cast<unsigned long long>(clock64() - w_p5));
        atomicAdd(&sh_ph[5], w_chk);
      }
      w_bar = clock64();
#endif
    }
    if (lane == 0) {
      const int my_checks = sh.wchecks[warp], my_added = sh.wadded[warp];
      if (my_checks | my_added) {
        atomicAdd(remote<CS>(&sh.checks_acc, 0), static_cast<unsigned long long>(my_checks));
        atomicAdd(remote<CS>(&sh.added_acc, 0), my_added);
        sh.wchecks[warp] = 0;
        sh.wadded[warp] = 0;
      }
    }
    cluster_barrier<CS>();  // [2] commits visible in every replica
#ifdef GMT_PHASE_TIMING
    if (lane == 0) atomicAdd(&sh_ph[6], static_cast<unsigned long long>(clock64() - w_bar));
    if (tid == 0) { const long long t_ = clock64(); sh_ph[3] += static_cast<unsigned long long>(t_ - ph_t); ph_t = t_; }
#endif

    if (rank == 0 && tid == 0) {  // IterationStats (planner.cpp:192-194)
      if (R.group_sizes) {
        const int p = sh.pass;
        R.group_sizes[p] = job.mode == kModeFmt ? 1 : sh.group_count;
        R.nodes_added[p] = sh.added_acc;
        R.checks[p] = static_cast<int64_t>(sh.checks_acc);
      }
      sh.total_checks += static_cast<long long>(sh.checks_acc);
      sh.added_acc = 0;
      sh.checks_acc = 0ull;
    }
    // Close the group, open the committed nodes (planner.cpp:178-190).
    for (int w = tid; w < W; w += nt) {
      const uint32_t gw = group_w[w];
      closed_w[w] |= gw;
      open_w[w] = (open_w[w] & ~gw) | newopen_w[w];
      newopen_w[w] = 0u;
      group_w[w] = 0u;
    }
    if (tid == 0) {
      sh.group_count = 0;
      sh.own_count = 0;
      sh.cand_count = 0;
      sh.iter = i + 1;
      sh.pass = sh.pass + 1;
      sh.next_own = kRows * nw;
      sh.next_cand = kRows * nw;
    }
    __syncthreads();
  }

#ifdef GMT_PHASE_TIMING
  if (tid == 0 && rank == 0 && R.counters)
    for (int k = 0; k < 8; ++k) atomicAdd(reinterpret_cast<unsigned long long*>(R.counters) + 4 + k, sh_ph[k]);
#endif
  if (counting) {
    long long c = cnt_open;
    for (int o = 16; o; o >>= 1) c += __shfl_xor_sync(kFull, c, o);
    if (lane == 0) {
      atomicAdd(reinterpret_cast<unsigned long long*>(R.counters + 2), static_cast<unsigned long long>(c));
    }
    if (tid == 0) {
      atomicAdd(reinterpret_cast<unsigned long long*>(R.counters + 0), sh.cnt_in);
      atomicAdd(reinterpret_cast<unsigned long long*>(R.counters + 1), sh.cnt_out);
    }
  }
  if (rank != 0) return;
  // Outputs (rank 0 holds the parent replica, or the parents are in HBM).
  if (R.label) {
    for (int v = tid; v < n; v += nt) {
      const uint32_t bit = 1u << (v & 31);
      R.label[v] = (open_w[v >> 5] & bit) ? 1 : ((closed_w[v >> 5] & bit) ? 2 : 0);
      R.tree_cost[v] = cost_s[v];
      if constexpr (kParentSmem) R.parent[v] = parent_s[v] == 0xffffu ? -1 : parent_s[v];
    }
  }
  if (tid == 0) {
    ResultScalars s;
    s.status = status;
    s.goal_node = goal;
    const int pass = sh.pass;
    s.iterations = sh.iter;
    s.tree_size = n;
    s.reserved = 0;
    s.num_stats = pass;
    s.total_checks = sh.total_checks;
    if (status == 0) {
      if (R.group_sizes) {  // final group pushes 0/0 (planner.cpp:151-152)
        R.group_sizes[pass] = sh.group_count;
        R.nodes_added[pass] = 0;
        R.checks[pass] = 0;
      }
      s.num_stats = pass + 1;
      s.cost = cost_s[goal];
      // finalize_success (planner.cpp:43-50): walk the parents.
      auto par = [&](int v) -> int {
        if constexpr (kParentSmem) {
          return parent_s[v] == 0xffffu ? -1 : parent_s[v];
        } else {
          return R.parent[v];
        }
      };
      int len = 0;
      for (int v = goal; v >= 0; v = par(v)) ++len;
      int k = len;
      if (R.path) {
        for (int v = goal; v >= 0; v = par(v)) R.path[--k] = v;
      }
      s.path_len = len;
    } else {
      s.cost = kInf;
      s.path_len = 0;
    }
    *R.scalars = s;
  }
}

// ---- dijkstra_oracle (planner.cpp:264-334) -------------------------------------
// Eager phase: every out-edge's motion is checked up front, warp per row,
// lanes per box (the same exact segment / polyline / trajectory tests the
// lazy check uses).  Euclidean graphs are symmetric: edge (u, v) with v < u
// reuses the check of (v, u), i.e. segment_free(x_v, x_u), and is not
// counted (planner.cpp:283-292).
template <int D>
__global__ void __launch_bounds__(256) eager_check_kernel(const DevInstance* __restrict__ inst,
                                                          uint8_t* __restrict__ ok,
                                                          unsigned long long* __restrict__ checks) {
  __shared__ DevInstance I_s;
  __shared__ Boxes bx_s;
  __shared__ double seg_s[8 * 32];
  if (threadIdx.x == 0) {
    I_s = *inst;
    Boxes b;
    b.lo = I_s.box_lo;
    b.hi = I_s.box_hi;
    b.lom = nullptr;
    b.him = nullptr;
    b.idx = nullptr;
    b.full = nullptr;
    b.bs = I_s.dim;
    b.as = 1;
    b.count = I_s.num_boxes;
    bx_s = b;
  }
  __syncthreads();
  const DevInstance& I = I_s;
  const int d = dims<D>(I.dim);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double* seg = seg_s + warp * 32;
  const bool symmetric = !I.directed;
  unsigned long long mine = 0;
  for (int u = blockIdx.x * 8 + warp; u < I.n; u += gridDim.x * 8) {
    for (int64_t e = I.out_ptr[u]; e < (I.out_end ? I.out_end[u] : I.out_ptr[u + 1]); ++e) {
      const int v = I.out_col[e];
      const int a = (symmetric && v < u) ? v : u, b = (symmetric && v < u) ? u : v;
      if (!(symmetric && v < u)) ++mine;
      bool free;
      if ((D == 0 || D == 6) && I.out_tau) {
        free = kino_edge_free_warp<D>(I, bx_s, u, v, I.out_tau[e], lane, seg);
      } else if (I.out_path) {
        free = polyline_free_warp<D>(I, d, bx_s, I.out_path[e], lane, seg);
      } else {
        free = segment_free_warp<D>(I.coords + static_cast<int64_t>(a) * d,
                                    I.coords + static_cast<int64_t>(b) * d, d, bx_s, lane, seg);
      }
      if (lane == 0) ok[e] = free ? 1 : 0;
    }
  }
  if (lane == 0 && mine) atomicAdd(checks, mine);
}

// segment_free / point_free (space.cpp:47-90) for `count` independent
// segments against one obstacle set, warp per segment: the very
// segment_free_ab the lazy checks run (the gmt_segment_free entry point).
template <int D>
__global__ void __launch_bounds__(256) segment_free_kernel(const double* __restrict__ a,
                                                           const double* __restrict__ b, int64_t count,
                                                           int d, const double* __restrict__ box_lo,
                                                           const double* __restrict__ box_hi, int nb,
                                                           uint8_t* __restrict__ out) {
  __shared__ double seg_s[8 * 32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double* seg = seg_s + warp * 32;
  Boxes bx;
  bx.lo = box_lo;
  bx.hi = box_hi;
  bx.lom = nullptr;
  bx.him = nullptr;
  bx.idx = nullptr;
  bx.full = nullptr;
  bx.bs = d;
  bx.as = 1;
  bx.count = nb;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * 8 + warp; i < count;
       i += static_cast<int64_t>(gridDim.x) * 8) {
    const bool free = segment_free_warp<D>(a + i * d, b + i * d, d, bx, lane, seg);
    if (lane == 0) out[i] = free ? 1 : 0;
  }
}

// Build-time waypoint tables of a kinodynamic instance's in-edges (the
// reference caches every edge's polyline when it builds the graph, graph.cpp
// edge_path): in-edge e = (in_col[e] -> x) gets rows 0..M of its trajectory
// from kino_fill_table, the very fill the solve's lazy check would run, so a
// check that reads the table sees the values it would have computed.  One
// warp per in-edge, a CTA per target vertex.
__global__ void __launch_bounds__(256) kino_table_kernel(const double* __restrict__ coords,
                                                         const int64_t* __restrict__ in_ptr,
                                                         const int32_t* __restrict__ in_col,
                                                         const double* __restrict__ in_tau, int n, int steering,
                                                         QuadParams QP, DiParams DP, double* __restrict__ wp) {
  __shared__ double seg_s[8][32];
  __shared__ double tab_s[8][144];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const bool quad = steering == GMT_STEER_QUADROTOR;
  const int dim = quad ? kQuadDim : kDiDim;
  const int M = quad ? QP.segments : DP.segments;
  const int W = (M + 1) * dim;
  double* seg = seg_s[warp];
  double* tab = tab_s[warp];
  for (int x = blockIdx.x; x < n; x += gridDim.x) {
    const int64_t e1 = in_ptr[x + 1];
    for (int64_t e = in_ptr[x] + warp; e < e1; e += 8) {
      const int u = in_col[e];
      const double tau = in_tau[e];
      __syncwarp();
      for (int j = lane; j < W; j += kWarp) tab[j] = 0.0;
      __syncwarp();
      if (lane < dim) {
        tab[lane] = coords[static_cast<int64_t>(u) * dim + lane];
        tab[M * dim + lane] = coords[static_cast<int64_t>(x) * dim + lane];
      }
      __syncwarp();
      if (tau != 0.0) kino_fill_table<0>(quad, dim, M, tau, lane, seg, tab, QP, DP, false);
      __syncwarp();
      for (int j = lane; j < W; j += kWarp) wp[e * W + j] = tab[j];
    }
  }
}

cudaError_t launch_kino_tables(const double* coords, const int64_t* in_ptr, const int32_t* in_col,
                               const double* in_tau, int n, int steering, const QuadParams& QP,
                               const DiParams& DP, double* wp, int sm_count, cudaStream_t stream) {
  if (n <= 0) return cudaSuccess;
  const int blocks = std::max(1, std::min(n, sm_count * 8));
  kino_table_kernel<<<blocks, 256, 0, stream>>>(coords, in_ptr, in_col, in_tau, n, steering, QP, DP, wp);
  return cudaGetLastError();
}

cudaError_t launch_segment_free(const double* a, const double* b, int64_t count, int d,
                                const double* box_lo, const double* box_hi, int nb, uint8_t* out,
                                int sm_count, cudaStream_t stream) {
  if (count <= 0) return cudaSuccess;
  const int blocks = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>((count + 7) / 8, sm_count * 8)));
  switch (d) {
    case 2: segment_free_kernel<2><<<blocks, 256, 0, stream>>>(a, b, count, d, box_lo, box_hi, nb, out); break;
    case 3: segment_free_kernel<3><<<blocks, 256, 0, stream>>>(a, b, count, d, box_lo, box_hi, nb, out); break;
    case 6: segment_free_kernel<6><<<blocks, 256, 0, stream>>>(a, b, count, d, box_lo, box_hi, nb, out); break;
    default: segment_free_kernel<0><<<blocks, 256, 0, stream>>>(a, b, count, d, box_lo, box_hi, nb, out); break;
  }
  return cudaGetLastError();
}

// Search phase: Dijkstra over the surviving edges from init, one CTA.  The
// reference's heap pops unsettled nodes in lexicographic (tentative cost,
// index) order, so each pop is a block argmin over the open nodes; the row
// of the popped node relaxes in parallel (each target appears once per row).
// Labels / costs / parents live in the result arrays (HBM).
template <int D>
__global__ void __launch_bounds__(1024) dijkstra_kernel(const SolveJob* __restrict__ jobs,
                                                        const uint8_t* __restrict__ ok,
                                                        const unsigned long long* __restrict__ checks) {
  __shared__ CtaShared sh;
  __shared__ double seg_s[32];
  __shared__ DevInstance I_s;
  __shared__ Boxes bx_s;
  const SolveJob job = jobs[blockIdx.x];
  if (threadIdx.x == 0) {
    I_s = *job.inst;
    Boxes b;
    b.lo = I_s.box_lo;
    b.hi = I_s.box_hi;
    b.lom = nullptr;
    b.him = nullptr;
    b.idx = nullptr;
    b.full = nullptr;
    b.bs = I_s.dim;
    b.as = 1;
    b.count = I_s.num_boxes;
    bx_s = b;
  }
  __syncthreads();
  const DevInstance& I = I_s;
  const DevResult& R = job.res;
  const int n = I.n, d = dims<D>(I.dim);
  const int tid = threadIdx.x, nt = blockDim.x, lane = tid & 31, warp = tid >> 5, nw = nt >> 5;
  const int init = job.init_index;
  if (warp == 0) {  // infeasible_input (planner.cpp:39-41, 269): empty tree
    const bool feas = I.goal_count > 0 &&
                      point_free_warp<D>(I.coords + static_cast<int64_t>(init) * d, d, bx_s, lane, seg_s);
    if (lane == 0) sh.feasible = feas ? 1 : 0;
  }
  __syncthreads();
  if (!sh.feasible) {
    if (tid == 0) {
      ResultScalars s{};
      s.status = 2;
      s.goal_node = -1;
      s.cost = kInf;
      *R.scalars = s;
    }
    return;
  }
  for (int v = tid; v < n; v += nt) {  // make_wavefront (planner.cpp:25-35)
    R.label[v] = v == init ? 1 : 0;
    R.tree_cost[v] = v == init ? 0.0 : kInf;
    R.parent[v] = -1;
    R.iter_added[v] = v == init ? 0 : -1;
  }
  __syncthreads();
  long long pops = 0;
  int status = 1, goal = -1;
  for (;;) {
    double zc = kInf;
    int32_t z = kNone;
    for (int v = tid; v < n; v += nt)
      if (R.label[v] == 1) argmin_step(zc, z, R.tree_cost[v], v);
    block_argmin(zc, z, sh, lane, warp, nw);
    if (z == kNone) break;  // failure_open_empty
    ++pops;
    __syncthreads();  // every thread has read the labels before z closes
    if (tid == 0) R.label[z] = 2;
    if (box_contains(I.goal_lo, I.goal_hi, d, I.coords + static_cast<int64_t>(z) * d)) {
      status = 0;
      goal = z;
      break;
    }
    const double cz = R.tree_cost[z];
    for (int64_t e = I.out_ptr[z] + tid; e < (I.out_end ? I.out_end[z] : I.out_ptr[z + 1]); e += nt) {
      if (!ok[e]) continue;
      const int v = I.out_col[e];
      if (v == z || R.label[v] == 2) continue;
      const double c = __dadd_rn(cz, I.out_cost[e]);
      if (c < R.tree_cost[v]) {
        R.tree_cost[v] = c;
        R.parent[v] = z;
        if (R.label[v] == 0) R.label[v] = 1;
      }
    }
    __syncthreads();
  }
  __syncthreads();
  if (tid == 0) {
    ResultScalars s{};
    s.status = status;
    s.goal_node = goal;
    s.iterations = pops;
    s.total_checks = static_cast<long long>(*checks);
    s.tree_size = n;
    s.num_stats = 0;  // the reference records no per-pass stats here
    if (status == 0) {
      s.cost = R.tree_cost[goal];
      int len = 0;
      for (int v = goal; v >= 0; v = R.parent[v]) ++len;
      int k = len;
      if (R.path)
        for (int v = goal; v >= 0; v = R.parent[v]) R.path[--k] = v;
      s.path_len = len;
    } else {
      s.cost = kInf;
      s.path_len = 0;
    }
    *R.scalars = s;
  }
}

template <int D>
static cudaError_t launch_dijkstra_d(const DevInstance* inst, const SolveJob* job, int n,
                                     uint8_t* ok, unsigned long long* checks, int sm_count,
                                     cudaStream_t stream) {
  const int blocks = std::max(1, std::min((n + 7) / 8, sm_count * 8));
  eager_check_kernel<D><<<blocks, 256, 0, stream>>>(inst, ok, checks);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  dijkstra_kernel<D><<<1, 1024, 0, stream>>>(job, ok, checks);
  return cudaGetLastError();
}

cudaError_t launch_dijkstra(const DevInstance* inst, const SolveJob* job, int n, int dim, uint8_t* ok,
                            unsigned long long* checks, int sm_count, cudaStream_t stream) {
  switch (dim) {
    case 2: return launch_dijkstra_d<2>(inst, job, n, ok, checks, sm_count, stream);
    case 3: return launch_dijkstra_d<3>(inst, job, n, ok, checks, sm_count, stream);
    case 6: return launch_dijkstra_d<6>(inst, job, n, ok, checks, sm_count, stream);
    default: return launch_dijkstra_d<0>(inst, job, n, ok, checks, sm_count, stream);
  }
}

template <int CS, int D, bool WIDE, bool COUNT, bool GS = false, bool POOL = false, int NW = 0>
static cudaError_t launch_cs(const SolveJob* jobs, int count, int threads, size_t smem,
                             int obs_in_smem, cudaStream_t stream) {
  auto kern = gmt_solve_kernel<CS, D, WIDE, COUNT, GS, POOL, NW>;
  // Function attributes are process-wide: the dynamic shared-memory limit
  // only ever grows (under a lock), so concurrent launches from several host
  // threads (each with its own context / stream) never see it shrink below
  // what they need.
  static std::mutex mu;
  static size_t granted = 0;
  static bool cluster_ok = false;
  {
    std::lock_guard<std::mutex> lock(mu);
    if (smem > granted) {
      const cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                 static_cast<int>(smem));
      if (e != cudaSuccess) return e;
      granted = smem;
    }
    if (CS > 8 && !cluster_ok) {
      const cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
      if (e != cudaSuccess) return e;
      cluster_ok = true;
    }
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(static_cast<unsigned>(count) * CS, 1, 1);
  cfg.blockDim = dim3(static_cast<unsigned>(threads), 1, 1);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  if (CS > 1) {
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = CS;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
  }
  return cudaLaunchKernelEx(&cfg, kern, jobs, obs_in_smem);
}

template <int CS, bool WIDE, bool COUNT = false, bool GS = false>
static cudaError_t launch_dim(const SolveJob* jobs, int count, int threads, size_t smem,
                              int obs_in_smem, int dim, cudaStream_t stream) {
  switch (dim) {
    case 2: return launch_cs<CS, 2, WIDE, COUNT, GS>(jobs, count, threads, smem, obs_in_smem, stream);
    case 3: return launch_cs<CS, 3, WIDE, COUNT, GS>(jobs, count, threads, smem, obs_in_smem, stream);
    case 6: return launch_cs<CS, 6, WIDE, COUNT, GS>(jobs, count, threads, smem, obs_in_smem, stream);
    default: return launch_cs<CS, 0, WIDE, COUNT, GS>(jobs, count, threads, smem, obs_in_smem, stream);
  }
}

cudaError_t launch_solve(const SolveJob* jobs, int count, int cluster, int threads, size_t smem,
                         int obs_in_smem, int dim, cudaStream_t stream, bool count_traffic, bool gstate,
                         bool pool) {
  if (cluster == 1 && dim == 6 && threads == 768 && !gstate) {  // the 24-warp latency shape (D = 6)
    if (pool)
      return count_traffic ? launch_cs<1, 6, false, true, false, true, 24>(jobs, count, threads, smem, obs_in_smem, stream)
                           : launch_cs<1, 6, false, false, false, true, 24>(jobs, count, threads, smem, obs_in_smem, stream);
    return count_traffic ? launch_cs<1, 6, false, true, false, false, 24>(jobs, count, threads, smem, obs_in_smem, stream)
                         : launch_cs<1, 6, false, false, false, false, 24>(jobs, count, threads, smem, obs_in_smem, stream);
  }
  if (pool) {  // shared-pool views (batched DI queries): single CTAs
    if (cluster != 1 || dim != 6 || gstate) return cudaErrorInvalidValue;
    if (threads > 256)
      return count_traffic ? launch_cs<1, 6, true, true, false, true>(jobs, count, threads, smem, obs_in_smem, stream)
                           : launch_cs<1, 6, true, false, false, true>(jobs, count, threads, smem, obs_in_smem, stream);
    return count_traffic ? launch_cs<1, 6, false, true, false, true>(jobs, count, threads, smem, obs_in_smem, stream)
                         : launch_cs<1, 6, false, false, false, true>(jobs, count, threads, smem, obs_in_smem, stream);
  }
  if (gstate) {  // global-memory wavefront: one wide CTA per query
    if (cluster != 1 || threads != 512) return cudaErrorInvalidValue;
    return launch_dim<1, true, false, true>(jobs, count, threads, 0, obs_in_smem, dim, stream);
  }
  switch (cluster) {
    case 1:
      if (count_traffic)
        return threads > 256 ? launch_dim<1, true, true>(jobs, count, threads, smem, obs_in_smem, dim, stream)
                             : launch_dim<1, false, true>(jobs, count, threads, smem, obs_in_smem, dim, stream);
      return threads > 256 ? launch_dim<1, true>(jobs, count, threads, smem, obs_in_smem, dim, stream)
                           : launch_dim<1, false>(jobs, count, threads, smem, obs_in_smem, dim, stream);
    case 2: return launch_dim<2, true>(jobs, count, threads, smem, obs_in_smem, dim, stream);
    case 4: return launch_dim<4, true>(jobs, count, threads, smem, obs_in_smem, dim, stream);
    case 8: return launch_dim<8, true>(jobs, count, threads, smem, obs_in_smem, dim, stream);
    case 16: return launch_dim<16, true>(jobs, count, threads, smem, obs_in_smem, dim, stream);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace gmtb
