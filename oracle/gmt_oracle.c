/*
 * gmt_oracle.c -- TEST INFRASTRUCTURE ONLY: the CPU oracle (checker).
 *
 * A plain-C restatement of the reference gmtplan algorithm on the GMT* hot
 * path, written against the flat structs of include/gmt_b200.h.  Each
 * function cites the reference file:line it restates (paths relative to
 * /root/reference/proj).  It is pinned against the unmodified reference
 * (oracle/_ref/libgmtref.so) and the committed golden vectors in
 * tests/test_oracle.py before any GPU result is compared with it.
 *
 * Floating point: compiled with -ffp-contract=off and no -march, i.e. plain
 * SSE2 IEEE double arithmetic with the reference's operation order, which is
 * what the reference's own Release build does (proj/CMakeLists.txt:8-10).
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline leg may
 * call this library.  The product library never links or loads it.
 */
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "gmt_b200.h"

#ifndef M_PI
#define M_PI 3.14159265358979323846
#endif

static __thread char g_err[512];

static int fail(int code, const char* msg) {
  snprintf(g_err, sizeof g_err, "%s", msg);
  return code;
}

const char* oracle_last_error(void) { return g_err; }

/* ---- sampling.cpp:13-51 ------------------------------------------------- */
static int is_prime(uint32_t v) { /* sampling.cpp:13-19 */
  if (v < 2) return 0;
  for (uint32_t p = 2; p * p <= v; ++p)
    if (v % p == 0) return 0;
  return 1;
}

static double halton_raw(uint64_t index, uint32_t base) { /* sampling.cpp:21-34 */
  double f = 1.0, r = 0.0;
  while (index > 0) {
    f /= base;
    r += f * (double)(index % base);
    index /= base;
  }
  return r;
}

int oracle_halton(uint64_t index, uint32_t base, double* out) {
  if (index == 0) return fail(GMT_E_INVALID_INPUT, "halton index is 1-based; got 0");
  if (!is_prime(base)) return fail(GMT_E_INVALID_INPUT, "halton base must be a prime >= 2");
  *out = halton_raw(index, base);
  return GMT_OK;
}

static uint32_t nth_prime_raw(int k) { /* sampling.cpp:36-44 */
  uint32_t candidate = 1;
  for (int found = 0; found < k;) {
    ++candidate;
    if (is_prime(candidate)) ++found;
  }
  return candidate;
}

int oracle_nth_prime(int k, uint32_t* out) {
  if (k < 1) return fail(GMT_E_INVALID_INPUT, "nth_prime is 1-based");
  *out = nth_prime_raw(k);
  return GMT_OK;
}

/* ---- rng.hpp:11-33 Pcg32 ------------------------------------------------ */
typedef struct {
  uint64_t state, inc;
} pcg32;

static uint32_t pcg_next(pcg32* g) {
  uint64_t old = g->state;
  g->state = old * 6364136223846793005ULL + g->inc;
  uint32_t xorshifted = (uint32_t)(((old >> 18u) ^ old) >> 27u);
  uint32_t rot = (uint32_t)(old >> 59u);
  return (xorshifted >> rot) | (xorshifted << ((32u - rot) & 31u));
}

static void pcg_seed(pcg32* g, uint64_t seed) { /* rng.hpp:16-22, seq = 0 */
  g->state = 0u;
  g->inc = (0u << 1u) | 1u;
  pcg_next(g);
  g->state += seed;
  pcg_next(g);
}

static double pcg_double(pcg32* g) { return pcg_next(g) * 0x1p-32; } /* rng.hpp:33 */

/* ---- space.cpp ---------------------------------------------------------- */
static int box_contains(const gmt_scene* s, int b, const double* p) { /* space.cpp:11-16 */
  const int d = s->dim;
  for (int k = 0; k < d; ++k) {
    if (p[k] < s->box_lo[b * d + k] || p[k] > s->box_hi[b * d + k]) return 0;
  }
  return 1;
}

static int goal_contains(const gmt_scene* s, const double* p) {
  for (int k = 0; k < s->dim; ++k)
    if (p[k] < s->goal_lo[k] || p[k] > s->goal_hi[k]) return 0;
  return 1;
}

static int point_in_cube(const double* p, int d) { /* space.cpp:40-45 */
  for (int k = 0; k < d; ++k)
    if (p[k] < 0.0 || p[k] > 1.0) return 0;
  return 1;
}

static int point_free_raw(const gmt_scene* s, const double* p) { /* space.cpp:47-54 */
  if (!point_in_cube(p, s->dim)) return 0;
  for (int b = 0; b < s->num_boxes; ++b)
    if (box_contains(s, b, p)) return 0;
  return 1;
}

int oracle_point_free(const gmt_scene* s, const double* p, int32_t* out) {
  *out = point_free_raw(s, p);
  return GMT_OK;
}

/* Closed slab clipping, space.cpp:60-78 (std::max/std::min/std::swap). */
static int segment_hits_box(const gmt_scene* s, int b, const double* a, const double* c) {
  const int d = s->dim;
  double tmin = 0.0, tmax = 1.0;
  for (int k = 0; k < d; ++k) {
    double dk = c[k] - a[k];
    double lo = s->box_lo[b * d + k], hi = s->box_hi[b * d + k];
    if (dk == 0.0) {
      if (a[k] < lo || a[k] > hi) return 0;
    } else {
      double t0 = (lo - a[k]) / dk;
      double t1 = (hi - a[k]) / dk;
      if (t0 > t1) {
        double t = t0;
        t0 = t1;
        t1 = t;
      }
      tmin = (tmin < t0) ? t0 : tmin; /* std::max(tmin, t0) */
      tmax = (t1 < tmax) ? t1 : tmax; /* std::min(tmax, t1) */
      if (tmin > tmax) return 0;
    }
  }
  return 1;
}

static int coords_equal(const double* a, const double* b, int d) {
  for (int k = 0; k < d; ++k)
    if (!(a[k] == b[k])) return 0;
  return 1;
}

static int segment_free_raw(const gmt_scene* s, const double* a, const double* b) {
  /* space.cpp:80-90 */
  if (coords_equal(a, b, s->dim)) return point_free_raw(s, a);
  if (!point_in_cube(a, s->dim) || !point_in_cube(b, s->dim)) return 0;
  for (int k = 0; k < s->num_boxes; ++k)
    if (segment_hits_box(s, k, a, b)) return 0;
  return 1;
}

int oracle_segment_free(const gmt_scene* s, const double* a, const double* b, int32_t* out) {
  *out = segment_free_raw(s, a, b);
  return GMT_OK;
}

static int polyline_free_raw(const gmt_scene* s, const double* pts, int64_t count) {
  /* space.cpp:92-99 */
  if (count == 1) return point_free_raw(s, pts);
  for (int64_t i = 0; i + 1 < count; ++i)
    if (!segment_free_raw(s, pts + i * s->dim, pts + (i + 1) * s->dim)) return 0;
  return 1;
}

static int validate_scene(const gmt_scene* s) { /* space.cpp:18-38 */
  if (s->dim < 1) return fail(GMT_E_INVALID_INPUT, "obstacle set dimension must be >= 1");
  for (int b = 0; b < s->num_boxes; ++b)
    for (int k = 0; k < s->dim; ++k)
      if (!(s->box_lo[b * s->dim + k] <= s->box_hi[b * s->dim + k]))
        return fail(GMT_E_INVALID_INPUT, "box has lo > hi");
  for (int k = 0; k < s->dim; ++k)
    if (!(s->goal_lo[k] <= s->goal_hi[k])) return fail(GMT_E_INVALID_INPUT, "box has lo > hi");
  return GMT_OK;
}

/* ---- exact-duplicate set (the std::set<std::vector<double>> of
 *      sampling.cpp:92,106): open-addressing hash on canonical bits ------- */
typedef struct {
  const double* pts; /* stored points live in the caller's coords array */
  int32_t* slots;    /* index into pts, -1 empty */
  int64_t cap;
  int d;
} dupset;

static uint64_t hash_pt(const double* p, int d) {
  uint64_t h = 0x9e3779b97f4a7c15ULL;
  for (int k = 0; k < d; ++k) {
    double v = p[k] == 0.0 ? 0.0 : p[k]; /* -0.0 == 0.0 under std::set order */
    uint64_t bits;
    memcpy(&bits, &v, 8);
    h ^= bits + 0x9e3779b97f4a7c15ULL + (h << 6) + (h >> 2);
    h *= 0xbf58476d1ce4e5b9ULL;
  }
  return h;
}

static int64_t dup_find(const dupset* s, const double* p) {
  int64_t i = (int64_t)(hash_pt(p, s->d) & (uint64_t)(s->cap - 1));
  while (s->slots[i] >= 0) {
    if (coords_equal(s->pts + (int64_t)s->slots[i] * s->d, p, s->d)) return i;
    i = (i + 1) & (s->cap - 1);
  }
  return -1 - i;
}

/* ---- sample_free (sampling.cpp:81-142) ---------------------------------- */
int oracle_sample_free(int32_t n, const gmt_scene* scene, const gmt_sample_source* src,
                       double* coords, double* heading, int32_t* goal_idx, int32_t* goal_count) {
  if (n < 1) return fail(GMT_E_INVALID_INPUT, "sample count must be >= 1");
  int rc = validate_scene(scene);
  if (rc) return rc;
  if (src->kind == GMT_SAMPLE_HALTON && src->start_index == 0)
    return fail(GMT_E_INVALID_INPUT, "halton start_index is 1-based; got 0");
  const int d = scene->dim;
  const uint64_t budget = 1000ULL * (uint64_t)n;
  uint32_t primes[64];
  for (int k = 0; k <= d && k < 64; ++k) primes[k] = nth_prime_raw(k + 1);

  dupset set;
  set.d = d;
  set.pts = coords;
  set.cap = 1;
  while (set.cap < 4 * (int64_t)n) set.cap <<= 1;
  set.slots = (int32_t*)malloc(sizeof(int32_t) * set.cap);
  for (int64_t i = 0; i < set.cap; ++i) set.slots[i] = -1;

  pcg32 rng;
  pcg_seed(&rng, src->seed);
  uint64_t next_index = src->start_index;
  double* cand = (double*)malloc(sizeof(double) * (d + 1));
  uint64_t attempts = 0;
  int32_t kept = 0;
  while (kept < n) {
    if (attempts == budget) {
      free(set.slots);
      free(cand);
      return fail(GMT_E_INFEASIBLE_SAMPLING, "rejection budget exhausted");
    }
    ++attempts;
    double h = 0.0;
    if (src->kind == GMT_SAMPLE_HALTON) { /* CandidateStream::draw, sampling.cpp:64-76 */
      for (int k = 0; k < d; ++k) cand[k] = halton_raw(next_index, primes[k]);
      if (src->with_heading) h = halton_raw(next_index, primes[d]) * 2.0 * M_PI;
      ++next_index;
    } else {
      for (int k = 0; k < d; ++k) cand[k] = pcg_double(&rng);
      if (src->with_heading) h = pcg_double(&rng) * 2.0 * M_PI;
    }
    if (!point_free_raw(scene, cand)) continue;
    int64_t pos = dup_find(&set, cand);
    if (pos >= 0) continue;
    memcpy(coords + (int64_t)kept * d, cand, sizeof(double) * d);
    if (heading) heading[kept] = h;
    set.slots[-1 - pos] = kept;
    ++kept;
  }

  int32_t gc = 0;
  for (int i = 0; i < n; ++i) /* sampling.cpp:110-112 */
    if (goal_contains(scene, coords + (int64_t)i * d)) goal_idx[gc++] = i;
  if (gc > 0) {
    *goal_count = gc;
    free(set.slots);
    free(cand);
    return GMT_OK;
  }

  /* Goal substitution, sampling.cpp:115-141.  `seen` loses the last sample. */
  {
    int64_t pos = dup_find(&set, coords + (int64_t)(n - 1) * d);
    /* rebuild the set without slot n-1 (simplest exact erase) */
    (void)pos;
    for (int64_t i = 0; i < set.cap; ++i) set.slots[i] = -1;
    for (int i = 0; i < n - 1; ++i) {
      int64_t p = dup_find(&set, coords + (int64_t)i * d);
      if (p < 0) set.slots[-1 - p] = i;
    }
  }
  double sub_h = 0.0;
  for (int k = 0; k < d; ++k) cand[k] = 0.5 * (scene->goal_lo[k] + scene->goal_hi[k]);
  if (!point_free_raw(scene, cand) || dup_find(&set, cand) >= 0) {
    int found = 0;
    for (uint64_t i = 1; i <= budget; ++i) {
      for (int k = 0; k < d; ++k) {
        double q = halton_raw(i, primes[k]);
        cand[k] = scene->goal_lo[k] + q * (scene->goal_hi[k] - scene->goal_lo[k]);
      }
      if (!point_free_raw(scene, cand) || dup_find(&set, cand) >= 0) continue;
      if (src->with_heading) sub_h = halton_raw(i, primes[d]) * 2.0 * M_PI;
      found = 1;
      break;
    }
    if (!found) {
      free(set.slots);
      free(cand);
      return fail(GMT_E_GOAL_BLOCKED, "no free sample could be placed in the goal region");
    }
  }
  memcpy(coords + (int64_t)(n - 1) * d, cand, sizeof(double) * d);
  if (heading) heading[n - 1] = sub_h;
  goal_idx[0] = n - 1;
  *goal_count = 1;
  free(set.slots);
  free(cand);
  return GMT_OK;
}

/* ---- append_init (sampling.cpp:144-154) --------------------------------- */
int oracle_append_init(int32_t dim, double* coords, double* heading, int32_t* n,
                       const double* init, int32_t init_has_heading, double init_heading,
                       const double* goal_lo, const double* goal_hi, int32_t* goal_idx,
                       int32_t* goal_count, int32_t* index_out) {
  /* With no heading array every sample's heading is nullopt. */
  for (int32_t i = 0; i < *n; ++i) {
    if (!coords_equal(coords + (int64_t)i * dim, init, dim)) continue;
    int same_heading = heading ? (init_has_heading && heading[i] == init_heading)
                               : !init_has_heading;
    if (same_heading) {
      *index_out = i;
      return GMT_OK;
    }
  }
  memcpy(coords + (int64_t)(*n) * dim, init, sizeof(double) * dim);
  if (heading) heading[*n] = init_heading;
  int32_t idx = (*n)++;
  int in_goal = 1;
  for (int k = 0; k < dim; ++k)
    if (init[k] < goal_lo[k] || init[k] > goal_hi[k]) in_goal = 0;
  if (in_goal) goal_idx[(*goal_count)++] = idx;
  *index_out = idx;
  return GMT_OK;
}

/* ---- graph.cpp:14-32 ---------------------------------------------------- */
int oracle_unit_ball_volume(int32_t d, double* out) {
  if (d < 1) return fail(GMT_E_INVALID_INPUT, "dimension must be >= 1");
  *out = pow(M_PI, 0.5 * d) / tgamma(0.5 * d + 1.0);
  return GMT_OK;
}

int oracle_connection_radius(int32_t dim, int64_t n_, double eta, double mu, double* out) {
  if (dim < 1) return fail(GMT_E_INVALID_INPUT, "dimension must be >= 1");
  if (n_ < 2) return fail(GMT_E_INVALID_INPUT, "connection radius needs n >= 2");
  if (!(eta >= 0.0)) return fail(GMT_E_INVALID_INPUT, "eta must be >= 0");
  if (!(mu > 0.0 && mu <= 1.0)) return fail(GMT_E_INVALID_INPUT, "mu_free must be in (0, 1]");
  double zeta;
  oracle_unit_ball_volume(dim, &zeta);
  double d = (double)dim, n = (double)n_;
  double inv_d = 1.0 / d;
  *out = 4.0 * pow(1.0 + eta, inv_d) * pow(inv_d, inv_d) * pow(mu / zeta, inv_d) *
         pow(log(n) / n, inv_d);
  return GMT_OK;
}

/* euclidean_distance, space.cpp:126-133: sequential sum of squares, sqrt. */
static double euclid(const double* a, const double* b, int d) {
  double sq = 0.0;
  for (int k = 0; k < d; ++k) {
    double t = a[k] - b[k];
    sq += t * t;
  }
  return sqrt(sq);
}

/* build_neighbor_graph, Euclidean (graph.cpp:117-188).  The reference's grid
 * prefilter is provably a no-op on the result (graph.hpp:57-59; its own test
 * test_graph.cpp:102-124 compares it with this brute-force double loop,
 * oracles.cpp:50-63), so the restatement is the brute force: out[u] = every
 * v != u with euclidean_distance(u, v) <= r, ascending v.                    */
int oracle_build_neighbor_graph(const double* coords, int32_t n, int32_t dim, double radius,
                                int32_t workers, int64_t* num_edges, int64_t* out_ptr,
                                int32_t* out_col, double* out_cost) {
  (void)workers;
  if (!(radius > 0.0)) return fail(GMT_E_INVALID_INPUT, "connection radius must be positive");
  if (n < 1) return fail(GMT_E_INVALID_INPUT, "cannot build a graph over zero samples");
  int64_t e = 0;
  for (int32_t u = 0; u < n; ++u) {
    if (out_ptr) out_ptr[u] = e;
    for (int32_t v = 0; v < n; ++v) {
      if (v == u) continue;
      double c = euclid(coords + (int64_t)u * dim, coords + (int64_t)v * dim, dim);
      if (c > radius) continue;
      if (out_col) {
        out_col[e] = v;
        out_cost[e] = c;
      }
      ++e;
    }
  }
  if (out_ptr) out_ptr[n] = e;
  *num_edges = e;
  return GMT_OK;
}

/* ---- planner.cpp -------------------------------------------------------- */
enum { UNEXPLORED = 0, OPEN = 1, CLOSED = 2 };

typedef struct {
  const int64_t *ptr;
  const int32_t *col, *path;
  const double* cost;
} rows;

static rows in_rows(const gmt_graph_view* g) {
  rows r;
  if (g->directed) {
    r.ptr = g->in_ptr, r.col = g->in_col, r.cost = g->in_cost, r.path = g->in_path;
  } else {
    r.ptr = g->out_ptr, r.col = g->out_col, r.cost = g->out_cost, r.path = g->out_path;
  }
  return r;
}

/* motion_free (planner.cpp:54-60): the in-edge's path id is the one
 * edge_path(from, to) returns (gmt_graph_view contract). */
static int motion_free(const gmt_scene* s, const double* coords, const gmt_graph_view* g,
                       int from, int to, int32_t path_id) {
  if (path_id >= 0) {
    int64_t a = g->path_ptr[path_id], b = g->path_ptr[path_id + 1];
    return polyline_free_raw(s, g->path_pts + a * s->dim, b - a);
  }
  return segment_free_raw(s, coords + (int64_t)from * s->dim, coords + (int64_t)to * s->dim);
}

typedef struct {
  int parent;
  double cost;
  int checked;
} cand_result;

/* connect_candidate (planner.cpp:62-90) */
static cand_result connect_candidate(int x, const uint8_t* label, const double* cost,
                                     const rows* in, const gmt_scene* s, const double* coords,
                                     const gmt_graph_view* g) {
  cand_result res = {-1, INFINITY, 0};
  int best = -1;
  int32_t best_path = -1;
  double best_cost = INFINITY;
  for (int64_t e = in->ptr[x]; e < in->ptr[x + 1]; ++e) {
    int y = in->col[e];
    if (label[y] != OPEN) continue;
    double c = cost[y] + in->cost[e];
    if (c < best_cost) {
      best_cost = c;
      best = y;
      best_path = in->path ? in->path[e] : -1;
    }
  }
  if (best < 0) return res;
  res.checked = 1;
  if (motion_free(s, coords, g, best, x, best_path)) {
    res.parent = best;
    res.cost = best_cost;
  }
  return res;
}

static void write_tree(gmt_plan_out* out, int n, const uint8_t* label, const double* cost,
                       const int32_t* parent, const int64_t* iter_added) {
  out->tree_size = n;
  for (int v = 0; v < n; ++v) {
    if (out->label) out->label[v] = label[v];
    if (out->tree_cost) out->tree_cost[v] = cost[v];
    if (out->parent) out->parent[v] = parent[v];
    if (out->iteration_added) out->iteration_added[v] = iter_added[v];
  }
}

static void push_stat(gmt_plan_out* out, int group, int added, int64_t checks) {
  int k = out->num_stats++;
  if (k < out->stats_cap) {
    if (out->group_sizes) out->group_sizes[k] = group;
    if (out->nodes_added) out->nodes_added[k] = added;
    if (out->collision_checks) out->collision_checks[k] = checks;
  }
}

static void reset_out(gmt_plan_out* out) {
  out->status = GMT_PLAN_INFEASIBLE_INPUT;
  out->goal_node = -1;
  out->cost = INFINITY;
  out->iterations = 0;
  out->total_collision_checks = 0;
  out->path_len = 0;
  out->num_stats = 0;
  out->tree_size = 0;
}

/* finalize_success (planner.cpp:43-50) */
static void finalize(gmt_plan_out* out, const double* cost, const int32_t* parent, int goal) {
  out->status = GMT_PLAN_SUCCESS;
  out->goal_node = goal;
  out->cost = cost[goal];
  int len = 0;
  for (int v = goal; v >= 0; v = parent[v]) ++len;
  out->path_len = len;
  if (out->path) {
    int k = len;
    for (int v = goal; v >= 0; v = parent[v]) out->path[--k] = v;
  }
}

static int validate_plan(const gmt_graph_view* g, int32_t n, int32_t init_index) {
  /* validate_plan_inputs, planner.cpp:17-23 */
  if (g->n != n) return fail(GMT_E_INVALID_INPUT, "graph was built over a different sample count");
  if (init_index < 0 || init_index >= n) return fail(GMT_E_INVALID_INPUT, "init_index out of range");
  return GMT_OK;
}

/* gmt_plan (planner.cpp:94-198), workers ignored: the map is order-free. */
int oracle_gmt_plan(const gmt_scene* s, const double* coords, int32_t n, int32_t goal_count,
                    const gmt_graph_view* g, int32_t init_index, double lambda, double radius,
                    int32_t workers, gmt_plan_out* out) {
  (void)workers;
  int rc = validate_plan(g, n, init_index);
  if (rc) return rc;
  if (!(lambda > 0.0 && lambda <= 1.0)) return fail(GMT_E_INVALID_INPUT, "lambda must be in (0, 1]");
  if (radius != g->radius)
    return fail(GMT_E_INVALID_INPUT, "params.radius differs from the graph's connection radius");
  const double delta = lambda * radius; /* GmtParams::delta, planner.hpp:32 */
  reset_out(out);
  /* infeasible_input (planner.cpp:39-41): empty tree */
  if (!point_free_raw(s, coords + (int64_t)init_index * s->dim) || goal_count == 0) return GMT_OK;

  uint8_t* label = (uint8_t*)calloc(n, 1);
  double* cost = (double*)malloc(sizeof(double) * n);
  int32_t* parent = (int32_t*)malloc(sizeof(int32_t) * n);
  int64_t* iter_added = (int64_t*)malloc(sizeof(int64_t) * n);
  int32_t* group = (int32_t*)malloc(sizeof(int32_t) * n);
  int32_t* cands = (int32_t*)malloc(sizeof(int32_t) * n);
  uint8_t* mark = (uint8_t*)calloc(n, 1);
  cand_result* results = (cand_result*)malloc(sizeof(cand_result) * n);
  for (int v = 0; v < n; ++v) cost[v] = INFINITY, parent[v] = -1, iter_added[v] = -1;
  label[init_index] = OPEN; /* make_wavefront, planner.cpp:25-35 */
  cost[init_index] = 0.0;
  iter_added[init_index] = 0;
  rows in = in_rows(g);
  long long i = 0;

  for (;;) {
    double min_open = INFINITY; /* planner.cpp:119-122 */
    for (int v = 0; v < n; ++v)
      if (label[v] == OPEN) min_open = min_open < cost[v] ? min_open : cost[v];
    if (min_open == INFINITY) { /* planner.cpp:123-127 */
      out->status = GMT_PLAN_FAILURE_OPEN_EMPTY;
      out->iterations = i;
      break;
    }
    if (min_open > i * delta) { /* fast-forward, planner.cpp:132-136 */
      long long jump = (long long)ceil(min_open / delta);
      i = jump > i + 1 ? jump : i + 1;
      while (min_open > i * delta) ++i;
    }
    int gsize = 0; /* planner.cpp:137-141 */
    for (int v = 0; v < n; ++v)
      if (label[v] == OPEN && cost[v] <= i * delta) group[gsize++] = v;

    int goal_node = -1; /* planner.cpp:145-149 */
    for (int k = 0; k < gsize; ++k) {
      int v = group[k];
      if (!goal_contains(s, coords + (int64_t)v * s->dim)) continue;
      if (goal_node < 0 || cost[v] < cost[goal_node]) goal_node = v;
    }
    if (goal_node >= 0) { /* planner.cpp:150-156 */
      push_stat(out, gsize, 0, 0);
      out->iterations = i;
      finalize(out, cost, parent, goal_node);
      break;
    }

    int ncand = 0; /* candidates, planner.cpp:159-166 (sorted unique) */
    for (int k = 0; k < gsize; ++k) {
      int gnode = group[k];
      for (int64_t e = g->out_ptr[gnode]; e < g->out_ptr[gnode + 1]; ++e) {
        int x = g->out_col[e];
        if (label[x] == UNEXPLORED && !mark[x]) {
          mark[x] = 1;
          ++ncand;
        }
      }
    }
    ncand = 0;
    for (int x = 0; x < n; ++x)
      if (mark[x]) cands[ncand++] = x, mark[x] = 0;

    for (int k = 0; k < ncand; ++k) /* parallel map, planner.cpp:171-176 */
      results[k] = connect_candidate(cands[k], label, cost, &in, s, coords, g);

    int added = 0; /* serial commit, planner.cpp:178-189 */
    long long checks = 0;
    for (int k = 0; k < ncand; ++k) {
      checks += results[k].checked;
      if (results[k].parent < 0) continue;
      int x = cands[k];
      label[x] = OPEN;
      cost[x] = results[k].cost;
      parent[x] = results[k].parent;
      iter_added[x] = i;
      ++added;
    }
    for (int k = 0; k < gsize; ++k) label[group[k]] = CLOSED; /* planner.cpp:190 */
    push_stat(out, gsize, added, checks);                   /* planner.cpp:192-194 */
    out->total_collision_checks += checks;
    ++i;
  }
  write_tree(out, n, label, cost, parent, iter_added);
  free(label), free(cost), free(parent), free(iter_added), free(group), free(cands), free(mark),
      free(results);
  return GMT_OK;
}

/* fmt_plan (planner.cpp:200-262) */
int oracle_fmt_plan(const gmt_scene* s, const double* coords, int32_t n, int32_t goal_count,
                    const gmt_graph_view* g, int32_t init_index, gmt_plan_out* out) {
  int rc = validate_plan(g, n, init_index);
  if (rc) return rc;
  reset_out(out);
  if (!point_free_raw(s, coords + (int64_t)init_index * s->dim) || goal_count == 0) return GMT_OK;
  uint8_t* label = (uint8_t*)calloc(n, 1);
  double* cost = (double*)malloc(sizeof(double) * n);
  int32_t* parent = (int32_t*)malloc(sizeof(int32_t) * n);
  int64_t* iter_added = (int64_t*)malloc(sizeof(int64_t) * n);
  cand_result* results = NULL;
  int64_t rcap = 0;
  for (int v = 0; v < n; ++v) cost[v] = INFINITY, parent[v] = -1, iter_added[v] = -1;
  label[init_index] = OPEN;
  cost[init_index] = 0.0;
  iter_added[init_index] = 0;
  rows in = in_rows(g);
  long long iter = 0;
  for (;;) {
    int z = -1;
    for (int v = 0; v < n; ++v)
      if (label[v] == OPEN && (z < 0 || cost[v] < cost[z])) z = v;
    if (z < 0) {
      out->status = GMT_PLAN_FAILURE_OPEN_EMPTY;
      out->iterations = iter;
      break;
    }
    if (goal_contains(s, coords + (int64_t)z * s->dim)) {
      push_stat(out, 1, 0, 0);
      out->iterations = iter;
      finalize(out, cost, parent, z);
      break;
    }
    int64_t a = g->out_ptr[z], b = g->out_ptr[z + 1];
    if (b - a > rcap) {
      rcap = b - a;
      results = (cand_result*)realloc(results, sizeof(cand_result) * rcap);
    }
    for (int64_t e = a; e < b; ++e) {
      cand_result none = {-1, INFINITY, 0};
      results[e - a] = none;
      if (label[g->out_col[e]] != UNEXPLORED) continue;
      results[e - a] = connect_candidate(g->out_col[e], label, cost, &in, s, coords, g);
    }
    int added = 0;
    long long checks = 0;
    for (int64_t e = a; e < b; ++e) {
      checks += results[e - a].checked;
      if (results[e - a].parent < 0) continue;
      int x = g->out_col[e];
      label[x] = OPEN;
      cost[x] = results[e - a].cost;
      parent[x] = results[e - a].parent;
      iter_added[x] = iter;
      ++added;
    }
    label[z] = CLOSED;
    push_stat(out, 1, added, checks);
    out->total_collision_checks += checks;
    ++iter;
  }
  write_tree(out, n, label, cost, parent, iter_added);
  free(label), free(cost), free(parent), free(iter_added), free(results);
  return GMT_OK;
}

/* ---- 6D double integrator (NEW model; no reference exists) ----
 * Independent C statement of the model the B200 library defines in
 * paper_1705_02403_b200/csrc/di.cuh: parity of this model
 * against the reference is UNPINNED; it is pinned by properties
 * (tests/test_di.py: Gramian-form cost, stationarity, brute-force duration
 * scan) and the planner on top of it is pinned against the reference's
 * gmt_plan on the injected directed graph with cached paths. */
static double di_vel(double s, double vmax) { return vmax * (2.0 * s - 1.0); }

typedef struct {
  double a, b, c0;
} di_coef_t;

static di_coef_t di_coef(const double* x0, const double* x1, double vmax, double w) {
  double sa = 0.0, sb = 0.0, sc = 0.0;
  for (int k = 0; k < 3; ++k) {
    double D = x1[k] - x0[k];
    double v0 = di_vel(x0[3 + k], vmax), v1 = di_vel(x1[3 + k], vmax);
    sa = sa + ((v0 * v0 + v0 * v1) + v1 * v1);
    sb = sb + D * (v0 + v1);
    sc = sc + D * D;
  }
  di_coef_t c;
  c.a = (4.0 * w) * sa;
  c.b = (-12.0 * w) * sb;
  c.c0 = (12.0 * w) * sc;
  return c;
}

static double di_g(di_coef_t c, double t) { return (((t * t - c.a) * t) - 2.0 * c.b) * t - 3.0 * c.c0; }
static double di_c(di_coef_t c, double t) { return t + ((c.c0 / t + c.b) / t + c.a) / t; }

double oracle_di_cost(const double* x0, const double* x1, double vmax, double w, double* tau) {
  di_coef_t c = di_coef(x0, x1, vmax, w);
  if (c.a == 0.0 && c.b == 0.0 && c.c0 == 0.0) {
    *tau = 0.0;
    return 0.0;
  }
  double T = c.a, b2 = 2.0 * (c.b < 0.0 ? -c.b : c.b), c3 = 3.0 * c.c0;
  if (b2 > T) T = b2;
  if (c3 > T) T = c3;
  T = 1.0 + T;
  double best_c = 0.0, best_t = 0.0;
  int have = 0;
  double t_hi = T, g_hi = di_g(c, t_hi);
  for (int j = 1; j <= 96; ++j) {
    double t_lo = t_hi * 0.75, g_lo = di_g(c, t_lo);
    if (g_lo <= 0.0 && g_hi > 0.0) {
      double lo = t_lo, hi = t_hi;
      for (int it = 0; it < 64; ++it) {
        double mid = 0.5 * (lo + hi);
        if (di_g(c, mid) > 0.0) hi = mid; else lo = mid;
      }
      double ct = di_c(c, hi);
      if (!have || ct <= best_c) {
        best_c = ct;
        best_t = hi;
        have = 1;
      }
    }
    t_hi = t_lo;
    g_hi = g_lo;
  }
  if (!have) {
    best_t = t_hi;
    best_c = di_c(c, best_t);
  }
  *tau = best_t;
  return best_c;
}

double oracle_di_coord(const double* x0, const double* x1, double tau, int k, int i, int M,
                       double vmax) {
  if (k <= 0 || tau == 0.0) return x0[i];
  if (k >= M) return x1[i];
  double t = (tau * (double)k) / (double)M;
  int a = i < 3 ? i : i - 3;
  double D = x1[a] - x0[a];
  double v0 = di_vel(x0[3 + a], vmax), v1 = di_vel(x1[3 + a], vmax);
  double tt = tau * tau;
  double c2 = (3.0 * D) / tt - (2.0 * v0 + v1) / tau;
  double c3 = (v0 + v1) / tt - (2.0 * D) / (tt * tau);
  if (i < 3) return x0[a] + t * (v0 + t * (c2 + t * c3));
  double v = v0 + t * (2.0 * c2 + t * (3.0 * c3));
  return 0.5 * (v / vmax + 1.0);
}

/* Brute-force directed r-disk graph of the double integrator (out-rows:
 * targets v != u with cost(u -> v) <= r, ascending) + per-edge durations. */
int oracle_build_di_graph(const double* coords, int32_t n, double vmax, double w, double radius,
                          int64_t* num_edges, int64_t* out_ptr, int32_t* out_col, double* out_cost,
                          double* out_tau) {
  int64_t e = 0;
  for (int32_t u = 0; u < n; ++u) {
    if (out_ptr) out_ptr[u] = e;
    for (int32_t v = 0; v < n; ++v) {
      if (v == u) continue;
      double t;
      double c = oracle_di_cost(coords + (int64_t)u * 6, coords + (int64_t)v * 6, vmax, w, &t);
      if (!(c <= radius)) continue;
      if (out_col) {
        out_col[e] = v;
        out_cost[e] = c;
        out_tau[e] = t;
      }
      ++e;
    }
  }
  if (out_ptr) out_ptr[n] = e;
  *num_edges = e;
  return GMT_OK;
}

/* Waypoints of every out-edge (pts[e][k][i], k = 0..M). */
void oracle_di_paths(const double* coords, int32_t n, const int64_t* ptr, const int32_t* col,
                     const double* tau, int M, double vmax, double* pts) {
  for (int32_t u = 0; u < n; ++u)
    for (int64_t e = ptr[u]; e < ptr[u + 1]; ++e)
      for (int k = 0; k <= M; ++k)
        for (int i = 0; i < 6; ++i)
          pts[(e * (M + 1) + k) * 6 + i] =
              oracle_di_coord(coords + (int64_t)u * 6, coords + (int64_t)col[e] * 6, tau[e], k, i, M, vmax);
}

/* ---- 12D linearised quadrotor (NEW model; no reference exists) -----------
 * Independent C statement of paper_1705_02403_b200/csrc/quad.cuh (DESIGN.md
 * §3.3), same operation order, -ffp-contract=off: parity against the
 * reference is UNPINNED; pinned by properties in tests/test_quad.py
 * (Gramian-form cost with numpy matrices, stationarity, duration scan,
 * trajectory endpoints and dynamics). */
static const double q_h2[2][2] = {{12.0, -6.0}, {-6.0, 4.0}};
static const double q_h4[4][4] = {{100800.0, -50400.0, 10080.0, -840.0},
                                  {-50400.0, 25920.0, -5400.0, 480.0},
                                  {10080.0, -5400.0, 1200.0, -120.0},
                                  {-840.0, 480.0, -120.0, 16.0}};
static const int q_map[4][4] = {{0, 3, 7, 10}, {1, 4, 6, 9}, {2, 5, -1, -1}, {8, 11, -1, -1}};

static double q_hinv(int m, int i, int j) { return m == 2 ? q_h2[i][j] : q_h4[i][j]; }
static double q_fact(int k) {
  double f = 1.0;
  for (int i = 2; i <= k; ++i) f = f * (double)i;
  return f;
}
static double q_pow(double t, int e) {
  double r = 1.0;
  for (int i = 0; i < e; ++i) r = r * t;
  return r;
}
static int q_order(int c) { return c < 2 ? 4 : 2; }
static double q_range(int idx, const gmt_quad_params* P) {
  if (idx == 6 || idx == 7) return P->amax;
  if (idx == 8) return P->ymax;
  if (idx >= 9) return P->wmax;
  return P->vmax;
}
static void q_chain(const double* x, int c, const gmt_quad_params* P, double* z) {
  for (int i = 0; i < q_order(c); ++i) {
    int idx = q_map[c][i];
    double v = idx < 3 ? x[idx] : q_range(idx, P) * (2.0 * x[idx] - 1.0);
    if (c == 0 && i >= 2) v = P->g * v;
    if (c == 1 && i >= 2) v = -(P->g * v);
    z[i] = v;
  }
}
static void q_delta(const double* z0, const double* z1, int m, double delta[4][4]) {
  for (int i = 0; i < m; ++i) {
    delta[i][0] = z1[i] - z0[i];
    for (int p = 1; p < m - i; ++p) delta[i][p] = -(z0[i + p] / q_fact(p));
  }
}
static void q_coef(const double* x0, const double* x1, const gmt_quad_params* P, double* C) {
  for (int k = 0; k <= 7; ++k) C[k] = 0.0;
  for (int c = 0; c < 4; ++c) {
    int m = q_order(c);
    double wc = c < 2 ? P->weight / (P->g * P->g) : P->weight;
    double z0[4], z1[4], delta[4][4];
    q_chain(x0, c, P, z0);
    q_chain(x1, c, P, z1);
    q_delta(z0, z1, m, delta);
    for (int i = 0; i < m; ++i)
      for (int j = 0; j < m; ++j) {
        double h = wc * q_hinv(m, i, j);
        for (int p = 0; p < m - i; ++p)
          for (int q = 0; q < m - j; ++q) {
            int k = 2 * m - i - j - 1 - p - q;
            C[k] = C[k] + (h * delta[i][p]) * delta[j][q];
          }
      }
  }
}
static double q_g(const double* C, double t) {
  double r = 1.0 * t;
  for (int k = 1; k <= 7; ++k) r = r * t - (double)k * C[k];
  return r;
}
static double q_c(const double* C, double t) {
  double r = C[7] / t;
  for (int k = 6; k >= 1; --k) r = (r + C[k]) / t;
  return t + r;
}

double oracle_quad_cost(const double* x0, const double* x1, const gmt_quad_params* P, double* tau) {
  double C[8];
  q_coef(x0, x1, P, C);
  int zero = 1;
  for (int k = 1; k <= 7; ++k) zero = zero && C[k] == 0.0;
  if (zero) {
    *tau = 0.0;
    return 0.0;
  }
  double T = 0.0;
  for (int k = 1; k <= 7; ++k) {
    double a = (double)k * C[k];
    a = a < 0.0 ? -a : a;
    if (a > T) T = a;
  }
  T = 1.0 + T;
  double best_c = 0.0, best_t = 0.0;
  int have = 0;
  double t_hi = T, g_hi = q_g(C, t_hi);
  for (int j = 1; j <= 96; ++j) {
    double t_lo = t_hi * 0.75, g_lo = q_g(C, t_lo);
    if (g_lo <= 0.0 && g_hi > 0.0) {
      double lo = t_lo, hi = t_hi;
      for (int it = 0; it < 64; ++it) {
        double mid = 0.5 * (lo + hi);
        if (q_g(C, mid) > 0.0) hi = mid; else lo = mid;
      }
      double ct = q_c(C, hi);
      if (!have || ct <= best_c) {
        best_c = ct;
        best_t = hi;
        have = 1;
      }
    }
    t_hi = t_lo;
    g_hi = g_lo;
  }
  if (!have) {
    best_t = t_hi;
    best_c = q_c(C, best_t);
  }
  *tau = best_t;
  return best_c;
}

double oracle_quad_coord(const double* x0, const double* x1, double tau, int k, int idx,
                         const gmt_quad_params* P) {
  int M = P->segments;
  if (k <= 0 || tau == 0.0) return x0[idx];
  if (k >= M) return x1[idx];
  int c = 0, i = 0;
  for (int cc = 0; cc < 4; ++cc)
    for (int ii = 0; ii < q_order(cc); ++ii)
      if (q_map[cc][ii] == idx) c = cc, i = ii;
  int m = q_order(c);
  double t = (tau * (double)k) / (double)M;
  double z0[4], z1[4], delta[4][4], d[4], lam[4];
  q_chain(x0, c, P, z0);
  q_chain(x1, c, P, z1);
  q_delta(z0, z1, m, delta);
  for (int j = 0; j < m; ++j) {
    double v = 0.0;
    for (int p = m - j - 1; p >= 0; --p) v = v * tau + delta[j][p];
    d[j] = v;
  }
  for (int j = 0; j < m; ++j) {
    double v = 0.0;
    for (int l = 0; l < m; ++l) v = v + (q_hinv(m, j, l) * d[l]) / q_pow(tau, 2 * m - j - l - 1);
    lam[j] = v;
  }
  double zi = 0.0;
  for (int q = m - 1; q >= i; --q) zi = zi + (z0[q] * q_pow(t, q - i)) / q_fact(q - i);
  int a = m - 1 - i;
  double u = tau - t;
  for (int j = 0; j < m; ++j) {
    int b = m - 1 - j;
    double I = 0.0;
    for (int r = 0; r <= b; ++r) {
      double num = (q_pow(u, b - r) / q_fact(b - r)) * q_pow(t, a + r + 1);
      double den = ((double)(a + r + 1) * q_fact(a)) * q_fact(r);
      I = I + num / den;
    }
    zi = zi + lam[j] * I;
  }
  double v = zi;
  if (c == 0 && i >= 2) v = zi / P->g;
  if (c == 1 && i >= 2) v = -(zi / P->g);
  if (idx < 3) return v;
  return 0.5 * (v / q_range(idx, P) + 1.0);
}

/* Brute-force directed r-disk graph of the quadrotor (as oracle_build_di_graph). */
int oracle_build_quad_graph(const double* coords, int32_t n, const gmt_quad_params* P, double radius,
                            int64_t* num_edges, int64_t* out_ptr, int32_t* out_col, double* out_cost,
                            double* out_tau) {
  int64_t e = 0;
  for (int32_t u = 0; u < n; ++u) {
    if (out_ptr) out_ptr[u] = e;
    for (int32_t v = 0; v < n; ++v) {
      if (v == u) continue;
      double t;
      double c = oracle_quad_cost(coords + (int64_t)u * 12, coords + (int64_t)v * 12, P, &t);
      if (!(c <= radius)) continue;
      if (out_col) {
        out_col[e] = v;
        out_cost[e] = c;
        out_tau[e] = t;
      }
      ++e;
    }
  }
  if (out_ptr) out_ptr[n] = e;
  *num_edges = e;
  return GMT_OK;
}

void oracle_quad_paths(const double* coords, int32_t n, const int64_t* ptr, const int32_t* col,
                       const double* tau, const gmt_quad_params* P, double* pts) {
  int M = P->segments;
  for (int32_t u = 0; u < n; ++u)
    for (int64_t e = ptr[u]; e < ptr[u + 1]; ++e)
      for (int k = 0; k <= M; ++k)
        for (int i = 0; i < 12; ++i)
          pts[(e * (M + 1) + k) * 12 + i] =
              oracle_quad_coord(coords + (int64_t)u * 12, coords + (int64_t)col[e] * 12, tau[e], k, i, P);
}
