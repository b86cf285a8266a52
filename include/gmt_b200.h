/*
 * gmt_b200.h -- C ABI of the B200-native Group Marching Tree (GMT*) planner.
 *
 * This is the drop-in boundary for the reference library `gmtplan`
 * (/root/reference/proj).  The reference exposes no FFI of its own: its
 * boundary is the set of free functions in `namespace gmt` that the CLI,
 * the simulator and the tests call.  Every entry point
 * below names the reference function it replaces (file:line, paths relative
 * to /root/reference/proj).  The header-only C++ shim `gmt_b200.hpp`
 * re-creates those exact `gmt::` signatures on top of this ABI.
 *
 * Conventions
 *   - Plain pointers and sizes only.  Host pointers unless a name says `dev`.
 *   - Every function returns an int error code (gmt_error); 0 is success.
 *     The reference throws exceptions; the ABI maps each exception type to a
 *     code and stores the message in a thread-local string (gmt_last_error).
 *   - Planning outcomes are values (gmt_plan_status), never errors, exactly
 *     like the reference (planner.hpp:14).
 *   - Nothing is retained between calls except explicit handles.
 *   - There is no CPU fallback: every compute call runs CUDA kernels on the
 *     context's device and fails with GMT_E_NO_DEVICE when there is none.
 */
#ifndef GMT_B200_H
#define GMT_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define GMT_B200_ABI_VERSION 2

/* Error codes.  Reference exception types: errors.hpp:9-21. */
typedef enum gmt_error {
  GMT_OK = 0,
  GMT_E_INVALID_INPUT = 1,        /* gmt::InvalidInputError        (errors.hpp:9-11)  */
  GMT_E_INFEASIBLE_SAMPLING = 2,  /* gmt::InfeasibleSamplingError  (errors.hpp:14-16) */
  GMT_E_GOAL_BLOCKED = 3,         /* gmt::GoalBlockedError         (errors.hpp:19-21) */
  GMT_E_CUDA = 4,                 /* CUDA runtime failure (no reference analogue)     */
  GMT_E_NO_DEVICE = 5,            /* no usable sm_100 device: the ABI never falls back */
  GMT_E_INTERNAL = 6,
  GMT_E_IO = 7                    /* graph-cache file I/O (the reference returns false) */
} gmt_error;

/* PlanStatus, same order as planner.hpp:14. */
typedef enum gmt_plan_status {
  GMT_PLAN_SUCCESS = 0,
  GMT_PLAN_FAILURE_OPEN_EMPTY = 1,
  GMT_PLAN_INFEASIBLE_INPUT = 2
} gmt_plan_status;

/* NodeLabel, same values as planner.hpp:16. */
typedef enum gmt_label {
  GMT_LABEL_UNEXPLORED = 0,
  GMT_LABEL_OPEN = 1,
  GMT_LABEL_CLOSED = 2
} gmt_label;

/* SampleSource::Kind (sampling.hpp:21). */
typedef enum gmt_sample_kind { GMT_SAMPLE_HALTON = 0, GMT_SAMPLE_UNIFORM = 1 } gmt_sample_kind;

/* ObstacleSet + GoalRegion (space.hpp:19-41), structure-of-arrays.
 *   box_lo[b*dim + k], box_hi[b*dim + k]   closed boxes, lo <= hi
 *   goal_lo[k], goal_hi[k]                  closed goal box            */
typedef struct gmt_scene {
  int32_t dim;
  int32_t num_boxes;
  const double* box_lo;
  const double* box_hi;
  const double* goal_lo;
  const double* goal_hi;
} gmt_scene;

/* SampleSource (sampling.hpp:20-29). */
typedef struct gmt_sample_source {
  int32_t kind;          /* gmt_sample_kind */
  int32_t with_heading;  /* Dubins headings (halton prime d+1 / extra uniform draw) */
  uint64_t start_index;  /* halton: first 1-based index */
  uint64_t seed;         /* uniform: Pcg32 seed */
} gmt_sample_source;

/* NeighborGraph (graph.hpp:31-54) as compressed rows.
 *   out row u: out_col[out_ptr[u] .. out_ptr[u+1]) targets, sorted ascending
 *   in  row x: in_col[in_ptr[x] .. in_ptr[x+1])   sources (list order is the
 *              reference's in-list order; ties in connect_candidate go to
 *              the earliest entry, planner.cpp:70-82)
 *   *_path: path id of the edge (graph.hpp:35) or -1 for exact straight
 *           edges; the whole array may be NULL (all exact).  in_path[e] must
 *           be the id that NeighborGraph::edge_path(source, x) returns
 *           (graph.cpp:34-40), i.e. the out-list's id.
 *   paths:  path p = path_pts[path_ptr[p]*dim .. path_ptr[p+1]*dim)
 * directed == 0 declares in == out (Euclidean graphs, graph.cpp:184-186);
 * the in_* pointers are then ignored.                                      */
typedef struct gmt_graph_view {
  int32_t n;
  int32_t dim;
  double radius;
  int32_t directed;
  int32_t reserved;
  const int64_t* out_ptr;
  const int32_t* out_col;
  const double* out_cost;
  const int32_t* out_path;
  const int64_t* in_ptr;
  const int32_t* in_col;
  const double* in_cost;
  const int32_t* in_path;
  int64_t num_paths;
  const int64_t* path_ptr;
  const double* path_pts;
} gmt_graph_view;

/* PlanResult (planner.hpp:43-51).  Scalars are always written.  Array
 * outputs are caller-owned and optional (NULL skips them):
 *   path            capacity n        (path_len entries, root..goal)
 *   label/tree_cost/parent/iteration_added   capacity n (tree_size entries;
 *                   tree_size is 0 for infeasible input, planner.cpp:108)
 *   group_sizes/nodes_added/collision_checks capacity stats_cap >= n + 1
 *                   (num_stats entries, IterationStats planner.hpp:36-40)  */
typedef struct gmt_plan_out {
  int32_t status; /* gmt_plan_status */
  int32_t goal_node;
  double cost;
  int64_t iterations;
  int64_t total_collision_checks;
  int32_t path_len;
  int32_t num_stats;
  int32_t tree_size;
  int32_t stats_cap;
  int32_t* path;
  uint8_t* label;
  double* tree_cost;
  int32_t* parent;
  int64_t* iteration_added;
  int32_t* group_sizes;
  int32_t* nodes_added;
  int64_t* collision_checks;
} gmt_plan_out;

/* Per-query summary record gathered after a batched solve. */
typedef struct gmt_plan_summary {
  int32_t status;
  int32_t goal_node;
  double cost;
  int64_t iterations;
  int64_t total_collision_checks;
  int32_t path_len;
  int32_t num_stats;
} gmt_plan_summary;

/* Steering models.  GMT_STEER_EUCLIDEAN is the reference's euclidean model
 * (steering.hpp:10); GMT_STEER_DOUBLE_INTEGRATOR is the NEW 6D double
 * integrator of SURVEY.md §8 row a22 (no reference):
 * state [p(3), s(3)] in [0,1]^6 with velocity v = vmax (2s - 1), cost
 * tau + weight * integral |u|^2, directed edges, `segments`-segment
 * trajectory polylines for the lazy check.                                 */
typedef enum gmt_steering {
  GMT_STEER_EUCLIDEAN = 0,
  GMT_STEER_DUBINS_AIRPLANE = 1,  /* steering.hpp:10, dubins.cpp (see gmt_dubins_params) */
  GMT_STEER_DOUBLE_INTEGRATOR = 2,
  GMT_STEER_QUADROTOR = 3
} gmt_steering;

typedef struct gmt_di_params {
  double vmax;
  double weight;
  int32_t segments;
  int32_t reserved;
} gmt_di_params;

/* GMT_STEER_DUBINS_AIRPLANE (SteeringModel, steering.hpp:9-23): planar
 * Dubins paths of turning radius rho in (x, y), altitude (coordinate 2, if
 * present) linear in arc length; cost sqrt(Lp^2 + dz^2) (or Lp when
 * planar_cost_only); paths discretised every discretization_step (0 means
 * rho / 10).  Samples carry a heading.  Costs match the reference to a few
 * ulps (its sin/cos/atan2/acos come from glibc).          */
typedef struct gmt_dubins_params {
  double rho;
  double discretization_step;
  int32_t planar_cost_only;
  int32_t reserved;
} gmt_dubins_params;

/* GMT_STEER_QUADROTOR: the NEW 12D linearised quadrotor of SURVEY.md §8 row
 * a22.  State [p(3), v(3), roll/pitch/yaw(3), rates(3)] in
 * [0,1]^12: v = vmax (2s - 1), roll/pitch = amax (2s - 1), yaw = ymax (2s - 1),
 * rates = wmax (2s - 1); hover linearisation with gravity g (workspace
 * units / s^2); cost tau + weight * integral of the squared torques and
 * thrust.                                                                  */
typedef struct gmt_quad_params {
  double g;
  double vmax;
  double amax;
  double ymax;
  double wmax;
  double weight;
  int32_t segments;
  int32_t reserved;
} gmt_quad_params;

/* ProblemFile (problem.hpp:17-29) minus the Dubins steering fields, plus the
 * double-integrator model (radius_override is required for it).          */
typedef struct gmt_problem {
  gmt_scene scene;
  const double* init;     /* dim coords */
  int32_t init_has_heading;
  double init_heading;
  int32_t n;
  double lambda;
  double eta;
  double radius_override; /* <= 0: use connection_radius (problem.cpp:342-351) */
  gmt_sample_source sampling;
  int32_t steering;       /* gmt_steering */
  int32_t reserved;
  gmt_di_params di;
  gmt_quad_params quad;
  gmt_dubins_params dubins;
} gmt_problem;

/* ---- gmt-problem/1 scene files (problem.hpp:14-34) ---------------------- */
/* parse_problem (problem.cpp:102-223) / load_problem (problem.cpp:225-231):
 * the same strict validation -- unknown keys rejected, every error named by
 * its field path (GMT_E_INVALID_INPUT with the reference's message, e.g.
 * "obstacles[3].lo: expected 2 coordinates, got 3"; malformed JSON gives
 * "invalid JSON: ..."), the Dubins-only fields, a free start state -- and
 * the same defaults.  The handle owns the arrays; gmt_problem_file_view
 * fills a flat gmt_problem pointing into it (valid until destroy) and the
 * optional notes string.  radius_override <= 0 means none.               */
typedef struct gmt_problem_file gmt_problem_file;
int gmt_problem_parse(const char* json_text, size_t length, gmt_problem_file** out);
int gmt_problem_load(const char* path, gmt_problem_file** out);
int gmt_problem_file_view(const gmt_problem_file* file, gmt_problem* view, const char** notes);
void gmt_problem_file_destroy(gmt_problem_file* file);

/* Replanning simulator (simulator.hpp:14-80): ScenarioConfig with its
 * PlanningSetup flattened.  scene = the static obstacles at t = 0 and the
 * goal; radius_override <= 0 means connection_radius.                    */
typedef struct gmt_scenario {
  gmt_scene scene;
  const double* init;       /* dim coords */
  int32_t n;                /* fresh samples per replan */
  int32_t trials;           /* per campaign cell */
  double lambda;
  double eta;
  double radius_override;
  double collapse_rate;     /* expected obstacle spawns per second */
  double spawn_box_size;
  double disturbance_sigma;
  double replan_latency;
  double control_dt;
  double robot_speed;
  double time_limit;
  uint64_t seed;            /* campaign master seed */
} gmt_scenario;

/* TrialOutcome::Result, same order as simulator.hpp:41. */
enum { GMT_TRIAL_REACHED_GOAL = 0, GMT_TRIAL_COLLIDED = 1, GMT_TRIAL_TIMED_OUT = 2 };

typedef struct gmt_trial_outcome {
  int32_t result;
  int32_t replans;
  int32_t spawned;
  int32_t noise_outliers;
  double time;
  int64_t path_len;         /* states in path_travelled (init included) */
} gmt_trial_outcome;

typedef struct gmt_ctx gmt_ctx;
typedef struct gmt_instance gmt_instance;
typedef struct gmt_batch gmt_batch;

/* ---- context ---------------------------------------------------------- */
const char* gmt_last_error(void);
int gmt_abi_version(void);
/* sizeof of the ABI structs, in the order gmt_scene, gmt_sample_source,
 * gmt_graph_view, gmt_plan_out, gmt_plan_summary, gmt_problem,
 * gmt_di_params, gmt_batch_host, gmt_quad_params, gmt_scenario,
 * gmt_trial_outcome, gmt_dubins_params (bindings check their layouts).    */
int gmt_struct_sizes(int64_t* out, int32_t count);
int gmt_ctx_create(int device, gmt_ctx** out);
void gmt_ctx_destroy(gmt_ctx* ctx);
void* gmt_ctx_stream(gmt_ctx* ctx); /* cudaStream_t every kernel of ctx runs on */
int gmt_ctx_synchronize(gmt_ctx* ctx);
int64_t gmt_launch_count(const gmt_ctx* ctx); /* kernels launched so far */
/* GMT_OPT_CLUSTER: CTAs cooperating on one single-query solve (1,2,4,8,16; 0 = auto)
 * GMT_OPT_THREADS: threads per CTA for single-query solves (0 = auto)
 * GMT_OPT_BATCH_THREADS: threads per CTA for batched solves (0 = auto)
 * GMT_OPT_BATCH_CLUSTER: CTAs per query in batched solves (default 1)
 * GMT_OPT_COUNTERS: 1 = solves launched from now on add their traffic
 *                   counts to the context counters (gmt_ctx_counters)      */
enum {
  GMT_OPT_CLUSTER = 1,
  GMT_OPT_THREADS = 2,
  GMT_OPT_BATCH_THREADS = 3,
  GMT_OPT_BATCH_CLUSTER = 4,
  GMT_OPT_COUNTERS = 5
};
int gmt_ctx_set_option(gmt_ctx* ctx, int option, int64_t value);
/* Traffic counters summed over counted solves: out[0] in-row edges read
 * (P5), out[1] out-row edges read (P4), out[2] in-edges whose source was
 * open (cost[y] gathers).  Synchronizes; reset != 0 zeroes them.          */
int gmt_ctx_counters(gmt_ctx* ctx, int64_t* out, int32_t reset);

/* ---- offline phase ---------------------------------------------------- */
/* unit_ball_volume, connection_radius (graph.cpp:14-32); host scalars. */
int gmt_unit_ball_volume(int32_t dim, double* out);
int gmt_connection_radius(int32_t dim, int64_t n, double eta, double mu_free, double* out);

/* sample_free (sampling.cpp:81-142): n free samples, goal tags, goal
 * substitution.  coords_out[n*dim], heading_out[n] (may be NULL unless
 * with_heading), goal_idx_out[n]; *goal_count_out entries are written.   */
int gmt_sample_free(gmt_ctx* ctx, int32_t n, const gmt_scene* scene, const gmt_sample_source* src,
                    double* coords_out, double* heading_out, int32_t* goal_idx_out,
                    int32_t* goal_count_out);

/* append_init (sampling.cpp:144-154) over host sample arrays of capacity
 * n+1: appends init at index n unless an exact duplicate (coords and
 * heading) exists.  Updates *n and the goal index list.                  */
int gmt_append_init(gmt_ctx* ctx, int32_t dim, double* coords, double* heading, int32_t* n,
                    const double* init, int32_t init_has_heading, double init_heading,
                    const double* goal_lo, const double* goal_hi, int32_t* goal_idx,
                    int32_t* goal_count, int32_t* index_out);

/* build_neighbor_graph (graph.cpp:117-188), Euclidean model: r-disk CSR
 * built on the device.  The out rows are the in rows (symmetric).
 * Two-call pattern: pass NULL arrays to get *num_edges, then call again
 * with out_ptr[n+1], out_col[E], out_cost[E].                            */
int gmt_build_neighbor_graph(gmt_ctx* ctx, const double* coords, int32_t n, int32_t dim,
                             double radius, int64_t* num_edges, int64_t* out_ptr,
                             int32_t* out_col, double* out_cost);

/* Double-integrator steering (NEW, row a22): cost and duration of `count`
 * state pairs x0s[i*6..], x1s[i*6..], evaluated on the device.           */
int gmt_di_costs(gmt_ctx* ctx, const double* x0s, const double* x1s, int64_t count,
                 const gmt_di_params* params, double* cost_out, double* tau_out);

/* Directed double-integrator r-disk graph over 6D samples, built on the
 * device in NeighborGraph conventions (graph.cpp:117-188): out-rows sorted
 * by target, in-rows by source, path ids = out-edge indices
 * (graph.cpp:172-183).  Two-call pattern (NULL out_ptr: count only).
 * out_tau / in_path / path_pts (E*(segments+1)*6 waypoints, the degenerate
 * zero-duration edge repeating its state) may be NULL.                   */
int gmt_build_di_graph(gmt_ctx* ctx, const double* coords, int32_t n, const gmt_di_params* params,
                       double radius, int64_t* num_edges, int64_t* out_ptr, int32_t* out_col,
                       double* out_cost, double* out_tau, int64_t* in_ptr, int32_t* in_col,
                       double* in_cost, int32_t* in_path, double* path_pts);

/* 12D quadrotor steering (NEW, row a22): the same pair of entry points for
 * the quadrotor model (states of 12 coordinates; path_pts E*(segments+1)*12). */
int gmt_quad_costs(gmt_ctx* ctx, const double* x0s, const double* x1s, int64_t count,
                   const gmt_quad_params* params, double* cost_out, double* tau_out);
int gmt_build_quad_graph(gmt_ctx* ctx, const double* coords, int32_t n,
                         const gmt_quad_params* params, double radius, int64_t* num_edges,
                         int64_t* out_ptr, int32_t* out_col, double* out_cost, double* out_tau,
                         int64_t* in_ptr, int32_t* in_col, double* in_cost, int32_t* in_path,
                         double* path_pts);

/* build_instance + gmt_plan for a batch of Euclidean problems (one common
 * dimension), or of double-integrator problems (derived from the shared
 * sample pool, see gmt_batch_create_problems): samples, init append and
 * graphs of all problems are built in batched device launches, then ONE
 * batched solve.  Problems that
 * need sample_free's rare paths (more candidates than the first chunk,
 * exact duplicates, goal substitution) use the single-instance builder, so
 * every result equals gmt_instance_build + gmt_plan bit for bit.
 * status_out[q]: GMT_OK, or the query's own build outcome
 * (GMT_E_GOAL_BLOCKED / GMT_E_INFEASIBLE_SAMPLING; summaries[q] is then
 * not written).  path_states (may be NULL): up to path_cap path states
 * (dim doubles each) of query q at q * path_cap * dim.  lambda per problem. */
int gmt_plan_problems(gmt_ctx* ctx, const gmt_problem* problems, int32_t count, int32_t* status_out,
                      gmt_plan_summary* summaries, int32_t path_cap, double* path_states);

/* ---- replanning simulator (simulator.hpp:53-74) -------------------------- */
/* run_trial (simulator.cpp:66-176): the trial state machine on the host,
 * bit-identical to the reference, every replan (sample_free -> append_init
 * -> graph -> gmt_plan) on the device.  path (may be NULL) receives up to
 * path_cap states of path_travelled (dim doubles each).                  */
int gmt_run_trial(gmt_ctx* ctx, const gmt_scenario* cfg, uint64_t trial_seed, gmt_trial_outcome* out,
                  double* path, int64_t path_cap);
/* run_campaign (simulator.cpp:178-227): the (latency x rate x sigma) grid,
 * cfg->trials trials per cell, seeds from the cell parameters; `workers`
 * host threads, each with its own context / stream on `device`.
 * successes[num_latencies * num_rates * num_sigmas], cell order as the
 * reference (latency outermost).                                         */
int gmt_run_campaign(int device, const gmt_scenario* cfg, const double* latencies,
                     int32_t num_latencies, const double* rates, int32_t num_rates,
                     const double* sigmas, int32_t num_sigmas, int32_t workers, int32_t* successes);

/* Dubins-airplane steering on the device (connect_cost, steering.cpp:104-112;
 * connect's segment count, steering.cpp:83): states are (x, y[, z],
 * heading), dim = position coordinates (2 or 3).  segments_out[i] = 0 for
 * the degenerate pair (path = {a}).                                      */
int gmt_dubins_costs(gmt_ctx* ctx, const double* x0s, const double* x1s, int64_t count, int32_t dim,
                     const gmt_dubins_params* params, double* cost_out, int32_t* segments_out);

/* ---- GMTG v1 graph cache (graph.hpp:56-65, graph.cpp:190-343) --------- */
/* problem_key (problem.cpp:281-303) of a Euclidean problem: the cache key
 * the reference's build_instance uses.                                   */
int gmt_problem_key(const gmt_problem* problem, uint64_t* key_out);
/* save_graph_cache (graph.cpp:240-276) of a host CSR (out-rows sorted by
 * target): little-endian GMTG v1, written to file.tmp and renamed.       */
int gmt_graph_cache_save(const char* file, uint64_t key, int32_t n, double radius,
                         const int64_t* row_ptr, const int32_t* col, const double* cost);
/* load_graph_cache (graph.cpp:278-343), Euclidean: *hit = 0 on a missing
 * file, any header mismatch (key, n, radius, model) or corruption.  Two-call
 * pattern: NULL row_ptr returns *hit and *num_edges only; the second call
 * passes row_ptr[n+1] and col/cost of edge_capacity entries and fails with
 * GMT_E_INVALID_INPUT (*num_edges = the file's count) when the file now
 * holds more edges than that.                                            */
int gmt_graph_cache_load(const char* file, uint64_t key, int32_t n, double radius, int32_t* hit,
                         int64_t* num_edges, int64_t edge_capacity, int64_t* row_ptr, int32_t* col,
                         double* cost);

/* ---- exact geometry ---------------------------------------------------- */
/* segment_free (space.hpp, space.cpp:80-90) of `count` independent segments
 * a[i*dim ..] -> b[i*dim ..] against one obstacle set (closed boxes,
 * box_lo/box_hi[b*dim + k]), evaluated on the device by the same warp test
 * every lazy check runs: the closed slab clip (space.cpp:60-78), the
 * endpoint cube test and the degenerate-point rule (point_free,
 * space.cpp:47-54).  free_out[i] = 1 when the segment is free.          */
int gmt_segment_free(gmt_ctx* ctx, int32_t dim, int32_t num_boxes, const double* box_lo,
                     const double* box_hi, const double* a, const double* b, int64_t count,
                     uint8_t* free_out);

/* ---- device-resident instances (ProblemInstance, problem.hpp:52-57) --- */
/* Upload host samples + graph + scene.  goal_count is samples.goal_indices
 * .size() (only its emptiness matters, planner.cpp:39-41).               */
int gmt_instance_upload(gmt_ctx* ctx, const gmt_scene* scene, const double* coords, int32_t n,
                        int32_t goal_count, const gmt_graph_view* graph, gmt_instance** out);
/* build_instance (problem.cpp:336-363) entirely on the device. */
int gmt_instance_build(gmt_ctx* ctx, const gmt_problem* problem, gmt_instance** out);
/* build_instance(problem, workers, cache_file) (problem.cpp:336-363),
 * Euclidean: on a cache hit the graph comes from the file (uploaded), else
 * it is built on the device and saved (a failed save is ignored, like the
 * reference's).  *cache_hit (may be NULL) reports which.                   */
int gmt_instance_build_cached(gmt_ctx* ctx, const gmt_problem* problem, const char* cache_file,
                              gmt_instance** out, int32_t* cache_hit);
/* save_graph_cache of a device instance's graph (Euclidean). */
int gmt_instance_cache_save(gmt_ctx* ctx, const gmt_instance* inst, const char* file, uint64_t key);
int gmt_instance_info(const gmt_instance* inst, int32_t* n, int32_t* dim, int32_t* init_index,
                      double* radius, int64_t* num_edges, int32_t* goal_count);
/* Copy samples / goal indices / graph of an instance back to the host
 * (any pointer may be NULL).                                             */
int gmt_instance_download(gmt_ctx* ctx, const gmt_instance* inst, double* coords,
                          int32_t* goal_idx, int64_t* out_ptr, int32_t* out_col,
                          double* out_cost);
void gmt_instance_destroy(gmt_instance* inst);

/* ---- online phase ------------------------------------------------------ */
/* gmt_plan (planner.cpp:94-198) on a device-resident instance. */
int gmt_plan(gmt_ctx* ctx, const gmt_instance* inst, int32_t init_index, double lambda,
             double radius, gmt_plan_out* out);

/* gmt_plan with every input in host memory (the drop-in call the C++ shim
 * makes): upload, solve, download inside one call.                        */
int gmt_plan_host(gmt_ctx* ctx, const gmt_scene* scene, const double* coords, int32_t n,
                  int32_t goal_count, const gmt_graph_view* graph, int32_t init_index,
                  double lambda, double radius, gmt_plan_out* out);

/* fmt_plan (planner.cpp:200-262): the lambda -> 0 baseline, one node per
 * iteration, on the device.                                              */
int gmt_fmt_plan(gmt_ctx* ctx, const gmt_instance* inst, int32_t init_index, gmt_plan_out* out);
/* dijkstra_oracle (planner.hpp:76-79, planner.cpp:264-334): every out-edge
 * checked eagerly on the device (Euclidean pairs share one check), then
 * exact Dijkstra from init over the surviving edges; iterations = pops.   */
int gmt_dijkstra_oracle(gmt_ctx* ctx, const gmt_instance* inst, int32_t init_index, gmt_plan_out* out);

/* Batched independent queries: one CTA (or cluster) per query, one launch.
 * init_index may be NULL (use each instance's built init index).
 * Lifetime: the batch reads the instances' device memory on every launch;
 * every instance must outlive the batch (destroy the batch first).       */
int gmt_batch_create(gmt_ctx* ctx, int32_t count, gmt_instance* const* insts,
                     const int32_t* init_index, double lambda, gmt_batch** out);
/* Batched independent PROBLEMS (scenes, not prebuilt instances): every
 * problem's instance (build_instance, problem.cpp:336-363) is derived on the
 * device, then solved by gmt_batch_launch.  Double-integrator problems with
 * Halton sampling that share the start index, radius_override and model
 * parameters take the shared sample pool of SURVEY.md §8(e): the context
 * keeps the first K Halton points and their directed graph (built once,
 * reused by later calls), and each query's graph is derived from it -- the
 * induced subgraph on its first n free points, re-indexed by rank, plus the
 * rows of its goal-substituted sample (sampling.cpp:115-141) and appended
 * init (sampling.cpp:144-154) -- bit-identical to gmt_instance_build.  Every
 * other problem (and the rare paths: pool too short, an init that duplicates
 * a sample) is built by gmt_instance_build.  status_out[q]: GMT_OK or the
 * query's own build error (GMT_E_GOAL_BLOCKED / GMT_E_INFEASIBLE_SAMPLING);
 * failed queries are left out of the batch (its query index k counts the
 * successful problems in order).  The batch owns the derived instances.   */
int gmt_batch_create_problems(gmt_ctx* ctx, const gmt_problem* problems, int32_t count,
                              int32_t* status_out, gmt_batch** out);
/* The context's shared sample pool: points K its graph covers, pool graph
 * edges, the wall time its last (re)build took, how many queries of the last
 * call took the single builder, and (GMT_POOL_TIMING=1) the last call's
 * device stage times in ms (stage_ms[8]: upload, free flags, select, subst +
 * init, special rows, layout, rows, descriptors).  Any pointer may be NULL. */
int gmt_ctx_pool_info(gmt_ctx* ctx, int32_t* pool_size, int64_t* num_edges, double* build_ms,
                      int32_t* last_fallbacks, double* stage_ms);
/* Graph of batch query q as compressed rows (in-rows with costs and
 * durations, out-row targets).  Two-call pattern: NULL in_ptr returns *n,
 * *num_in and *num_out; then coords[n*dim] (may be NULL), in_ptr[n+1],
 * in_col/in_cost/in_tau[num_in] (cost/tau may be NULL), out_ptr[n+1],
 * out_col[num_out].                                                      */
int gmt_batch_graph(gmt_ctx* ctx, gmt_batch* batch, int32_t query, int32_t* n, int64_t* num_in,
                    int64_t* num_out, double* coords, int64_t* in_ptr, int32_t* in_col, double* in_cost,
                    double* in_tau, int64_t* out_ptr, int32_t* out_col);
int gmt_batch_launch(gmt_ctx* ctx, gmt_batch* batch); /* async on gmt_ctx_stream */
int gmt_batch_summaries(gmt_ctx* ctx, gmt_batch* batch, gmt_plan_summary* out);
int gmt_batch_result(gmt_ctx* ctx, gmt_batch* batch, int32_t query, gmt_plan_out* out);
void gmt_batch_destroy(gmt_batch* batch);

/* Batched drop-in with host inputs (Euclidean graphs): `count` independent
 * queries packed back to back in host arrays (pinned memory recommended).
 * Query q owns nodes [node_off[q], node_off[q+1]), edges [edge_off[q],
 * edge_off[q+1]) and boxes [box_off[q], box_off[q+1]); its row_ptr block
 * holds n_q+1 entries starting at row_ptr[node_off[q] + q], relative to
 * edge_off[q].  One H2D copy per array, one solve launch, D2H of the
 * summaries and (optionally) paths [total_nodes] and full trees.         */
typedef struct gmt_batch_host {
  int32_t count;
  int32_t dim;
  const int64_t* node_off;   /* [count+1] */
  const int64_t* edge_off;   /* [count+1] */
  const int32_t* box_off;    /* [count+1] */
  const double* coords;      /* [total_nodes*dim] */
  const double* box_lo;      /* [total_boxes*dim] */
  const double* box_hi;
  const double* goal_lo;     /* [count*dim] */
  const double* goal_hi;
  const int64_t* row_ptr;    /* [total_nodes+count] */
  const int32_t* col;        /* [total_edges] */
  const double* cost;        /* [total_edges] */
  const int32_t* goal_count; /* [count] */
  const int32_t* init_index; /* [count] */
  const double* radius;      /* [count] graph radius == params.radius */
} gmt_batch_host;

/* paths / label / tree_cost / parent / iteration_added are [total_nodes]
 * arrays indexed like coords (any may be NULL); summaries [count].        */
int gmt_plan_batch_host(gmt_ctx* ctx, const gmt_batch_host* batch, double lambda,
                        gmt_plan_summary* summaries, int32_t* paths, uint8_t* label,
                        double* tree_cost, int32_t* parent, int64_t* iteration_added);

/* Host buffers the library pins for faster H2D/D2H (cudaHostAlloc). */
int gmt_host_alloc(size_t bytes, void** out);
void gmt_host_free(void* p);

#ifdef __cplusplus
}
#endif

#endif /* GMT_B200_H */
