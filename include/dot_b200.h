/*
 * dot_b200.h -- C ABI of the B200-native Dynamic PlenOctree (DOT) hot path.
 *
 * Drop-in boundary for the reference's operator layer `octrf._kernels`
 * (/root/reference/pkg/src/octrf/_kernels.py), which `octrf/render.py`,
 * `octrf/calibrate.py` and `octrf/optim.py` call with flat arrays,
 * caller-allocated outputs and no exceptions.  Every entry point here takes
 * plain device pointers + sizes + a cudaStream_t (as void*), returns a
 * dot_status, never frees caller memory and never synchronises unless the
 * comment says so.  Scratch memory is stream-ordered (cudaMallocAsync).
 *
 * Tree layout (canonical BFS):
 *   node[i] >= 0 : internal node, its 8 children are node[i] .. node[i]+7
 *                  in octant order (x -> bit 0, y -> bit 1, z -> bit 2);
 *   node[i] <  0 : leaf, payload row = ~node[i] (the reference's pool id).
 *   Node centres are not stored: c_child = c_parent +/- h_child in fp64,
 *   which reproduces the reference's stored centres bit-exactly
 *   (octree.py:228-238, 411-414).
 *   sigma[capacity] f32, sh[capacity * sh_stride] f32 channel-major
 *   (sh[k*B + b], octree.py:48-50), rows padded to a multiple of 4 floats.
 */
#ifndef DOT_B200_H
#define DOT_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum dot_status {
    DOT_OK = 0,
    DOT_BAD_ARG = 1,   /* maps to octrf.errors.InputError / ConfigError     */
    DOT_OOM = 2,       /* scratch allocation failed                          */
    DOT_CUDA_ERR = 3,  /* launch / runtime failure, see dot_last_error()    */
    DOT_NO_DEVICE = 4  /* no sm_100 device visible                           */
} dot_status;

typedef struct dot_tree_view {
    const int32_t* node;      /* [n_nodes] canonical node words (device)     */
    int64_t n_nodes;
    const float* sigma;       /* [capacity] (device)                          */
    const float* sh;          /* [capacity * sh_stride] (device)              */
    int64_t capacity;
    int32_t basis_count;      /* 1, 4, 9 or 16                               */
    int32_t sh_stride;        /* floats per row, multiple of 4, >= 3*B       */
    double center[3];         /* root cube centre                            */
    double half_extent;       /* root cube half edge                         */
    int32_t max_depth;
    int32_t locate_level;     /* L of the locate table, 0 = none             */
    const int32_t* locate;    /* [8^L] from dot_locate_build, or NULL        */
} dot_tree_view;

/* Library identity / diagnostics. */
int dot_abi_version(void);
const char* dot_last_error(void);
int dot_device_check(void);

/* --- exp of the reference (glibc's exp, restated bit-exactly; used for
 *     every alpha = exp(-sigma * delta) of the kernels): host loop and a
 *     device kernel over n doubles, for parity tests. */
void dot_exp_ref_host(const double* x, double* y, int64_t n);
int dot_exp_ref_device(const double* x, double* y, int64_t n, void* stream);

/* --- locate table (no reference counterpart; accelerates _descend,
 *     _kernels.py:56-68): for a dyadic root (half_extent a power of two,
 *     centre a multiple of half * 2^-20, max_depth <= 21, capacity < 2^26)
 *     table[x + (y << L) + (z << 2L)] (8^L int32, device) receives the node
 *     word at depth L on the path to grid cell (x, y, z), or
 *     INT32_MIN | depth << 26 | pool_id for a leaf shallower than L.  The
 *     traversal kernels then replace the first L dependent node loads of
 *     every root descent by one table load (exact: same leaf as the fp64
 *     descent).  Set view.locate / view.locate_level to use it; a view whose
 *     root is not dyadic ignores it.  Returns DOT_BAD_ARG for non-dyadic
 *     roots or L outside 1..9. */
int dot_locate_supported(const dot_tree_view* tree);
int dot_locate_build(const dot_tree_view* tree, int32_t level, int32_t* table, void* stream);

/* --- traversal (replaces count_segments_kernel / fill_segments_kernel,
 *     _kernels.py:161-182, driven by render.segment_batch render.py:105-124) */
int dot_trace_count(const dot_tree_view* tree, const double* origins, const double* dirs,
                    int64_t n_rays, double t_near, double t_far, int64_t* counts,
                    void* stream);
int dot_trace_fill(const dot_tree_view* tree, const double* origins, const double* dirs,
                   int64_t n_rays, double t_near, double t_far, const int64_t* offsets,
                   int64_t* seg_leaf, double* seg_t, double* seg_delta, void* stream);

/* --- fused forward: traverse + composite with early termination
 *     (replaces segment_batch + composite_kernel, _kernels.py:185-224, as
 *     called by render.render_rays render.py:134-152).  Any output may be
 *     NULL.  depth = sum_i T_i Q_i (t_i + delta_i/2) (not in the reference). */
int dot_render_fwd(const dot_tree_view* tree, const double* origins, const double* dirs,
                   int64_t n_rays, const double* background, double early_stop_eps,
                   double t_near, double t_far, float* rgb, float* t_final, float* wsum,
                   float* depth, void* stream);

/* --- camera rendering with in-kernel rays (render.render_image,
 *     render.py:228-241, over scene_io.Camera.rays, scene_io.py:77-91):
 *     cam_to_world is the host 4x4 row-major matrix (f64, read at launch),
 *     rgb is f32 [height*width*3] row-major; t_final / depth may be NULL.
 *     Each warp renders an 8x4 pixel tile. */
int dot_render_camera(const dot_tree_view* tree, const double* cam_to_world, double focal,
                      int32_t width, int32_t height, const double* background,
                      double early_stop_eps, float* rgb, float* t_final, float* depth,
                      void* stream);

/* --- many views in one launch (render_image over a camera list): n_views
 *     host 4x4 cam_to_world matrices (row-major, [n_views][16]) and focal
 *     lengths, one shared width/height; rgb is [n_views][height][width][3]
 *     f32, t_final / depth [n_views][height][width] or NULL.  One launch
 *     drains one wave tail instead of one per view. */
int dot_render_cameras(const dot_tree_view* tree, const double* cam_to_world, const double* focal,
                       int32_t n_views, int32_t width, int32_t height, const double* background,
                       double early_stop_eps, float* rgb, float* t_final, float* depth, void* stream);

/* --- fused forward + backward + signal (replaces segment_batch + grad_kernel
 *     + scatter_kernel, _kernels.py:227-346, as called by
 *     render.render_and_backprop render.py:175-225).
 *     Accumulates (+=) into grad_sigma[capacity] f32, grad_sh[capacity*gsh_stride]
 *     f32, signal[capacity] f64, loss_sum[1] f64 (sum over rays of the squared
 *     error; the caller divides by n), and sets touched[capacity] u8 to 1 for
 *     every traversed leaf (post-cut segments included, like scatter_kernel).
 *     grad_scale is the reference's 2/n (2/n_global when rays are sharded).
 *     origins/dirs/targets hold n_pool rays; ray_index (may be NULL =
 *     0..n_rays-1, then n_pool >= n_rays) names the n_rays rays to process:
 *     ray r of the batch is origins/dirs/targets[ray_index[r]], read in place
 *     (a coherence-sorted order, or a batch drawn from a larger resident ray
 *     pool, without gathering).  An index outside [0, n_pool) skips that ray
 *     and makes loss_sum NaN (kernels cannot raise).  rgb_out (f32, indexed
 *     like the arrays) may be NULL.  warp_order (may be NULL): block b
 *     processes batch rays [32 w, 32 w + 32) with w = warp_order[b], a
 *     permutation of 0..ceil(n/32)-1 (dot_sched_order); results do not depend
 *     on it.  ray_used (may be NULL) receives each batch ray's
 *     cost (composited + post-cut / 2 segments, u16, saturating) for
 *     dot_sched_update; ray_cost (may be NULL, indexed like the arrays)
 *     receives the same value at each ray's own index (a ray pool's cost
 *     column for dot_sched_order_costs).
 *     weight_sum / weight_max (f64 [capacity], may be NULL; no reference
 *     counterpart, defined by oracle_weights): per leaf += / max= the
 *     compositing weight T_i Q_i of every composited segment.
 *     flags: 0, or bit 15 = per-lane REDs instead of the warp-cooperative
 *     SH-row scatter (implied for capacity > 2^27); other bits are rejected. */
int dot_render_bwd(const dot_tree_view* tree, const double* origins, const double* dirs,
                   const double* targets, int64_t n_pool, const int64_t* ray_index,
                   const int32_t* warp_order, uint16_t* ray_used, uint16_t* ray_cost, int64_t n_rays,
                   const double* background, double early_stop_eps, double t_near, double t_far,
                   double grad_scale, float* grad_sigma, float* grad_sh, int32_t gsh_stride,
                   double* signal, uint8_t* touched, double* loss_sum, float* rgb_out,
                   double* weight_sum, double* weight_max, int32_t flags, void* stream);

/* --- signal-only forward (the training signal of grad_kernel +
 *     scatter_kernel, _kernels.py:249-282, 337, without gradients; what
 *     signals.SignalBuffer.accumulate, signals.py:58-69, consumes): per
 *     composited (pre-cut) segment signal[leaf] += Q = 1 - exp(-sigma delta),
 *     weight_sum[leaf] += T_i Q_i, weight_max[leaf] = max(., T_i Q_i) (f64
 *     [capacity] each), touched[leaf] = 1 for every traversed leaf including
 *     post-cut ones; every output may be NULL (at least one must be given).
 *     Reads sigma only (no SH rows).  Rays as in dot_render_bwd; indices
 *     outside [0, n_pool) are skipped and counted into *invalid_rays (u64,
 *     device, may be NULL). */
int dot_signal_fwd(const dot_tree_view* tree, const double* origins, const double* dirs, int64_t n_pool,
                   const int64_t* ray_index, int64_t n_rays, double early_stop_eps, double t_near,
                   double t_far, double* signal, double* weight_sum, double* weight_max,
                   uint8_t* touched, uint64_t* invalid_rays, void* stream);

/* --- deterministic fused forward + backward: same inputs and outputs as
 *     dot_render_bwd (accumulates into the same buffers; rgb not returned),
 *     but the per-leaf reduction runs in the reference's order --
 *     scatter_kernel (_kernels.py:327-346) sums each leaf's contributions
 *     serially over rays in batch order -- via per-segment records, a radix
 *     sort by (leaf, original ray index) and a sequential f64 sum per leaf.
 *     Results are bit-identical across runs.  ray_index (may be NULL) must
 *     be a permutation of 0..n-1: rays are read at ray_index[r] and the
 *     reduction order is the order of the caller's arrays, so the batch may
 *     be processed in any (e.g. coherence-sorted) order.  warp_order and
 *     ray_used as in dot_render_bwd (may be NULL).  Synchronises the stream
 *     (the record count sizes the sort). */
int dot_render_bwd_sorted(const dot_tree_view* tree, const double* origins, const double* dirs,
                          const double* targets, const int64_t* ray_index,
                          const int32_t* warp_order, uint16_t* ray_used, int64_t n_rays,
                          const double* background, double early_stop_eps, double t_near,
                          double t_far, double grad_scale, float* grad_sigma, float* grad_sh,
                          int32_t gsh_stride, double* signal, uint8_t* touched, double* loss_sum,
                          void* stream);

/* --- warp scheduling from a learned cost table (no reference
 *     counterpart): table is u16 [2^24 + 2^27]: a coarse part indexed by the
 *     top 24 bits and a fine part by the top 27 bits of the 31-bit coherence
 *     key (dot_ray_keys32) of a warp's first ray, each holding a decaying
 *     max of the per-warp max composited-segment count seen there (the fine
 *     entry is used when populated).
 *     dot_sched_order writes warp_order[ceil(n/32)]: chunks of consecutive
 *     warps of the key-sorted batch (16 warps, doubled until at most 2048
 *     chunks), costliest predicted chunk first; dot_sched_update folds a
 *     finished batch's ray_used into the table.  Order only: results are identical for any order. */
int dot_sched_order(const int32_t* sorted_keys, int64_t n_rays, const uint16_t* table, int32_t* warp_order,
                    void* stream);
int dot_sched_update(const int32_t* sorted_keys, const uint16_t* ray_used, int64_t n_rays, uint16_t* table,
                     void* stream);

/* --- warp order from per-ray costs (no reference counterpart; order only):
 *     ray_cost is a cost column indexed like the ray arrays (u16: composited +
 *     post-cut / 2 segments, what dot_ray_costs computes and dot_render_bwd
 *     refreshes through its ray_cost output); slot i of the batch costs
 *     ray_cost[ray_index[i]] (ray_index may be NULL; an index outside
 *     [0, n_costs) costs 0); a warp costs the max of
 *     its 32 slots, chunks of
 *     `chunk` consecutive warps are ranked by their costliest warp, descending
 *     (longest first), and warp_order[ceil(n/32)] lists the warps in that
 *     order for dot_render_bwd. */
int dot_sched_order_costs(const uint16_t* ray_cost, int64_t n_costs, const int64_t* ray_index, int64_t n_rays,
                          int32_t chunk, int32_t* warp_order, void* stream);

/* --- per-ray schedule cost of a ray set (no reference counterpart):
 *     cost[i] = composited + post-cut / 2 segments of ray ray_index[i] (or i),
 *     u16 saturating -- what dot_render_bwd reports per slot in ray_used --
 *     for the first epoch of a ray pool (later epochs reuse the backward's own
 *     counts).  Rays as in dot_render_bwd; out-of-range indices get 0. */
int dot_ray_costs(const dot_tree_view* tree, const double* origins, const double* dirs, int64_t n_pool,
                  const int64_t* ray_index, int64_t n_rays, double early_stop_eps, double t_near,
                  double t_far, uint16_t* cost, void* stream);

/* --- coherence keys (no reference counterpart): keys[i] = (origin Morton
 *     << 32) | octahedral-direction Morton; sorting a batch by them puts rays
 *     that walk the same cells into the same warps.  Results are sums over
 *     rays, so the order changes only speed. */
int dot_ray_keys(const dot_tree_view* tree, const double* origins, const double* dirs,
                 int64_t n_rays, uint64_t* keys, void* stream);
/* 31-bit keys (origin 4 bits/axis, direction 10x9 bits): half the sort
 * passes.  n_pool / ray_index (may be NULL) as in dot_render_bwd; an
 * out-of-range index gets key 0. */
int dot_ray_keys32(const dot_tree_view* tree, const double* origins, const double* dirs, int64_t n_pool,
                   const int64_t* ray_index, int64_t n_rays, int32_t* keys, void* stream);

/* keys[i] = pool_keys[ray_index[i]] (0 for an index outside [0, n_pool)):
 * a batch's keys gathered from its resident pool's dot_ray_keys32 keys. */
int dot_gather_keys(const int32_t* pool_keys, int64_t n_pool, const int64_t* ray_index, int64_t n_rays,
                    int32_t* keys, void* stream);

/* The batch's coherence order: radix sort of keys (dot_ray_keys32) by bits
 * [begin_bit, 31) carrying ray_index (NULL: the batch positions) as the
 * value, so sorted_index is directly the ray_index of dot_render_bwd and
 * sorted_keys feeds dot_sched_order / dot_sched_update.  Ties keep the
 * batch order (stable). */
int dot_plan_sort(const int32_t* keys, const int64_t* ray_index, int64_t n_rays, int32_t begin_bit,
                  int32_t* sorted_keys, int64_t* sorted_index, void* stream);

/* Coherence order of a batch from a RANKED ray pool, without a sort (no
 * reference counterpart; replaces dot_gather_keys / dot_ray_keys32 +
 * dot_plan_sort + dot_sched_order_costs).  rank[ray] is the pool ray's
 * position in key order, order[position] the ray there (inverse
 * permutations, built once per pool, e.g. from dot_ray_keys + a sort); rank
 * == NULL: ray_index already holds key positions.  ray_index[i] names the
 * batch's i-th ray in the pool.  sorted_index receives the batch in key
 * order, as
 *   DOT_PLAN_POSITIONS  key positions (the pool's arrays stored in key
 *                       order: the positions ARE the rays; fastest)
 *   DOT_PLAN_POOL_RAYS  pool rays order[position] (order required)
 *   DOT_PLAN_SLOTS      batch slots i (a staged batch whose arrays hold the
 *                       rays by slot; ray_index = their dataset ids)
 * Repeated rays and indices outside [0, n_pool) follow the placed ones, so
 * sorted_index is always a permutation of the batch.  warp_order
 * (optional, [ceil(n_rays / 32)]): the backward's warp launch order from
 * ray_cost (u16, indexed by sorted_index's values: [n_pool] for positions /
 * pool rays, [n_rays] for slots): sorted_index is then also regrouped --
 * inside each window of 128 slots the rays are re-sorted by cost
 * (descending, ties in key order) so each warp holds rays of similar
 * length -- and the warps are ordered in chunks of `chunk` consecutive
 * warps by descending max cost, a short last chunk last (what
 * dot_sched_order_costs gives for the regrouped sorted_index).  One
 * cooperative launch (one block per SM).  workspace:
 * dot_plan_ranked_workspace(n_pool, n_rays, mode) bytes, 256-byte aligned,
 * ZEROED before its first use; every call leaves it reusable, also for
 * smaller batches of the same pool.  Calls sharing a workspace must be
 * stream-ordered.  n_pool, n_rays < 2^31. */
enum { DOT_PLAN_POSITIONS = 0, DOT_PLAN_POOL_RAYS = 1, DOT_PLAN_SLOTS = 2 };
int64_t dot_plan_ranked_workspace(int64_t n_pool, int64_t n_rays, int32_t mode);
int dot_plan_ranked(const int32_t* rank, const int32_t* order, int64_t n_pool, const int64_t* ray_index,
                    int64_t n_rays, int32_t mode, const uint16_t* ray_cost, int32_t chunk, int32_t* warp_order,
                    void* workspace, int64_t workspace_bytes, int64_t* sorted_index, void* stream);

/* --- workload statistics (measurement helper, no reference counterpart):
 *     totals[0] += traversed segments, totals[1] += composited (pre-cut)
 *     segments, totals[2] += composited segments with q > 0. */
int dot_ray_stats(const dot_tree_view* tree, const double* origins, const double* dirs,
                  int64_t n_rays, double early_stop_eps, uint64_t* totals, void* stream);

/* --- refine (DOT calibration, calibrate.py:202-238) ------------------------
 * One call runs prune (one-shot or recursive) then sample on the post-prune
 * topology and writes the refined tree directly in canonical BFS order
 * (scene_io.py:529-541).  Inputs: the tree view (payload rows indexed by
 * pool id = ~leaf word), pool_id[n_nodes] (pool id of every canonical node,
 * NULL = identity), acc[capacity] f64 accumulated signals (ignored when
 * use_sigma), parameters as CalibrationConfig (recursive: 1 = repeat the
 * prune to a fixed point, 0 = one round, -1 = no prune at all, i.e. the
 * reference's sample() alone; gamma = 0 and use_threshold = 0 disable the
 * sample, i.e. prune() alone).  Because the output size is
 * data dependent, the call is split in two:
 *   dot_refine_plan_create -> computes the selections and output sizes on the
 *       device and stores them in an opaque plan (one stream synchronisation
 *       at the end, plus one per round when recursive).  level_offsets
 *       (host, n_level_offsets = levels + 1, BFS level boundaries) may be
 *       NULL, in which case they are recomputed with one sync per level.
 *   dot_refine_apply -> writes the new node words / payload / remap and the
 *       new tree's level offsets (host array of max_levels + 1 entries).
 * Outputs of apply (device, caller-allocated to the sizes the plan reports):
 *   new_node[n_new] i32, new_sigma[n_new] f32, new_sh[n_new*sh_stride] f32
 *   (pool id == canonical id in the result; internal rows are zero),
 *   src_index[n_new] i64: canonical old node a new node descends from
 *     (itself for surviving nodes, the split leaf for its new children),
 *   src_kind[n_new] u8: 0 kept, 1 merged parent (now a leaf), 2 child of a
 *     split (payload copied), 3 split parent (now internal).
 */
typedef struct dot_refine_plan dot_refine_plan;
typedef struct dot_refine_stats {
    int64_t leaves_before, leaves_after;
    int64_t merges_applied, splits_applied, recursion_rounds;
    int64_t n_new_nodes;
} dot_refine_stats;

int dot_refine_plan_create(const dot_tree_view* tree, const int32_t* pool_id,
                           const double* acc, int32_t use_sigma, double tau, double gamma,
                           int32_t recursive, int32_t use_threshold, double threshold,
                           const int64_t* level_offsets, int32_t n_level_offsets,
                           dot_refine_plan** plan, dot_refine_stats* stats, void* stream);
/* Merged-parent (by round, then canonical index) and split-leaf (ascending)
 * lists in canonical old indices, computed on first call (synchronises).
 * Pointers stay valid until dot_refine_plan_destroy. */
int dot_refine_plan_lists(dot_refine_plan* plan, const int64_t** merge_parents,
                          int64_t* n_merge, const int64_t** split_leaves, int64_t* n_split,
                          const int32_t** merge_round, void* stream);
int dot_refine_apply(const dot_refine_plan* plan, const dot_tree_view* tree,
                     int32_t* new_node, float* new_sigma, float* new_sh,
                     int64_t* src_index, uint8_t* src_kind, int64_t* level_offsets_out,
                     int32_t max_levels, int32_t* n_levels_out, void* stream);
/* Per old canonical node, the prune round (1-based) that merged it, 0 = not
 * merged: out[n_nodes] i32 device (optimizer-state remap, optim.py:89-104). */
int dot_refine_plan_merge_rounds(const dot_refine_plan* plan, int32_t* out, void* stream);
void dot_refine_plan_destroy(dot_refine_plan* plan);

/* --- optimizer (optim.rmsprop_step, optim.py:107-135): sparse RMSProp over
 *     leaves with touched[pid] != 0; sigma clamped >= 0.  v_* are f64.
 *     flags bit 0 ("consume"): zero each updated row's gradients after use,
 *     so the next batch can accumulate into the same buffers without a
 *     memset (rows that were not touched hold zero gradients already). */
int dot_rmsprop_step(float* sigma, float* sh, int32_t sh_stride, int32_t n_sh,
                     double* v_sigma, double* v_sh, float* grad_sigma,
                     float* grad_sh, int32_t gsh_stride, const uint8_t* touched,
                     int64_t capacity, double beta, double eps, double lr_sigma,
                     double lr_sh, int32_t flags, void* stream);

/* The same update for a sparse step (a small batch touches few rows): the
 * touched rows are listed first and only they are visited (the dense update's
 * grid covers the whole capacity).  Same arguments and results; layouts the
 * vectorised update does not take fall back to dot_rmsprop_step. */
int dot_rmsprop_step_sparse(float* sigma, float* sh, int32_t sh_stride, int32_t n_sh,
                            double* v_sigma, double* v_sh, float* grad_sigma,
                            float* grad_sh, int32_t gsh_stride, const uint8_t* touched,
                            int64_t capacity, double beta, double eps, double lr_sigma,
                            double lr_sh, int32_t flags, void* stream);

/* --- the same update with f32 second moments (opt-in, no reference
 *     counterpart: octrf keeps f64 state, optim.py:70-72).  Arithmetic is
 *     f64 with v widened on read and rounded once on store; results are
 *     within float tolerance of dot_rmsprop_step and the state traffic is
 *     halved.  sh, grad_sh and v_sh must be 16-byte aligned. */
int dot_rmsprop_step_f32state(float* sigma, float* sh, int32_t sh_stride, int32_t n_sh,
                              float* v_sigma, float* v_sh, float* grad_sigma, float* grad_sh,
                              int32_t gsh_stride, const uint8_t* touched, int64_t capacity,
                              double beta, double eps, double lr_sigma, double lr_sh,
                              int32_t flags, void* stream);

/* --- multi-GPU update fused with its collective (one node, peer memory
 *     over NVLink/NVSwitch; replaces all-reduce + rmsprop_step of the
 *     data-parallel step).  Rank `rank` of `world` calls it for the rows it
 *     owns, [row_lo, row_hi), once every rank's backward has finished: the
 *     kernel sums the W partial gradient rows (rank order, f64), applies
 *     RMSProp with the local v_* (capacity-sized; only owned rows are
 *     current), stores the updated row into every rank's payload replica and
 *     (flags bit 0) zeroes the W consumed gradient rows.  All pointers are
 *     device addresses valid on the calling GPU (peer-mapped for r != rank,
 *     e.g. torch symmetric memory); a second barrier must separate it from
 *     the next backward. */
#define DOT_MAX_PEERS 8
typedef struct dot_peer_rows {
    float* sigma[DOT_MAX_PEERS];
    float* sh[DOT_MAX_PEERS];
    float* grad_sigma[DOT_MAX_PEERS];
    float* grad_sh[DOT_MAX_PEERS];
    const uint8_t* touched[DOT_MAX_PEERS];
    int32_t world;
    int32_t rank;
} dot_peer_rows;
int dot_rmsprop_step_peers(const dot_peer_rows* peers, int32_t sh_stride, int32_t n_sh,
                           int32_t gsh_stride, double* v_sigma, double* v_sh, int64_t row_lo,
                           int64_t row_hi, double beta, double eps, double lr_sigma, double lr_sh,
                           int32_t flags, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* DOT_B200_H */
