/*
 * lc.h -- C ABI of the B200 (sm_100a) loop-closing fuse/correct core.
 *
 * The data-parallel core of the GPU loop-closing module of arXiv 2603.17201
 * ("FastLoop", an ORB-SLAM3 loop closer), re-designed for B200:
 *
 *   lc_upload_map            GPU-resident keyframe / map-point storage, each
 *                            keyframe transferred once as a "lightweight wrapper
 *                            structure" (§IV.A; §IV.E)
 *   lc_correct_sim3          Sim3 correction of the window keyframes and the map
 *                            points they observe (§III.B), and
 *                            propagation of optimised keyframe Sim3s to the whole
 *                            map (§IV.F)
 *   lc_fuse                  loop fusion: project the loop map points into every
 *                            connected keyframe, match descriptors "within close
 *                            spatial proximity", merge duplicates (
 *                            PAPER.md:226-228 §IV.D.3)
 *   lc_search_by_projection  batched projection search PS1 / PS2a||PS2b / PS3a-c
 *                            over (keyframe, Sim3, parameter set) pairs, results
 *                            returned as one batch per pair (§IV.C;
 *                            PAPER.md:215-224 §IV.D.1-2)
 *
 * The paper states no matching constants or tie-breaks; the readings this ABI
 * implements are listed in DESIGN.md ("Readings", A1-A32) and are identical to
 * the CPU oracle's (oracle/lc_oracle.c), which shares no code with this library.
 *
 * Conventions
 *  - Poses are world->camera Sim3 transforms, p_c = s * (R p) + t, R row-major
 *    (reading A1). Keyframe poses are SE3 (s = 1) in the store.
 *  - Indices are dense and 0-based: keyframe k, map point q, feature f. A
 *    keyframe's features are the global range [kf_feat_begin[k], kf_feat_begin[k+1]);
 *    "local feature index" = global index - kf_feat_begin[k].
 *  - Packed match words: (H << 32) | q as int64, H = Hamming distance in
 *    [0, 256]; LC_NONE (INT64_MAX) = empty. Signed int64 so that an NCCL MIN
 *    all-reduce merges them (lowest H, then lowest q).
 *  - Pointers marked [host|dev] may be host memory (pageable or pinned) or
 *    device memory of the context's device; the library detects which
 *    (cudaPointerGetAttributes): device data is used in place, page-locked host
 *    data is copied directly, pageable host data through the CUDA driver's staging
 *    (or the library's chunked pinned ring with LC_STAGE=1; measured slower, see
 *    lc_upload_map). Small control arrays marked [host] travel in one page-locked
 *    argument block per call (a ring of 8, so the host only waits when it laps
 *    it). Pointers marked [host] must be host memory (arrays the library
 *    validates and uses to configure launches).
 *  - Asynchrony: every call enqueues work on `cuda_stream` (a cudaStream_t,
 *    NULL = legacy default stream) and returns; outputs (device or host) are
 *    valid once that stream has reached the call's work. Inputs must stay valid
 *    until then (as with cuBLAS). A context is single-stream and not
 *    thread-safe; use one per device per process.
 *  - Ownership: the library owns the device map store (allocated once by
 *    lc_upload_map and reused) and a scratch arena that only grows (no
 *    allocation in steady state). Caller buffers are borrowed for the call.
 *  - Errors: every call returns an lc_status; no C++ exception crosses the ABI.
 *    LC_EINVAL / LC_ERANGE / LC_ECAPACITY / LC_ESTATE are detected before any
 *    work is enqueued. LC_ECUDA makes the context unusable until lc_destroy.
 *    lc_last_error() describes the last failure.
 */
#ifndef LC_H_
#define LC_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define LC_ABI_VERSION 2
#define LC_NONE INT64_MAX
#define LC_MAX_FEAT_PER_KF 8192
#define LC_MAX_LEVELS 16

typedef struct lc_ctx lc_ctx;

typedef enum {
  LC_OK = 0,
  LC_EINVAL = -1,     /* malformed argument (null required pointer, bad size, bad params) */
  LC_ESTATE = -2,     /* call not valid in the context's state (e.g. no map uploaded)    */
  LC_ECUDA = -3,      /* CUDA runtime failure; context unusable                         */
  LC_ENOMEM = -4,     /* device or pinned allocation failed                             */
  LC_ERANGE = -5,     /* index out of range (keyframe, map point, feature, octave)       */
  LC_ECAPACITY = -6   /* a per-keyframe limit was exceeded (LC_MAX_FEAT_PER_KF)          */
} lc_status;

/* Sim3 / SE3 transform: p' = s * (R p) + t, R row-major. 104 bytes. */
typedef struct { double R[9]; double t[3]; double s; } lc_sim3;

/* Camera: model 0 = pinhole, 1 = Kannala-Brandt-8 (reading A29). Image bounds
 * are half-open [min_x, max_x) x [min_y, max_y) (reading A4). */
typedef struct {
  int32_t model;
  int32_t reserved;
  double fx, fy, cx, cy;
  double k[4];
  double min_x, max_x, min_y, max_y;
} lc_camera;

/* Scale pyramid and grid: n_levels (<= LC_MAX_LEVELS), scale_factor (ORB: 8, 1.2),
 * per-keyframe feature grid grid_cols x grid_rows (ORB: 64 x 48). */
typedef struct {
  int32_t n_levels;
  int32_t grid_cols, grid_rows;
  int32_t reserved;
  double scale_factor;
} lc_map_params;

/* SoA view of the map to upload. All arrays [host|dev], borrowed for the call. */
typedef struct {
  int32_t n_kf, n_feat, n_mp;
  int32_t reserved;
  const lc_sim3* kf_pose;        /* [n_kf] world->camera, s = 1                     */
  const int32_t* kf_cam;         /* [n_kf] camera index                             */
  const int32_t* kf_feat_begin;  /* [n_kf+1] CSR into the feature arrays            */
  const float* feat_uv;          /* [n_feat][2] keypoint pixel (u, v)               */
  const uint8_t* feat_octave;    /* [n_feat] pyramid level < n_levels               */
  const float* feat_angle;       /* [n_feat] keypoint angle, degrees                */
  const uint8_t* feat_desc;      /* [n_feat][32] 256-bit ORB descriptor             */
  const int32_t* feat_mp;        /* [n_feat] associated map point, -1 = none        */
  const float* mp_pos;           /* [n_mp][3] world position                        */
  const float* mp_normal;        /* [n_mp][3] mean viewing direction (unit)         */
  const float* mp_max_dist;      /* [n_mp] scale-invariance max distance dmax       */
  const uint8_t* mp_desc;        /* [n_mp][32] representative descriptor           */
  const float* mp_angle;         /* [n_mp] angle of the reference observation, deg  */
  const int32_t* mp_ref_kf;      /* [n_mp] reference keyframe                       */
  const uint8_t* mp_flags;       /* [n_mp] bit0 = bad                               */
} lc_map_view;

/* Mutable map state, for download/inspection. Any pointer may be NULL (skipped). */
typedef struct {
  lc_sim3* kf_pose;              /* [n_kf]                                          */
  int32_t* feat_mp;              /* [n_feat] original feature order                 */
  float* mp_pos;                 /* [n_mp][3]                                       */
  uint8_t* mp_flags;             /* [n_mp]                                          */
  int32_t* mp_replaced_by;       /* [n_mp] survivor of a fused victim, -1 = none    */
  int32_t* mp_nobs;              /* [n_mp] number of slots holding the map point    */
  float* mp_normal;              /* [n_mp][3] viewing direction (lc_refresh_mappoints) */
  float* mp_max_dist;            /* [n_mp] depth-range bound                        */
  uint8_t* mp_desc;              /* [n_mp][32] distinctive descriptor               */
} lc_map_state;

/* Matching parameters (readings A8-A15). th: window half-size at level 0 in px
 * (Fuse: 4); max_hamming: inclusive threshold in [0, 256]; ratio test enabled
 * iff ratio_den > 0, rejecting iff ratio_den*best > ratio_num*second;
 * check_orientation: 30-bin rotation histogram, keep the three maxima. */
typedef struct {
  int32_t th;
  int32_t max_hamming;
  int32_t ratio_num, ratio_den;
  int32_t check_orientation;
} lc_match_params;

/* Optional per-query debug outputs [host|dev], indexed by query (see lc_fuse /
 * lc_search_by_projection). best: status < 0 (cull code, LC_Q_*) or
 * (H_best << 48) | (H_second << 32) | uint32(local feature f_best), with
 * H_best = H_second = 256 and f = 0xFFFFFFFF when the window is empty;
 * uv: projected pixel (fp64, 2 per query; 0 when culled before projection);
 * ncand: number of candidates |C(k,q)|. Any member may be NULL. */
typedef struct {
  int64_t* best;
  double* uv;
  int32_t* ncand;
} lc_query_debug;

/* query cull codes in lc_query_debug.best */
enum { LC_Q_BAD = -1, LC_Q_FOUND = -2, LC_Q_DEPTH = -3, LC_Q_BOUNDS = -4,
       LC_Q_DIST = -5, LC_Q_ANGLE = -6 };

/* Counter slots of out_counts (int64, overwritten by each call). */
enum {
  LC_COUNT_QUERIES = 0,    /* (keyframe, map point) queries                          */
  LC_COUNT_SKIP_BAD,       /* query map point flagged bad                            */
  LC_COUNT_SKIP_FOUND,     /* map point already in the keyframe (reading A19)        */
  LC_COUNT_CULL_DEPTH,     /* z <= 0                                                 */
  LC_COUNT_CULL_BOUNDS,    /* projection outside the image                           */
  LC_COUNT_CULL_DIST,      /* outside [0.8 dmax / s_{L-1}, 1.2 dmax]                 */
  LC_COUNT_CULL_ANGLE,     /* PO . n < 0.5 |PO|                                      */
  LC_COUNT_CANDIDATES,     /* sum |C(k,q)|: candidate Hamming matches (the metric)   */
  LC_COUNT_NO_CAND,        /* queries with an empty window                           */
  LC_COUNT_OVER_TH,        /* best H > max_hamming                                   */
  LC_COUNT_RATIO_REJ,      /* ratio test failed                                      */
  LC_COUNT_PROPOSALS,      /* (keyframe, feature, q, H) proposals                    */
  LC_COUNT_WINNERS,        /* features with a winning proposal                       */
  LC_COUNT_ORIENT_REJ,     /* winners removed by the rotation histogram              */
  LC_COUNT_ADD,            /* fuse: winner on an empty slot                          */
  LC_COUNT_VICTIM_PROP,    /* fuse: winner on a slot holding a fusable map point     */
  LC_COUNT_LOOP_SKIP,      /* fuse: slot holds a loop map point (reading A21)        */
  LC_COUNT_BAD_SLOT,       /* fuse: slot holds a bad map point                       */
  LC_COUNT_VICTIMS,        /* fuse apply: distinct victims                           */
  LC_COUNT_REWIRED,        /* fuse apply: slots redirected to a survivor             */
  LC_COUNT_DUP_CLEARED,    /* fuse apply: duplicate slots cleared (reading A22)      */
  LC_COUNT_ADDED,          /* fuse apply: new associations kept                      */
  LC_COUNT_CORR_KF,        /* correction: keyframe poses written                     */
  LC_COUNT_CORR_MP,        /* correction: map points moved                           */
  LC_COUNT_REFRESH_MP,     /* refresh: map points refreshed (not bad, >= 1 observation) */
  LC_COUNT_REFRESH_OBS,    /* refresh: observations visited                           */
  LC_COUNT_CONN_KF,        /* connections: keyframes recounted                        */
  LC_COUNT_CONN_EDGES,     /* connections: edges kept (before max_edges truncation)   */
  LC_COUNT_RANSAC_HYP,     /* Sim3 RANSAC: hypotheses evaluated (valid samples)       */
  LC_COUNT_RANSAC_INLIERS, /* Sim3 RANSAC: inliers of the selected models             */
  LC_COUNT_REFINE_ITERS,   /* Sim3 refinement: Gauss-Newton steps taken              */
  LC_COUNT_REFINE_INLIERS, /* Sim3 refinement: inliers under the refined models      */
  LC_COUNT_PGO_ITERS,      /* pose graph: Levenberg-Marquardt iterations (linear solves) */
  LC_COUNT_PGO_ACCEPTED,   /* pose graph: accepted steps                             */
  LC_COUNT_PGO_SOLVER_ITERS, /* pose graph: conjugate-gradient iterations, all solves */
  LC_COUNT_PGO_STOP,       /* pose graph: stop reason (LC_PGO_STOP_*)                 */
  LC_COUNT_PGO_BAND,       /* pose graph: 1 + block bandwidth of the banded solve, 0 = CG */
  LC_COUNT_FORCED,         /* fuse: forced loop matches turned into an ADD or a victim (O9.4) */
  LC_COUNT_EDGE_AMB,       /* queries whose bounds or window decision lies within 1e-4 px of
                              the edge (SURVEY.md §8(c) "Edge-ambiguous"): the only queries
                              where a differently-rounded projection may decide otherwise */
  LC_COUNT_PGO_CR_LEVELS,  /* pose graph: block cyclic-reduction levels (0 = not that solver) */
  LC_NCOUNT
};

/* lc_correct_sim3 modes */
#define LC_CORRECT_WINDOW 1
#define LC_CORRECT_ALL 2
#define LC_DRY_RUN 4          /* with LC_CORRECT_WINDOW: a batch of corrections, nothing written back */
/* lc_fuse phases */
#define LC_FUSE_PLAN 1
#define LC_FUSE_APPLY 2
#define LC_FUSE_ALL 3

/* ---------------------------------------------------------------------------
 * Context
 * ------------------------------------------------------------------------- */

/* Create a context on CUDA device `device` (sm_100a). *out receives it.
 * Errors: LC_EINVAL (out NULL), LC_ECUDA (no such device / not sm_100). */
lc_status lc_create(lc_ctx** out, int32_t device);

/* Destroy a context and free everything it owns (synchronises its device). */
lc_status lc_destroy(lc_ctx* ctx);

/* Message of the last failure on ctx (static storage owned by ctx), or of the
 * last lc_create failure when ctx is NULL. Never NULL. */
const char* lc_last_error(const lc_ctx* ctx);

/* Number of this library's kernels launched by ctx since creation (evidence
 * for the benchmark's gpu_launches). */
int64_t lc_kernel_launches(const lc_ctx* ctx);

/* ---------------------------------------------------------------------------
 * Device-time accounting (tracing). When enabled, each launch group of the
 * families below is bracketed by CUDA events on the call's stream; lc_profile_read
 * waits for the recorded events and returns the accumulated device milliseconds
 * and kernel launches per family since the last enable (ms/launches [host],
 * LC_NPROF entries each). Enabling (on = 1) resets the accumulators; on = 0 stops.
 * ------------------------------------------------------------------------- */
enum { LC_PROF_UPLOAD = 0, LC_PROF_CORRECT_WINDOW, LC_PROF_CORRECT_ALL, LC_PROF_FUSE_PREP,
       LC_PROF_MATCH, LC_PROF_RESOLVE, LC_PROF_APPLY, LC_PROF_SBP_MATCH, LC_PROF_SBP_RESOLVE,
       LC_PROF_STATE, LC_PROF_PROJECT, LC_PROF_REFRESH, LC_PROF_CONN, LC_PROF_RANSAC, LC_PROF_REFINE,
       LC_PROF_PGO, LC_NPROF };
lc_status lc_profile_enable(lc_ctx* ctx, int32_t on);
lc_status lc_profile_read(lc_ctx* ctx, double* ms, int64_t* launches);

/* ---------------------------------------------------------------------------
 * lc_refresh_mappoints -- map-point refresh after a merge (
 * PAPER.md:95 "identify and merge duplicate map points" -- the refresh of the
 * merged points is inherited ORB-SLAM3 behaviour, readings A33-A37).
 *
 * For each selected map point that is not bad and has >= 1 observation (the
 * (keyframe, feature) slots holding it, in ascending global feature order, A34):
 *   what & LC_REFRESH_DESC  : descriptor <- the observation descriptor with the
 *     least median Hamming distance to all observation descriptors (median =
 *     element floor((N-1)/2) of the sorted row, first observation on ties, A35);
 *   what & LC_REFRESH_NORMAL: normal <- fl32((sum_i (p - O_i) / |p - O_i|) / N) in
 *     fp64, observation order, O_i the camera centre of the observing keyframe
 *     (zero-length terms skipped and not counted, A36); depth bound dmax <-
 *     fl32(|p - O_ref| * s_level), level = octave of the reference keyframe's first
 *     observation; unchanged when the reference keyframe does not observe it (A37).
 *   n, mp_idx [host|dev] nullable: the points to refresh (NULL: all n_mp, n ignored);
 *     out-of-range indices are skipped.
 *   out_counts [host|dev] nullable, [LC_NCOUNT] (REFRESH_MP, REFRESH_OBS).
 * Errors: LC_EINVAL (bad what / n < 0), LC_ESTATE (no map).
 * ------------------------------------------------------------------------- */
enum { LC_REFRESH_DESC = 1, LC_REFRESH_NORMAL = 2 };
lc_status lc_refresh_mappoints(lc_ctx* ctx, int32_t n, const int32_t* mp_idx, int32_t what,
                               int64_t* out_counts, void* cuda_stream);

/* ---------------------------------------------------------------------------
 * lc_update_connections -- covisibility recount after the merge (SURVEY.md §8(f)
 * f4; "creates new connections in the covisibility and essential
 * graphs"; readings A38-A40). The paper keeps this step on
 * the CPU; here it runs on the device observation lists.
 *
 * For each selected keyframe k (kf_idx [host|dev] nullable: all n_kf, n ignored):
 *   weight(k, k2) = number of distinct non-bad map points held by both k and k2 != k;
 *   edges: every k2 with weight >= th, or, if there is none, the single strongest
 *   (max weight, lowest id); ordered by weight descending, then keyframe id.
 *   out_n [host|dev] [n]: number of edges of row i (may exceed max_edges; any number
 *   of edges is ranked exactly -- the first 2048 in shared memory, beyond that against
 *   the weight array);
 *   out_kf, out_w [host|dev] nullable, [n][max_edges]: the first min(out_n[i],
 *   max_edges) edges of row i (the rest of the row is left unchanged).
 *   out_counts [host|dev] nullable, [LC_NCOUNT] (CONN_KF, CONN_EDGES).
 * Errors: LC_EINVAL (n < 0, max_edges < 0, th < 1, n_kf > 40000), LC_ESTATE (no map).
 * ------------------------------------------------------------------------- */
lc_status lc_update_connections(lc_ctx* ctx, int32_t n, const int32_t* kf_idx, int32_t th,
                                int32_t max_edges, int32_t* out_n, int32_t* out_kf,
                                int32_t* out_w, int64_t* out_counts, void* cuda_stream);

/* ---------------------------------------------------------------------------
 * lc_sim3_ransac -- batched Sim3 estimation of region detection (SURVEY.md §8(f)
 * f3; "estimating the relative pose between the new keyframe and the
 * matched one"; PAPER.md:200 hypotheses evaluated in parallel; DESIGN.md readings
 * A41-A44). One problem per candidate keyframe pair b, correspondences
 * [prob_begin[b], prob_begin[b+1]) (CSR):
 *   P1, P2 [host|dev] [n_corr][3] fp64: the matched map points in camera-1 / camera-2
 *     coordinates; uv1, uv2 [host|dev] [n_corr][2]: their keypoints; sigma2_1,
 *     sigma2_2 [host|dev] [n_corr]: level variances; cam1, cam2 [host] [n_prob]:
 *     camera indices of the uploaded cameras.
 *   samples [host|dev] [n_prob][n_iter][3]: the RANSAC draws (indices local to the
 *     problem; random numbers are inputs, A41); a sample with a repeated or
 *     out-of-range index is skipped.
 *   Per valid sample: S12 (p1 ~ s R p2 + t) by Horn's closed form (A42, fix_scale:
 *   s = 1); inliers = correspondences whose reprojection errors in both images are
 *   below chi2 * sigma^2 (A43). The selected model has the most inliers (first
 *   iteration on ties); with refit != 0 it is re-estimated on all its inliers (A44).
 *   out_S12 [host|dev] [n_prob] (all zero if no valid sample), out_inliers
 *   [host|dev] [n_prob], out_mask [host|dev] [n_corr] (inliers of the selected
 *   sample model); out_counts [LC_NCOUNT] (RANSAC_HYP, RANSAC_INLIERS).
 * Errors: LC_EINVAL (bad sizes, camera index), LC_ESTATE (no map: cameras).
 * ------------------------------------------------------------------------- */
lc_status lc_sim3_ransac(lc_ctx* ctx, int32_t n_prob, const int32_t* prob_begin, const double* P1,
                         const double* P2, const float* uv1, const float* uv2, const float* sigma2_1,
                         const float* sigma2_2, const int32_t* cam1, const int32_t* cam2,
                         const int32_t* samples, int32_t n_iter, double chi2, int32_t fix_scale,
                         int32_t refit, lc_sim3* out_S12, int32_t* out_inliers, uint8_t* out_mask,
                         int64_t* out_counts, void* cuda_stream);

/* ---------------------------------------------------------------------------
 * lc_sim3_refine -- Sim3 refinement of region detection (
 * SPEC.md refine_sim3; readings A45-A48): Gauss-Newton on the same
 * problems and correspondence arrays as lc_sim3_ransac, from S_init [host|dev]
 * [n_prob] (e.g. its output). Update S <- (Cayley(w), tau, 1 + sig) o S (A45),
 * central-difference Jacobians (h = 1e-6, A46), Huber weights with delta =
 * sqrt(th2) on each image's chi2, H + lambda diag(H) solved by Cholesky (A47);
 * phase 1 (<= 5 steps) on all correspondences, then those with a chi2 >= th2 are
 * dropped, phase 2 (<= max_iter steps) on the rest (EXT OptimizeSim3); a phase ends
 * when |d|^2 < 1e-20 or H is not positive definite. out_S [n_prob], out_inliers,
 * out_mask: both chi2 < th2 under the final model (A48). out_counts (REFINE_ITERS,
 * REFINE_INLIERS). Errors as lc_sim3_ransac.
 * ------------------------------------------------------------------------- */
lc_status lc_sim3_refine(lc_ctx* ctx, int32_t n_prob, const int32_t* prob_begin, const double* P1,
                         const double* P2, const float* uv1, const float* uv2, const float* sigma2_1,
                         const float* sigma2_2, const int32_t* cam1, const int32_t* cam2,
                         const lc_sim3* S_init, int32_t max_iter, double th2, double lambda,
                         lc_sim3* out_S, int32_t* out_inliers, uint8_t* out_mask, int64_t* out_counts,
                         void* cuda_stream);

/* ---------------------------------------------------------------------------
 * CUDA-graph capture: one loop event (lc_correct_sim3 WINDOW -> lc_fuse ->
 * lc_correct_sim3 ALL, or any sequence of lc_correct_sim3 / lc_fuse /
 * lc_search_by_projection calls) recorded once and replayed as a single graph
 * launch, removing per-call host work and inter-kernel launch gaps.
 *
 * lc_graph_begin(ctx, stream): opens a capture on `stream` (non-NULL, owned by
 *   the caller; relaxed capture mode). Until lc_graph_end, the calls above on
 *   `stream` are validated and RECORDED, not executed. Their [host] control
 *   arrays (window, window_S, parameters, ...) are copied at capture time into
 *   graph-owned device memory and are constants of the graph. Their [host|dev]
 *   data buffers must be device memory or page-locked host memory: they are
 *   read/written at every replay (so a pinned input can be refreshed between
 *   replays). Every other lc call, and any call on another stream, fails with
 *   LC_ESTATE while a capture is open. A failing call aborts the capture.
 * lc_graph_end(ctx, stream, out): closes the capture, instantiates the graph
 *   and returns it in *out (owned by the caller; lc_graph_destroy).
 * lc_graph_launch(ctx, graph, stream): replays the recorded calls on `stream`
 *   (stream-ordered; any stream). Each replay of a fuse call takes a fresh
 *   LoopSet epoch from a device counter, so replays are independent loop events.
 *   Profiling families are not recorded for replays; lc_kernel_launches counts
 *   the graph's kernels per replay. The host-side validation mirror of the
 *   stored WINDOW corrections reflects the capture, not the replays.
 * lc_graph_destroy(ctx, graph): synchronises the device and frees the graph and
 *   its buffers. Errors: LC_EINVAL (NULL / foreign graph), LC_ESTATE (no map,
 *   capture already open / not open), LC_ECUDA (capture or instantiate failed).
 * ------------------------------------------------------------------------- */
typedef struct lc_graph lc_graph;
lc_status lc_graph_begin(lc_ctx* ctx, void* cuda_stream);
lc_status lc_graph_end(lc_ctx* ctx, void* cuda_stream, lc_graph** out);
lc_status lc_graph_launch(lc_ctx* ctx, lc_graph* graph, void* cuda_stream);
lc_status lc_graph_destroy(lc_ctx* ctx, lc_graph* graph);

/* ---------------------------------------------------------------------------
 * lc_upload_map -- GPU-resident keyframe storage (§IV.A: "transfer
 * each newly created keyframe to GPU-resident KeyFrame Storage"; §IV.E:
 * allocated once, pinned memory).
 *
 * Packs the SoA view into the device store: map-point records (position, dmax,
 * normal, angle, descriptor) as 64-byte AoS rows; keyframe features re-ordered per
 * keyframe by a GPU counting sort into per-octave grids (octave o: the grid_cols x
 * grid_rows grid coarsened by scale_factor^o, over [min_x,max_x) x [min_y,max_y) of the
 * keyframe's camera; cell = floor((u-min_x) * cols_o / (max_x-min_x)), clamped), keeping
 * the original local index; association slots, angles and poses in original order.
 *   flags LC_UPLOAD_REPLACE: the view is the whole map; replaces any previous one.
 *   flags LC_UPLOAD_APPEND : the view holds NEW keyframes and NEW map points only,
 *     appended after the stored ones (the paper's per-keyframe transfer): keyframe i of
 *     the view becomes store keyframe n_kf_old + i, map point j becomes n_mp_old + j;
 *     feat_mp and mp_ref_kf use STORE indices (old or new entries); cams / n_cams / prm
 *     are ignored (the stored ones apply); n_obs of every referenced point is updated.
 *     The store grows geometrically (no re-allocation on most appends); a saved state
 *     (lc_state_save) is dropped. N appends give the same store as one REPLACE of the
 *     concatenated map, byte for byte.
 * Host arrays may be page-locked (copied directly: C5's 558 MB in 36-64 ms) or pageable
 * (copied by the CUDA driver's own staging, 91-108 ms; the library's chunked pinned ring,
 * LC_STAGE=1, measured slower -- 118 ms -- so it is off by default).
 * Synchronises the stream before returning (validation reads back one error count).
 *   map   [host] struct; its arrays [host|dev]
 *   cams  [host] n_cams cameras; prm [host]
 * Errors: LC_EINVAL (null arrays, n_* < 0, non-monotone kf_feat_begin, camera
 * bounds empty, n_levels outside [1, LC_MAX_LEVELS], scale_factor <= 1, grid
 * outside [1, 1024]^2 or more than 24576 cells over the octave grids, bad flags),
 * LC_ESTATE (APPEND before a map), LC_ERANGE (feat_mp / mp_ref_kf / kf_cam / octave
 * out of range), LC_ECAPACITY (a keyframe with more than LC_MAX_FEAT_PER_KF
 * features), LC_ENOMEM, LC_ECUDA. */
#define LC_UPLOAD_REPLACE 0
#define LC_UPLOAD_APPEND 1
lc_status lc_upload_map(lc_ctx* ctx, const lc_map_view* map, const lc_camera* cams,
                        int32_t n_cams, const lc_map_params* prm, int32_t flags, void* cuda_stream);

/* Copy the mutable map state out (any member NULL = skipped). [host|dev]. */
lc_status lc_download_map(lc_ctx* ctx, const lc_map_state* out, void* cuda_stream);

/* Save / restore the mutable map state (poses, associations, positions, flags,
 * replaced_by, n_obs, loop state) to / from a device-side copy: checkpoint and
 * resume of the store without host round trips. restore before save -> LC_ESTATE. */
lc_status lc_state_save(lc_ctx* ctx, void* cuda_stream);
lc_status lc_state_restore(lc_ctx* ctx, void* cuda_stream);

/* ---------------------------------------------------------------------------
 * lc_correct_sim3 -- Sim3 pose correction (§III.B).
 *
 * mode LC_CORRECT_WINDOW (reading O3; old poses read before any write-back),
 *   n_batch = 1, window = window_kf[window_begin[0] .. window_begin[1]):
 *   for window position i (window[0] must be cur_kf[0]):
 *     S_i^corr = (T_iw * inverse(T_cw)) * S_cw_corr   (S_c^corr = S_cw_corr);
 *   every non-bad map point observed by the window is re-anchored through its
 *   owner o = the first window keyframe (list order) observing it:
 *     p <- fl32( inverse(S_o^corr)( T_ow(p) ) );
 *   then T_iw <- SE3(S_i^corr) = (R, t/s). S_i^corr is kept (loop state) as the
 *   default projection transform of lc_fuse and as S^pre of LC_CORRECT_ALL.
 *   out_S_corr [host|dev] nullable, [n_window]. out_mp_* ignored.
 * mode LC_CORRECT_WINDOW | LC_DRY_RUN (reading O3', PAPER.md:200
 *   §IV.C: loop candidates are evaluated in batches): n_batch >= 1 hypotheses
 *   b = (cur_kf[b], S_cw_corr[b], window_kf[window_begin[b] .. window_begin[b+1]),
 *   window_kf[window_begin[b]] == cur_kf[b]); each gets the WINDOW arithmetic above
 *   against the map as it is, and NOTHING is written back (no pose, point or loop
 *   state changes; hypotheses are independent):
 *     out_S_corr [host|dev] required, [window_begin[n_batch]]: S_i^corr per slot;
 *     out_mp_begin [host|dev] required, [n_batch + 1]: CSR of the corrected points;
 *     out_mp_idx [out_capacity] / out_mp_pos [out_capacity][3] [host|dev]: the owned
 *       non-bad map points of hypothesis b in ascending index, fl32 positions.
 *   The call reads the point total back (one stream synchronisation) and returns
 *   LC_ECAPACITY when it exceeds out_capacity (out_mp_begin is complete, points
 *   beyond the capacity are not written). Not capturable into a graph.
 * mode LC_CORRECT_ALL (reading O10; propagation after pose-graph optimisation):
 *   S_k^pre = S_k^corr if k was in the last window, else T_kw;
 *   every non-bad map point p <- fl32( inverse(S_r^opt)( S_r^pre(p) ) ) with
 *   r = its window owner if corrected by the last WINDOW call, else mp_ref_kf;
 *   then T_kw <- SE3(S_k^opt) for every k. Consumes the loop state.
 *   S_opt [host|dev] [n_kf]. Every other argument ignored (may be NULL).
 * cur_kf, S_cw_corr, window_begin, window_kf [host] (WINDOW modes).
 * All transforms are evaluated in fp64 in the order of DESIGN.md "Sim3
 * arithmetic"; positions are stored fp32 (round to nearest).
 * out_counts [host|dev] nullable, [LC_NCOUNT] (CORR_KF, CORR_MP).
 * Errors: LC_ESTATE (no map), LC_EINVAL (bad mode, n_batch != 1 without DRY_RUN,
 * an empty window, window[0] != cur_kf, duplicate keyframes in a window, null
 * required pointer), LC_ERANGE (keyframe index), LC_ECAPACITY (DRY_RUN). */
lc_status lc_correct_sim3(lc_ctx* ctx, int32_t mode, int32_t n_batch, const int32_t* cur_kf,
                          const lc_sim3* S_cw_corr, const int32_t* window_begin,
                          const int32_t* window_kf, const lc_sim3* S_opt, lc_sim3* out_S_corr,
                          int32_t* out_mp_begin, int32_t* out_mp_idx, float* out_mp_pos,
                          int64_t out_capacity, int64_t* out_counts, void* cuda_stream);

/* ---------------------------------------------------------------------------
 * lc_fuse -- loop fusion (§IV.D.3), readings O4-O9.
 *
 * Every window keyframe k (window position i) is matched against its loop
 * map-point list L_i (win_list_begin != NULL: CSR mp_list[win_list_begin[i] ..
 * win_list_begin[i+1]); NULL: the whole mp_list for every keyframe, as
 * ORB-SLAM3's single loop-point list). For each query (k, q), q in L_i, not bad
 * and not already associated in k: project with SE3(S_k) (window_S[i], or the
 * S^corr stored by the last WINDOW correction when window_S is NULL), cull
 * (depth, bounds, distance range, view angle), predict level n, take the
 * candidates f of k with |u_f-u| < r, |v_f-v| < r, r = th * 1.2^n, octave in
 * [n-1, n]; best = argmin (H, f), second = min H of the rest (256 if none);
 * propose (k, f_best, (H<<32)|q) if H <= max_hamming and the ratio test passes.
 * Per feature the least proposal wins; the orientation filter removes winners
 * per keyframe. A winner on an empty slot is an ADD; on a slot holding a bad
 * map point or a map point of LoopSet (union of all L_i) nothing; otherwise it
 * proposes its word as the victim word of the slot's map point m (least wins).
 * APPLY (snapshot semantics, reading A18): every slot in the map holding a
 * victim m is redirected to survivor(m) = low 32 bits of victim[m]; ADDs fill
 * their slots; in each keyframe a map point occupying several slots keeps the
 * least (priority, f) slot, priority 0 unchanged / 1 ADD / 2 redirected; victims
 * get flags |= bad and replaced_by = survivor; n_obs is updated.
 *
 * Forced loop matches (reading O9.4 / A23; EXT CorrectLoop fuses the loop map
 * points matched to the current keyframe during detection before the search):
 * forced_mp [host|dev] nullable, [F(cur_kf)], cur_kf a window keyframe. For each
 * feature f with q = forced_mp[f] >= 0, q not bad, against the slot's occupant m:
 * m == q or m bad or m in LoopSet -> nothing; m == -1 -> ADD; else m is a victim
 * with survivor q. These tables are applied (as APPLY below) at the start of PLAN,
 * so the search sees the updated map. Re-running them on an already forced map
 * changes nothing (every shard's PLAN may carry them).
 *
 * phase LC_FUSE_PLAN  : [forced matches, then] steps up to the victim words, for
 *                       window positions [w_lo, w_hi) only (a keyframe shard);
 *                       every word of io_winner outside the shard and every word
 *                       of io_victim is LC_NONE or a proposal of this call
 *                       afterwards. Map unchanged (except the forced matches).
 * phase LC_FUSE_APPLY : apply from io_winner / io_victim (e.g. after an NCCL MIN
 *                       all-reduce of the shards' tables). w_lo / w_hi ignored.
 * phase LC_FUSE_ALL   : PLAN over the whole window, then APPLY.
 *   window_kf [host]; win_list_begin (nullable) [host|dev]; window_S (nullable) [host|dev];
 *   n_window >= 1. A DEVICE win_list_begin (e.g. lc_loop_lists' device offsets) is not
 *   read back: n_list is then the list buffer's capacity (>= win_list_begin[n_window]),
 *   mp_list must be device memory, every list must hold <= 261888 entries, and only a
 *   full-window PLAN / ALL without forced matches or dbg is accepted (LC_EINVAL
 *   otherwise); each window keyframe is then one block (its own CTA).
 *   distinct keyframes; mp_list [host|dev] n_list entries, each list ascending
 *   and unique (not checked on device; duplicates give duplicate queries).
 *   A host mp_list with per-keyframe lists (win_list_begin) on a full-range PLAN
 *   (>= 2^18 entries, no dbg, not capturing) is uploaded in 4 chunks on a private
 *   stream while the matching of the chunks already resident runs (same results;
 *   the buffer must stay unchanged until the call stream has passed the call).
 *   io_winner [host|dev] nullable (internal), [sum_i F(window_kf[i])] window-major,
 *     local feature order: the surviving winner word per window feature.
 *   io_victim [host|dev] nullable (internal), [n_mp].
 *   out_action [host|dev] nullable, [sum_i F(window_kf[i])]: 0 none, 1 add,
 *     2 victim proposal, 3 loop point in slot, 4 orientation-rejected, 5 bad slot.
 *   dbg [host] nullable; query index = win_list_begin[i] + j (CSR) or
 *     i * n_list + j (shared list) for the j-th entry of L_i.
 *   out_counts [host|dev] nullable, [LC_NCOUNT].
 * Errors: LC_ESTATE (no map, or window_S NULL and a window keyframe without a
 * stored correction), LC_EINVAL, LC_ERANGE (keyframe index), LC_ECAPACITY. */
lc_status lc_fuse(lc_ctx* ctx, int32_t phase, int32_t w_lo, int32_t w_hi, int32_t n_window,
                  const int32_t* window_kf, const lc_sim3* window_S,
                  const int32_t* win_list_begin, const int32_t* mp_list, int64_t n_list,
                  const lc_match_params* params, int32_t cur_kf, const int32_t* forced_mp,
                  int64_t* io_winner, int64_t* io_victim,
                  int8_t* out_action, const lc_query_debug* dbg, int64_t* out_counts,
                  void* cuda_stream);

/* ---------------------------------------------------------------------------
 * lc_loop_lists -- the loop map-point lists, built on the device from the resident map
 * (SURVEY.md §8(d) "Loop list = MPs of the matched pass-A KF and its top-10 covisibles,
 * ascending unique"; C5 "MPs of its 10 nearest pass-A KFs"; EXT LoopClosing
 * mvpLoopMapPoints; oracle orc_loop_lists). The paper assembles them on the CPU; here a
 * loop event uploads keyframe ids (C5: 110 KB) instead of map-point lists (35 MB).
 *
 * List l = the ascending unique map points (>= 0; bad ones included -- the queries skip
 * them, reading O4) associated with the keyframes src_kf[src_begin[l] .. src_begin[l+1]),
 * from the CURRENT associations (after any fuse / append). The result is the
 * (win_list_begin, mp_list) pair lc_fuse takes.
 *   src_begin [host] [n+1], src_kf [host]; out_begin [host|dev] [n+1] (written);
 *   out_list [host|dev] capacity entries.
 * Host out_begin: synchronises the stream (the offsets come back to the host). A list
 * may hold at most 24576 distinct map points.
 * Device out_begin (device offsets): nothing is read back and the call does not
 * synchronise; the offsets are a device scan of the lists' counts, so lc_fuse can take
 * (out_begin, out_list) as its (win_list_begin, mp_list) with no host round trip. Then
 * out_list must be device memory of capacity >= U = the sum over lists of their source
 * keyframes' feature counts (an upper bound of the total, known before the lists are
 * built), each list's bound must be <= 261888 and the map must hold <= 1835008 map points
 * (every list's id range fits one shared-memory bitmap); otherwise LC_ECAPACITY.
 * Errors: LC_ESTATE (no map), LC_EINVAL, LC_ERANGE (keyframe id), LC_ECAPACITY (total >
 * capacity -- out_begin is complete -- or a list over the limit). */
lc_status lc_loop_lists(lc_ctx* ctx, int32_t n, const int32_t* src_begin, const int32_t* src_kf,
                        int32_t* out_begin, int32_t* out_list, int64_t capacity, void* cuda_stream);

/* ---------------------------------------------------------------------------
 * lc_fuse_adds -- the sparse ADD exchange of a keyframe-sharded fusion (SURVEY.md §8(e):
 * "all_gather of ADD lists, as (global feature index, q) pairs"; the
 * window keyframes are independent, so each rank plans a shard).
 *
 * APPLY reads a winner word only where the slot is empty (an ADD); every other effect of
 * PLAN travels in the victim words. So after PLAN on window positions [w_lo, w_hi):
 *   op LC_ADDS_PACK  : compacts the winner words of that shard whose slot is empty into
 *                      (io_idx[i] = window-major feature index, io_word[i] = winner word),
 *                      i < *io_n (written; order unspecified). LC_ECAPACITY (nothing
 *                      written beyond capacity, *io_n = the required count) if too small.
 *   op LC_ADDS_UNPACK: io_winner[0 .. sum F(window)) <- LC_NONE, then io_winner[io_idx[i]]
 *                      = io_word[i] for i < *io_n (the all_gathered lists of every rank):
 *                      the dense table APPLY takes.
 * io_winner [host|dev] [sum_i F(window_kf[i])]; io_idx, io_word [host|dev] int64,
 * capacity entries; io_n [host]. window_kf [host] as in lc_fuse. PACK synchronises the
 * stream (it reads the count back).
 * Errors: LC_ESTATE (no map), LC_EINVAL, LC_ERANGE, LC_ECAPACITY. */
#define LC_ADDS_PACK 1
#define LC_ADDS_UNPACK 2
lc_status lc_fuse_adds(lc_ctx* ctx, int32_t op, int32_t n_window, const int32_t* window_kf, int32_t w_lo,
                       int32_t w_hi, int64_t* io_winner, int64_t* io_idx, int64_t* io_word, int64_t* io_n,
                       int64_t capacity, void* cuda_stream);

/* ---------------------------------------------------------------------------
 * lc_set_point_range / lc_mp_positions -- the map-point slices of a sharded correction
 * (SURVEY.md §8(e) "Correction": "ALL mode is sharded by MP index range, followed by
 * all_gather of corrected position slices"; WINDOW "point correction is sharded by MP
 * index range, followed by all_gather of the slices"; §III.B).
 *
 * lc_set_point_range: every later lc_correct_sim3 call (LC_CORRECT_WINDOW, LC_CORRECT_ALL;
 *   not LC_DRY_RUN) rewrites the positions of the map points in [mp_lo, mp_hi) only, and
 *   its CORR_MP counter counts those. Everything else it does stays replicated on every
 *   rank: keyframe poses, S^corr, the owner election and the per-point corr_ref record of
 *   which window keyframe re-anchored a point (so the ranks' stores stay identical once
 *   the position slices are exchanged). mp_hi < 0 restores "all points". Persists until
 *   changed; lc_upload_map resets it. Errors: LC_ESTATE (no map), LC_EINVAL
 *   (mp_lo < 0, mp_lo > mp_hi, mp_hi > number of map points).
 * lc_mp_positions: op LC_POS_GET copies the fp32 positions of map points [mp_lo, mp_hi)
 *   into xyz, op LC_POS_SET writes xyz into the store; xyz [host|dev] [(mp_hi - mp_lo) * 3]
 *   (x, y, z per point). Errors: LC_ESTATE, LC_EINVAL (op, range, null xyz with a
 *   non-empty range). */
lc_status lc_set_point_range(lc_ctx* ctx, int32_t mp_lo, int32_t mp_hi);
#define LC_POS_GET 1
#define LC_POS_SET 2
lc_status lc_mp_positions(lc_ctx* ctx, int32_t op, int32_t mp_lo, int32_t mp_hi, float* xyz, void* cuda_stream);

/* ---------------------------------------------------------------------------
 * lc_search_by_projection -- batched read-only projection search
 * (PAPER.md:200). Pair p = (keyframe pair_kf[p], transform
 * pair_S[p], parameter set params[pair_param[p]], list mp_list[pair_list_begin[p]
 * .. pair_list_begin[p+1])). Same projection/matching/conflict/orientation steps
 * as lc_fuse, except "already found" (reading A19): features whose entry in
 * pair_taken is >= 0 are not candidates and map points present in pair_taken are
 * skipped. No fusion; the map is not modified.
 *   pair_kf, pair_S, pair_param, params, pair_list_begin [host]; mp_list [host|dev].
 *   pair_taken [host|dev] nullable, pair-major [sum_p F(pair_kf[p])], -1 = free.
 *   out_feat_mp / out_feat_dist [host|dev] pair-major [sum_p F(pair_kf[p])]:
 *     taken entries are copied (dist -1); otherwise the winning map point and
 *     its H, or -1 / -1.
 *   dbg [host] nullable; query index = position in mp_list.
 *   out_counts [host|dev] nullable, [n_pairs][LC_NCOUNT].
 * Errors: LC_ESTATE (no map), LC_EINVAL (n_pairs < 0, n_params < 1, bad params,
 * pair_param out of range, null S), LC_ERANGE (keyframe index). */
lc_status lc_search_by_projection(lc_ctx* ctx, int32_t n_pairs, const int32_t* pair_kf,
                                  const lc_sim3* pair_S, const int32_t* pair_param,
                                  const lc_match_params* params, int32_t n_params,
                                  const int32_t* pair_list_begin, const int32_t* mp_list,
                                  const int32_t* pair_taken, int32_t* out_feat_mp,
                                  int32_t* out_feat_dist, const lc_query_debug* dbg,
                                  int64_t* out_counts, void* cuda_stream);

/* ---------------------------------------------------------------------------
 * lc_pgo_sim3 -- essential-graph Sim3 pose-graph optimisation (
 * PAPER.md:244-248 §IV.F "an essential (pose) graph optimization to propagate the
 * loop correction to the rest of the map", Jacobians by "automatic differentiation";
 * "Levenberg-Marquardt" (Conclusion); SPEC.md pose-graph; readings A49-A54).
 * Its output S_opt is what lc_correct_sim3(LC_CORRECT_ALL) propagates to the map.
 * Needs a context, not a map.
 *
 *   n_v vertices: S_init [host|dev] [n_v] world->camera Sim3 estimates; fixed [host]
 *     [n_v] (non-zero = held constant, e.g. the loop keyframe).
 *   n_e edges: edge_ij [host] [n_e][2] (i, j), i != j, both < n_v; M [host|dev] [n_e]
 *     the measurement, S_j o S_i^-1 when the edge was made. Residual
 *     e = log(M o S_i o S_j^-1) (7-vector (omega, upsilon, sigma), A49/A50), identity
 *     information; chi2 = sum_e |e|^2. Updates S <- exp(delta) o S.
 *   Levenberg-Marquardt (A52/A53): linearise (Jacobians by forward-mode dual numbers),
 *     solve (H + lambda diag(H)) delta = -b over the free vertices (A54) by a banded
 *     Cholesky factorisation in a reverse Cuthill-McKee order (a non-positive pivot is
 *     a failed solve -> lambda *= 4), or by block-Jacobi preconditioned conjugate
 *     gradients (stop when |r| <= cg_tol |b| or after cg_max_iter; a non-SPD diagonal
 *     block or p^T A p <= 0 is a failed solve); params->solver selects. |delta| < eps_dx stops; a trial exp(delta_v) o S_v is accepted iff
 *     chi2 decreases (lambda <- max(lambda / 2, 1e-12); stop when the relative
 *     decrease < eps_chi2), else lambda *= 4; lambda > 1e8 stops; max_iter solves.
 *   out_S [host|dev] [n_v] the optimised estimates (fixed vertices unchanged).
 *   out_trace [host|dev] nullable [max_iter][6] per iteration: chi2, lambda, trial
 *     chi2 (-1: solve failed; chi2 when the |delta| test stopped), accepted (0/1),
 *     |delta| (-1 if failed), solver iterations (CG iterations; 1 for the banded solve).
 *   out_chi2 [host|dev] nullable [2]: initial and final chi2.
 *   out_counts [host|dev] nullable [LC_NCOUNT] (PGO_ITERS, PGO_ACCEPTED,
 *     PGO_SOLVER_ITERS, PGO_STOP, PGO_BAND, PGO_CR_LEVELS).
 * The whole loop runs in one cooperative kernel (no host round trip per iteration);
 * results are deterministic for a given problem. Capturable (lc_graph_*): the edge
 * list, fixed flags and the host-built incidence / RCM order are constants of the graph.
 * Errors: LC_EINVAL (null pointers, sizes, params, i == j), LC_ERANGE (vertex index),
 * LC_ECUDA (cooperative launch failed).
 * ------------------------------------------------------------------------- */
typedef struct {
  int32_t max_iter;      /* Levenberg-Marquardt iterations (linear solves), >= 0 (ORB-SLAM3: 20) */
  int32_t cg_max_iter;   /* CG iterations per solve, >= 1                                */
  double lambda0;        /* initial damping, > 0 (SPEC: 1e-4)                            */
  double eps_dx;         /* stop when |delta| < eps_dx (1e-8)                            */
  double eps_chi2;       /* stop when an accepted step lowers chi2 by < eps_chi2 relative */
  double cg_tol;         /* CG relative residual target (1e-10)                          */
  int32_t solver;        /* LC_PGO_SOLVER_AUTO / _BAND / _CG / _CR                        */
  int32_t reserved;
} lc_pgo_params;

/* Linear solver of lc_pgo_sim3 (A54, A54b), all in the reverse Cuthill-McKee order of the
 * free vertices (block bandwidth bw). CR: block cyclic reduction -- the band cut into
 * super-blocks of max(bw, 1) positions is block tridiagonal; odd-even elimination over
 * log2(n_v / bw) levels, each level's eliminations and Schur updates spread over the SMs
 * (LC_EINVAL if bw > 18: a super-block must fit one CTA's shared memory). BAND: the
 * banded Cholesky chain in one CTA (LC_EINVAL if bw > 28). CG: block-Jacobi
 * preconditioned conjugate gradients. AUTO: CR when bw <= 18 and n_v >= 4 max(bw, 1),
 * else BAND when bw <= 28, else CG. CR and BAND are the same factorisation up to
 * rounding (the order of the eliminations differs). */
enum { LC_PGO_SOLVER_AUTO = 0, LC_PGO_SOLVER_BAND = 1, LC_PGO_SOLVER_CG = 2, LC_PGO_SOLVER_CR = 3 };

enum { LC_PGO_STOP_DX = 1, LC_PGO_STOP_CHI2 = 2, LC_PGO_STOP_MAX_ITER = 3, LC_PGO_STOP_LAMBDA = 4,
       LC_PGO_STOP_ZERO = 5 };

lc_status lc_pgo_sim3(lc_ctx* ctx, int32_t n_v, const lc_sim3* S_init, const uint8_t* fixed, int32_t n_e,
                      const int32_t* edge_ij, const lc_sim3* M, const lc_pgo_params* params,
                      lc_sim3* out_S, double* out_trace, double* out_chi2, int64_t* out_counts,
                      void* cuda_stream);

#ifdef __cplusplus
}
#endif
#endif /* LC_H_ */
