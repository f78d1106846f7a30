/*
 * lc_oracle.c -- plain, slow, obviously-correct CPU oracle for the loop-closing
 * fuse/correct hot path of arXiv 2603.17201 ("FastLoop").
 *
 * TEST INFRASTRUCTURE ONLY. Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library. The product path
 * (paper_2603_17201_b200/, csrc/) never links, imports or calls it, and this file
 * shares no code, header, table or constant generator with csrc/.
 *
 * What it computes (PAPER.md line + section; SURVEY.md §8(c) reading ids):
 *   - Loop-correction Sim3 pose correction of the window keyframes and the map
 *     points they observe ("correcting their poses using the estimated Sim3
 *     transformation", §III.B)                     -> orc_correct_window  (O3)
 *   - Loop fusion: project the loop map points into every window keyframe,
 *     match by descriptor "within close spatial proximity", and merge
 *     duplicates (§III.B; §IV.D.3)  -> orc_fuse        (O4-O9)
 *     including the forced loop matches of the current keyframe, fused first
 *     (O9.4, reading A23)
 *   - the same window correction as a batch of dry runs (no write-back), one per
 *     loop-candidate hypothesis (§IV.C: candidates in batches)
 *                                                               -> orc_correct_window_batch (O3')
 *   - the loop map-point lists (MPs of the matched keyframe's covisibles), built
 *     from the map (SURVEY.md §8(d) "Loop list")           -> orc_loop_lists
 *   - a thread-parallel, cell-grid version of the fuse PLAN for TIMING ONLY (the
 *     CPU baseline); it is tested equal to the brute-force definition
 *                                                               -> orc_fuse_plan_grid
 *   - Projection search PS1 / PS2a||PS2b / PS3a-c, one result batch per
 *     (keyframe, transform) pair (§IV.C; §IV.D.1-2)
 *                                                               -> orc_search_by_projection
 *   - Propagation of the optimised Sim3 of every keyframe to the whole map
 *     ("propagates the loop correction to the rest of the map")
 *                                                               -> orc_correct_all   (O10)
 *   - Map-point refresh after a merge: distinctive descriptor + normal and depth
 *     range ("merge duplicate map points"; the
 *     refresh itself is inherited ORB-SLAM3 behaviour, readings A33-A37)
 *                                                               -> orc_refresh       (O11)
 *   - Covisibility recount after the merge ("creates new connections in the
 *     covisibility and essential graphs"; SURVEY.md
 *     §8(f) f4, readings A38-A40)                               -> orc_update_connections (O12)
 *   - Region-detection Sim3 estimation: RANSAC over minimal 3-point samples,
 *     closed-form Horn similarity, symmetric reprojection inlier test ("estimating
 *     the relative pose between the new keyframe and the matched one", PAPER.md:89;
 *     SURVEY.md §8(f) f3, readings A41-A44)                     -> orc_sim3_ransac (O13)
 *   - its Gauss-Newton Sim3 refinement with a Huber kernel (SPEC.md refine_sim3;
 *     readings A45-A48)                                        -> orc_sim3_refine (O14)
 *   - Essential-graph Sim3 pose-graph optimisation: Levenberg-Marquardt with
 *     automatic-differentiation Jacobians and an LDLT linear solve ("we use
 *     automatic differentiation", "Eigen LDLT for the linear solver",
 *     PAPER.md:244-248 §IV.F, readings A49-A53)
 *                                                               -> orc_pgo (O15)
 * The paper gives no matching math (SURVEY.md §0 "Key finding"); every
 * constant and tie-break is a DESIGN.md reading (A1-A32), noted inline.
 *
 * Style: brute force, ascending loops, fp64 arithmetic evaluated in the order
 * written (compile with -O2 -ffp-contract=off, no -ffast-math), fp32 only for
 * stored values. No grid, no atomics, no reordering.
 *
 * Parity status: every function is pinned by tests/test_oracle_pins.py (O1-O14),
 * tests/test_oracle_pgo.py (O15: scipy expm/logm, central differences, the hand-derived
 * adjoint, closed forms, exact-truth recovery) and tests/test_oracle_pins_r2.py (O9.4
 * forced matches against an independent restatement of EXT Replace; O3' dry runs against
 * the O3 invariant and 4x4 products; the A15 bin mapping by a histogram that floor(),
 * 30-degree bins or a missing 30 -> 0 wrap each change; the edge flag at constructed
 * distances; grid PLAN == brute-force PLAN). The orientation rule itself (three maxima,
 * 0.1 ratio) remains "parity unpinned" against the paper, which prints nothing about it.
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define ORC_NONE INT64_MAX

/* counter slots (same meaning/order as DESIGN.md "Counters"; tests match by name) */
enum {
  C_QUERIES = 0, C_SKIP_BAD, C_SKIP_FOUND, C_CULL_DEPTH, C_CULL_BOUNDS, C_CULL_DIST,
  C_CULL_ANGLE, C_CANDIDATES, C_NO_CAND, C_OVER_TH, C_RATIO_REJ, C_PROPOSALS,
  C_WINNERS, C_ORIENT_REJ, C_ADD, C_VICTIM_PROP, C_LOOP_SKIP, C_BAD_SLOT,
  C_VICTIMS, C_REWIRED, C_DUP_CLEARED, C_ADDED, C_CORR_KF, C_CORR_MP,
  C_REFRESH_MP, C_REFRESH_OBS, C_CONN_KF, C_CONN_EDGES, C_RANSAC_HYP, C_RANSAC_INLIERS,
  C_REFINE_ITERS, C_REFINE_INLIERS, C_PGO_ITERS, C_PGO_ACCEPTED, C_PGO_SOLVER_ITERS,
  C_PGO_STOP, C_PGO_BAND, C_FORCED, C_EDGE_AMB, C_PGO_CR_LEVELS /* device solver only: always 0 */, C_N
};

/* query status codes written to out_status (negative = culled/skipped) */
enum { Q_MATCHED_STAGE = 0, Q_BAD = -1, Q_FOUND = -2, Q_DEPTH = -3, Q_BOUNDS = -4,
       Q_DIST = -5, Q_ANGLE = -6 };

typedef struct {
  int32_t model;            /* 0 pinhole, 1 Kannala-Brandt-8 */
  double fx, fy, cx, cy;
  double k[4];
  double min_x, max_x, min_y, max_y;
} orc_camera;

typedef struct {
  int32_t th, max_hamming, ratio_num, ratio_den, check_orientation;
} orc_params;

typedef struct {
  int32_t n_kf, n_feat, n_mp, n_levels;
  double scale_factor;
  double *kf_pose;          /* [n_kf][13] R row-major, t, s  (mutable: corrections) */
  const int32_t *kf_cam;
  const int32_t *kf_feat_begin;
  const float *feat_uv;     /* [n_feat][2] */
  const uint8_t *feat_octave;
  const float *feat_angle;
  const uint8_t *feat_desc; /* [n_feat][32] */
  int32_t *feat_mp;         /* mutable (fusion) */
  float *mp_pos;            /* [n_mp][3] mutable (corrections) */
  float *mp_normal;         /* [n_mp][3] mutable (refresh) */
  float *mp_max_dist;       /* mutable (refresh) */
  uint8_t *mp_desc;         /* [n_mp][32] mutable (refresh) */
  const float *mp_angle;
  const int32_t *mp_ref_kf;
  uint8_t *mp_flags;        /* bit0 = bad */
  int32_t *mp_replaced_by;  /* -1 = none */
  int32_t *mp_nobs;
  /* loop state created by orc_correct_window, consumed by orc_correct_all */
  int32_t *mp_corr_ref;     /* [n_mp] owner KF of this loop's correction, -1 = none */
  int32_t *kf_in_window;    /* [n_kf] 1 if corrected by the last window correction */
  double *kf_S_corr;        /* [n_kf][13] S_iw^corr (= S^pre for O10) */
  const orc_camera *cams;
  int32_t n_cams;
} orc_map;

/* ------------------------------------------------------------------------- */
/* O1  Hamming distance of two 256-bit descriptors: number of differing bits.  */
/* "descriptor similarity". Bit-by-bit count.      */
/* ------------------------------------------------------------------------- */
int orc_hamming(const uint8_t *a, const uint8_t *b) {
  int n = 0;
  for (int i = 0; i < 32; ++i) {
    unsigned x = (unsigned)(a[i] ^ b[i]);
    for (int bit = 0; bit < 8; ++bit) n += (x >> bit) & 1u;
  }
  return n;
}

/* ------------------------------------------------------------------------- */
/* O2  Sim3 algebra, S = (R, t, s), S(p) = s*(R p) + t  (reading A1).          */
/* Row products are evaluated ((a0*b0 + a1*b1) + a2*b2).                     */
/* ------------------------------------------------------------------------- */
static double row3(const double *r, const double *p) {
  return (r[0] * p[0] + r[1] * p[1]) + r[2] * p[2];
}
static double col3(const double *R, int i, const double *p) { /* (R^T p)_i */
  return (R[0 + i] * p[0] + R[3 + i] * p[1]) + R[6 + i] * p[2];
}

void orc_sim3_apply(const double *S, const double *p, double *out) {
  double q[3];
  for (int i = 0; i < 3; ++i) q[i] = row3(S + 3 * i, p);
  for (int i = 0; i < 3; ++i) out[i] = S[12] * q[i] + S[9 + i];
}

void orc_sim3_compose(const double *A, const double *B, double *out) {
  double o[13];
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j)
      o[3 * i + j] = (A[3 * i + 0] * B[0 + j] + A[3 * i + 1] * B[3 + j]) + A[3 * i + 2] * B[6 + j];
  for (int i = 0; i < 3; ++i) o[9 + i] = A[12] * row3(A + 3 * i, B + 9) + A[9 + i];
  o[12] = A[12] * B[12];
  memcpy(out, o, sizeof(o));
}

void orc_sim3_inverse(const double *S, double *out) {
  double o[13];
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) o[3 * i + j] = S[3 * j + i];
  for (int i = 0; i < 3; ++i) o[9 + i] = -col3(S, i, S + 9) / S[12];
  o[12] = 1.0 / S[12];
  memcpy(out, o, sizeof(o));
}

/* SE3 part of a Sim3: (R, t/s, 1)  (reading A2) */
void orc_sim3_se3(const double *S, double *out) {
  double o[13];
  memcpy(o, S, 9 * sizeof(double));
  for (int i = 0; i < 3; ++i) o[9 + i] = S[9 + i] / S[12];
  o[12] = 1.0;
  memcpy(out, o, sizeof(o));
}

/* scale table s_0 = 1, s_n = s_{n-1} * f (fp64) */
void orc_scale_table(int32_t L, double f, double *out) {
  out[0] = 1.0;
  for (int n = 1; n < L; ++n) out[n] = out[n - 1] * f;
}

/* ------------------------------------------------------------------------- */
/* Camera projection pi(p_c) (reading A29 for Kannala-Brandt-8).              */
/* ------------------------------------------------------------------------- */
void orc_project(const orc_camera *c, const double *pc, double *uv) {
  double x = pc[0], y = pc[1], z = pc[2];
  if (c->model == 0) {
    uv[0] = ((c->fx * x) / z) + c->cx;
    uv[1] = ((c->fy * y) / z) + c->cy;
    return;
  }
  double rho = sqrt((x * x) + (y * y));
  if (rho == 0.0) { uv[0] = c->cx; uv[1] = c->cy; return; }
  double th = atan2(rho, z);
  double t2 = th * th;
  double a = c->k[3];
  a = c->k[2] + t2 * a;
  a = c->k[1] + t2 * a;
  a = c->k[0] + t2 * a;
  a = 1.0 + t2 * a;
  double r = th * a;
  uv[0] = ((c->fx * r) * (x / rho)) + c->cx;
  uv[1] = ((c->fy * r) * (y / rho)) + c->cy;
}

/* predicted level (reading A7): smallest n with d*s_n >= dmax, else L-1 */
int orc_predict_level(double d, double dmax, const double *scale, int32_t L) {
  for (int n = 0; n < L; ++n)
    if (d * scale[n] >= dmax) return n;
  return L - 1;
}

/* ------------------------------------------------------------------------- */
/* O4-O6 one query: keyframe k seen through S_kw, map point q.               */
/* Returns status (0 = reached matching, <0 = cull code).                    */
/* ------------------------------------------------------------------------- */
typedef struct {
  int32_t status;
  double u, v;
  int32_t level;
  double radius;
  int32_t ncand;
  int32_t best_f;           /* KF-local original feature index, -1 = none */
  int32_t best_h, second_h; /* 256 when absent */
  int32_t edge;             /* 1 if a window/bounds decision is within 1e-4 px */
} orc_qres;

#define EDGE_EPS 1e-4

static int found_in_kf(const orc_map *m, int32_t k, int32_t q) {
  for (int32_t f = m->kf_feat_begin[k]; f < m->kf_feat_begin[k + 1]; ++f)
    if (m->feat_mp[f] == q) return 1;
  return 0;
}

static int found_in_taken(const int32_t *taken, int32_t nf, int32_t q) {
  for (int32_t f = 0; f < nf; ++f)
    if (taken[f] == q) return 1;
  return 0;
}

/* mode 0 = fuse (already found = associated in k), 1 = SBP (already found = in taken) */
static void query_one(const orc_map *m, int32_t k, const double *S_kw, int32_t q,
                      const orc_params *prm, const int32_t *taken, int mode,
                      const double *scale, orc_qres *r) {
  memset(r, 0, sizeof(*r));
  r->best_f = -1; r->best_h = 256; r->second_h = 256; r->level = -1;
  int32_t nf = m->kf_feat_begin[k + 1] - m->kf_feat_begin[k];
  if (m->mp_flags[q] & 1u) { r->status = Q_BAD; return; }
  if (mode == 0 ? found_in_kf(m, k, q) : (taken && found_in_taken(taken, nf, q))) {
    r->status = Q_FOUND; return;
  }
  double T[13], Ow[3], p[3], pc[3];
  orc_sim3_se3(S_kw, T);                                  /* A2 */
  for (int i = 0; i < 3; ++i) Ow[i] = -col3(T, i, T + 9);
  for (int i = 0; i < 3; ++i) p[i] = (double)m->mp_pos[3 * q + i];
  for (int i = 0; i < 3; ++i) pc[i] = row3(T + 3 * i, p) + T[9 + i];
  if (pc[2] <= 0.0) { r->status = Q_DEPTH; return; }      /* A3 */
  const orc_camera *cam = &m->cams[m->kf_cam[k]];
  double uv[2];
  orc_project(cam, pc, uv);
  r->u = uv[0]; r->v = uv[1];
  if (fabs(uv[0] - cam->min_x) < EDGE_EPS || fabs(uv[0] - cam->max_x) < EDGE_EPS ||
      fabs(uv[1] - cam->min_y) < EDGE_EPS || fabs(uv[1] - cam->max_y) < EDGE_EPS) r->edge = 1;
  if (!(uv[0] >= cam->min_x && uv[0] < cam->max_x && uv[1] >= cam->min_y && uv[1] < cam->max_y)) {
    r->status = Q_BOUNDS; return;                         /* A4 */
  }
  double PO[3];
  for (int i = 0; i < 3; ++i) PO[i] = p[i] - Ow[i];
  double d = sqrt((PO[0] * PO[0] + PO[1] * PO[1]) + PO[2] * PO[2]);
  double dmax = (double)m->mp_max_dist[q];
  double dmin_inv = 0.8 * (dmax / scale[m->n_levels - 1]);
  double dmax_inv = 1.2 * dmax;
  if (d < dmin_inv || d > dmax_inv) { r->status = Q_DIST; return; }  /* A5 */
  double n[3];
  for (int i = 0; i < 3; ++i) n[i] = (double)m->mp_normal[3 * q + i];
  if (row3(PO, n) < 0.5 * d) { r->status = Q_ANGLE; return; }        /* A6 */
  int lvl = orc_predict_level(d, dmax, scale, m->n_levels);          /* A7 */
  double rad = (double)prm->th * scale[lvl];                          /* A8, A11 */
  r->level = lvl; r->radius = rad;
  int32_t f0 = m->kf_feat_begin[k];
  const uint8_t *dq = m->mp_desc + 32 * (size_t)q;
  for (int32_t f = 0; f < nf; ++f) {                                  /* O5 brute force */
    if (taken && taken[f] >= 0) continue;                             /* A19 (SBP) */
    int oct = m->feat_octave[f0 + f];
    if (oct < lvl - 1 || oct > lvl) continue;                         /* A9 */
    double du = fabs((double)m->feat_uv[2 * (f0 + f)] - uv[0]);
    double dv = fabs((double)m->feat_uv[2 * (f0 + f) + 1] - uv[1]);
    if (du < rad + EDGE_EPS && dv < rad + EDGE_EPS &&
        (du > rad - EDGE_EPS || dv > rad - EDGE_EPS)) r->edge = 1;
    if (!(du < rad && dv < rad)) continue;
    r->ncand++;
    int h = orc_hamming(dq, m->feat_desc + 32 * (size_t)(f0 + f));
    if (h < r->best_h || (h == r->best_h && f < r->best_f)) {          /* O6, A12, A13 */
      if (r->best_f >= 0 && r->best_h < r->second_h) r->second_h = r->best_h;
      r->best_h = h; r->best_f = f;
    } else if (h < r->second_h) {
      r->second_h = h;
    }
  }
  r->status = Q_MATCHED_STAGE;
}

/* exposed for pin tests */
void orc_query(const orc_map *m, int32_t k, const double *S_kw, int32_t q,
               const orc_params *prm, const int32_t *taken, int32_t mode, orc_qres *r) {
  double scale[64];
  orc_scale_table(m->n_levels, m->scale_factor, scale);
  query_one(m, k, S_kw, q, prm, taken, mode, scale, r);
}

/* proposal test O6 (A10 threshold inclusive, A14 integer ratio) */
static int proposal_ok(const orc_qres *r, const orc_params *prm, int64_t *cnt) {
  if (r->ncand == 0) { cnt[C_NO_CAND]++; return 0; }
  if (r->best_h > prm->max_hamming) { cnt[C_OVER_TH]++; return 0; }
  if (prm->ratio_den > 0 &&
      (int64_t)prm->ratio_den * r->best_h > (int64_t)prm->ratio_num * r->second_h) {
    cnt[C_RATIO_REJ]++; return 0;
  }
  cnt[C_PROPOSALS]++;
  return 1;
}

/* O8 rotation-consistency filter over the winners of one keyframe (A15).
 * winners: [nf] packed (H<<32)|q or ORC_NONE; removes rejected ones. */
static void orientation_filter(const orc_map *m, int32_t k, int64_t *win, int32_t nf,
                               int64_t *cnt) {
  int hist[30];
  memset(hist, 0, sizeof(hist));
  int32_t f0 = m->kf_feat_begin[k];
  int *bin_of = (int *)malloc(sizeof(int) * (nf > 0 ? nf : 1));
  for (int32_t f = 0; f < nf; ++f) {
    bin_of[f] = -1;
    if (win[f] == ORC_NONE) continue;
    int32_t q = (int32_t)(win[f] & 0xffffffff);
    float rot = m->feat_angle[f0 + f] - m->mp_angle[q];
    if (rot < 0.0f) rot += 360.0f;
    long b = lroundf(rot * (30.0f / 360.0f));
    if (b == 30) b = 0;
    bin_of[f] = (int)b;
    hist[b]++;
  }
  int max1 = 0, max2 = 0, max3 = 0, ind1 = -1, ind2 = -1, ind3 = -1;
  for (int i = 0; i < 30; ++i) {                           /* ComputeThreeMaxima (EXT) */
    int s = hist[i];
    if (s > max1) { max3 = max2; max2 = max1; max1 = s; ind3 = ind2; ind2 = ind1; ind1 = i; }
    else if (s > max2) { max3 = max2; max2 = s; ind3 = ind2; ind2 = i; }
    else if (s > max3) { max3 = s; ind3 = i; }
  }
  if ((float)max2 < 0.1f * (float)max1) { ind2 = -1; ind3 = -1; }
  else if ((float)max3 < 0.1f * (float)max1) { ind3 = -1; }
  for (int32_t f = 0; f < nf; ++f) {
    if (win[f] == ORC_NONE) continue;
    int b = bin_of[f];
    if (b != ind1 && b != ind2 && b != ind3) { win[f] = ORC_NONE; cnt[C_ORIENT_REJ]++; }
  }
  free(bin_of);
}

/* ------------------------------------------------------------------------- */
/* O3 window correction (SPEC.md:391-399 gives the shape).       */
/* ------------------------------------------------------------------------- */
/* O3 steps 1-2: S_iw^corr of every window keyframe from the OLD poses, and the
 * owner (first window keyframe in list order observing it) of every non-bad map point. */
static void window_sim3_owner(const orc_map *m, int32_t cur_kf, const double *S_cw_corr, int32_t n_w,
                              const int32_t *window, double *Sc, int32_t *owner) {
  double Tc_inv[13];
  orc_sim3_inverse(m->kf_pose + 13 * (size_t)cur_kf, Tc_inv);
  for (int32_t i = 0; i < n_w; ++i) {
    int32_t k = window[i];
    if (k == cur_kf) { memcpy(Sc + 13 * i, S_cw_corr, 13 * sizeof(double)); continue; }
    double S_ic[13];
    orc_sim3_compose(m->kf_pose + 13 * (size_t)k, Tc_inv, S_ic);
    orc_sim3_compose(S_ic, S_cw_corr, Sc + 13 * i);
  }
  for (int32_t q = 0; q < m->n_mp; ++q) owner[q] = -1;
  for (int32_t i = 0; i < n_w; ++i) {
    int32_t k = window[i];
    for (int32_t f = m->kf_feat_begin[k]; f < m->kf_feat_begin[k + 1]; ++f) {
      int32_t q = m->feat_mp[f];
      if (q < 0 || (m->mp_flags[q] & 1u)) continue;
      if (owner[q] < 0) owner[q] = i;
    }
  }
}

/* O3 step 3: p <- fl32( inverse(S_owner^corr)( T_owner,w^old (p) ) ) */
static void window_point(const orc_map *m, const double *T_old, const double *S_corr, int32_t q, float *out) {
  double p[3], pc[3], pw[3], Sinv[13];
  for (int j = 0; j < 3; ++j) p[j] = (double)m->mp_pos[3 * q + j];
  orc_sim3_apply(T_old, p, pc);                                /* T_owner,w^old (p) */
  orc_sim3_inverse(S_corr, Sinv);
  orc_sim3_apply(Sinv, pc, pw);                                /* inverse(S^corr)(.) */
  for (int j = 0; j < 3; ++j) out[j] = (float)pw[j];
}

int orc_correct_window(orc_map *m, int32_t cur_kf, const double *S_cw_corr, int32_t n_w,
                       const int32_t *window, double *out_S_corr, int64_t *cnt) {
  if (n_w <= 0 || window[0] != cur_kf) return -1;
  for (int32_t i = 0; i < m->n_mp; ++i) m->mp_corr_ref[i] = -1;
  for (int32_t k = 0; k < m->n_kf; ++k) m->kf_in_window[k] = 0;
  double *Sc = (double *)malloc(sizeof(double) * 13 * (size_t)n_w);
  int32_t *owner = (int32_t *)malloc(sizeof(int32_t) * (size_t)(m->n_mp > 0 ? m->n_mp : 1));
  window_sim3_owner(m, cur_kf, S_cw_corr, n_w, window, Sc, owner);   /* 1, 2 */
  for (int32_t q = 0; q < m->n_mp; ++q) {                              /* 3, 4 */
    if (owner[q] < 0) continue;
    int32_t i = owner[q];
    int32_t k = window[i];
    window_point(m, m->kf_pose + 13 * (size_t)k, Sc + 13 * i, q, m->mp_pos + 3 * (size_t)q);
    m->mp_corr_ref[q] = k;
    cnt[C_CORR_MP]++;
  }
  /* 5. write back T_iw <- SE3(S_iw^corr); keep S^corr as S^pre for O10 */
  for (int32_t i = 0; i < n_w; ++i) {
    int32_t k = window[i];
    memcpy(m->kf_S_corr + 13 * (size_t)k, Sc + 13 * i, 13 * sizeof(double));
    m->kf_in_window[k] = 1;
    orc_sim3_se3(Sc + 13 * i, m->kf_pose + 13 * (size_t)k);
    if (out_S_corr) memcpy(out_S_corr + 13 * i, Sc + 13 * i, 13 * sizeof(double));
    cnt[C_CORR_KF]++;
  }
  free(owner);
  free(Sc);
  return 0;
}

/* O3' the window correction of several loop-candidate hypotheses as dry runs (SURVEY.md
 * §8(d) C4: "32 lc_correct_sim3 dry runs"; §IV.C processes loop candidates
 * in batches). Batch b = (cur_kf[b], S_cw_corr[b], window wbeg[b]..wbeg[b+1]) gets O3
 * steps 1-3 against the map as it is (nothing is written back, batches are independent):
 * out_S [sum window][13] = S_iw^corr; out_mp_begin [n_batch+1] = CSR of the corrected
 * points, out_mp_idx / out_mp_pos = the owned map points of the batch in ascending index
 * with their corrected positions. Returns -1 on bad arguments, -2 if the points do not
 * fit in `capacity` (out_mp_begin is still complete). */
int orc_correct_window_batch(const orc_map *m, int32_t n_batch, const int32_t *cur_kf,
                             const double *S_cw_corr, const int32_t *wbeg, const int32_t *window,
                             double *out_S, int32_t *out_mp_begin, int32_t *out_mp_idx,
                             float *out_mp_pos, int64_t capacity, int64_t *cnt) {
  if (n_batch < 0 || wbeg[0] != 0) return -1;
  for (int32_t b = 0; b < n_batch; ++b)
    if (wbeg[b + 1] <= wbeg[b] || window[wbeg[b]] != cur_kf[b]) return -1;
  int32_t *owner = (int32_t *)malloc(sizeof(int32_t) * (size_t)(m->n_mp > 0 ? m->n_mp : 1));
  /* pass 1: point counts */
  out_mp_begin[0] = 0;
  for (int32_t b = 0; b < n_batch; ++b) {
    const int32_t n_w = wbeg[b + 1] - wbeg[b];
    double *Sc = out_S + 13 * (size_t)wbeg[b];
    window_sim3_owner(m, cur_kf[b], S_cw_corr + 13 * (size_t)b, n_w, window + wbeg[b], Sc, owner);
    int32_t n = 0;
    for (int32_t q = 0; q < m->n_mp; ++q) n += owner[q] >= 0;
    out_mp_begin[b + 1] = out_mp_begin[b] + n;
  }
  if ((int64_t)out_mp_begin[n_batch] > capacity) { free(owner); return -2; }
  /* pass 2: the corrected points */
  for (int32_t b = 0; b < n_batch; ++b) {
    const int32_t n_w = wbeg[b + 1] - wbeg[b];
    const int32_t *win = window + wbeg[b];
    const double *Sc = out_S + 13 * (size_t)wbeg[b];
    window_sim3_owner(m, cur_kf[b], S_cw_corr + 13 * (size_t)b, n_w, win, out_S + 13 * (size_t)wbeg[b], owner);
    int32_t o = out_mp_begin[b];
    for (int32_t q = 0; q < m->n_mp; ++q) {
      if (owner[q] < 0) continue;
      const int32_t i = owner[q];
      out_mp_idx[o] = q;
      window_point(m, m->kf_pose + 13 * (size_t)win[i], Sc + 13 * i, q, out_mp_pos + 3 * (size_t)o);
      ++o;
      cnt[C_CORR_MP]++;
    }
    cnt[C_CORR_KF] += n_w;
  }
  free(owner);
  return 0;
}

/* ------------------------------------------------------------------------- */
/* O10 propagation of the optimised Sim3 of every keyframe.    */
/* ------------------------------------------------------------------------- */
int orc_correct_all(orc_map *m, const double *S_opt, int64_t *cnt) {
  double *Spre = (double *)malloc(sizeof(double) * 13 * (size_t)m->n_kf);
  for (int32_t k = 0; k < m->n_kf; ++k)
    memcpy(Spre + 13 * k, m->kf_in_window[k] ? m->kf_S_corr + 13 * (size_t)k
                                             : m->kf_pose + 13 * (size_t)k, 13 * sizeof(double));
  for (int32_t q = 0; q < m->n_mp; ++q) {
    if (m->mp_flags[q] & 1u) continue;
    int32_t r = m->mp_corr_ref[q] >= 0 ? m->mp_corr_ref[q] : m->mp_ref_kf[q];   /* A26 */
    double p[3], pc[3], pw[3], Sinv[13];
    for (int j = 0; j < 3; ++j) p[j] = (double)m->mp_pos[3 * q + j];
    orc_sim3_apply(Spre + 13 * (size_t)r, p, pc);
    orc_sim3_inverse(S_opt + 13 * (size_t)r, Sinv);
    orc_sim3_apply(Sinv, pc, pw);
    for (int j = 0; j < 3; ++j) m->mp_pos[3 * q + j] = (float)pw[j];
    cnt[C_CORR_MP]++;
  }
  for (int32_t k = 0; k < m->n_kf; ++k) {
    orc_sim3_se3(S_opt + 13 * (size_t)k, m->kf_pose + 13 * (size_t)k);
    cnt[C_CORR_KF]++;
  }
  for (int32_t q = 0; q < m->n_mp; ++q) m->mp_corr_ref[q] = -1;   /* loop state consumed */
  for (int32_t k = 0; k < m->n_kf; ++k) m->kf_in_window[k] = 0;
  free(Spre);
  return 0;
}

/* ------------------------------------------------------------------------- */
/* O4-O9 loop fusion.                        */
/*  phase 1 = PLAN over window positions [w_lo, w_hi) (winner + victim words)  */
/*  phase 2 = APPLY from the (merged) winner/victim tables                    */
/*  phase 3 = both, over the whole window                                     */
/* ------------------------------------------------------------------------- */
static void list_of(int32_t i, const int32_t *wb, const int32_t *mp_list, int32_t n_list,
                    const int32_t **lst, int32_t *n) {
  if (wb) { *lst = mp_list + wb[i]; *n = wb[i + 1] - wb[i]; }
  else { *lst = mp_list; *n = n_list; }
}

/* O9.3 apply of a winner table (window-major, woff) and a victim table to the map:
 * (i) every association of a victim -> its survivor (priority 2); (ii) ADDs on empty
 * window slots (priority 1); (iii) per keyframe, a map point in > 1 slot keeps the
 * least (priority, f); (iv) victims flagged bad with replaced_by; (v) n_obs recount. */
static void apply_tables(orc_map *m, int32_t n_w, const int32_t *window, const int64_t *woff,
                         const int64_t *io_winner, const int64_t *io_victim, int64_t *cnt) {
  int32_t *win_pos = (int32_t *)malloc(sizeof(int32_t) * (size_t)(m->n_kf > 0 ? m->n_kf : 1));
  for (int32_t k = 0; k < m->n_kf; ++k) win_pos[k] = -1;
  for (int32_t i = 0; i < n_w; ++i) win_pos[window[i]] = i;
  for (int32_t q = 0; q < m->n_mp; ++q) if (io_victim[q] != ORC_NONE) cnt[C_VICTIMS]++;
  for (int32_t k = 0; k < m->n_kf; ++k) {
    int32_t f0 = m->kf_feat_begin[k], nf = m->kf_feat_begin[k + 1] - f0;
    int32_t *nv = (int32_t *)malloc(sizeof(int32_t) * (size_t)(nf > 0 ? nf : 1));
    int *prio = (int *)malloc(sizeof(int) * (size_t)(nf > 0 ? nf : 1));
    for (int32_t f = 0; f < nf; ++f) {
      int32_t s = m->feat_mp[f0 + f];
      nv[f] = s; prio[f] = 0;
      if (s >= 0 && io_victim[s] != ORC_NONE) {
        nv[f] = (int32_t)(io_victim[s] & 0xffffffff); prio[f] = 2; cnt[C_REWIRED]++;
      } else if (s < 0 && win_pos[k] >= 0 && io_winner[woff[win_pos[k]] + f] != ORC_NONE) {
        nv[f] = (int32_t)(io_winner[woff[win_pos[k]] + f] & 0xffffffff); prio[f] = 1;
      }
    }
    /* (iii) keep the least (priority, f) slot of every MP occupying > 1 slot (A22) */
    uint8_t *clear = (uint8_t *)calloc((size_t)(nf > 0 ? nf : 1), 1);
    for (int32_t f = 0; f < nf; ++f) {
      if (nv[f] < 0) continue;
      for (int32_t g = 0; g < nf; ++g)
        if (g != f && nv[g] == nv[f] && (prio[g] < prio[f] || (prio[g] == prio[f] && g < f)))
          clear[f] = 1;
    }
    for (int32_t f = 0; f < nf; ++f) {
      if (clear[f]) { nv[f] = -1; cnt[C_DUP_CLEARED]++; }
      else if (prio[f] == 1) cnt[C_ADDED]++;
      m->feat_mp[f0 + f] = nv[f];
    }
    free(clear);
    free(nv); free(prio);
  }
  for (int32_t q = 0; q < m->n_mp; ++q) {                             /* (iv) */
    if (io_victim[q] == ORC_NONE) continue;
    m->mp_flags[q] |= 1u;
    m->mp_replaced_by[q] = (int32_t)(io_victim[q] & 0xffffffff);
  }
  for (int32_t q = 0; q < m->n_mp; ++q) m->mp_nobs[q] = 0;             /* (v) recount */
  for (int32_t f = 0; f < m->n_feat; ++f)
    if (m->feat_mp[f] >= 0) m->mp_nobs[m->feat_mp[f]]++;
  free(win_pos);
}

/* O9.4 forced loop matches of the current keyframe (reading A23; EXT CorrectLoop fuses
 * mvpLoopMatchedMPs -- the loop map points matched to the current keyframe's features
 * during detection -- before SearchAndFuse). forced_mp [F(cur_kf)]: -1 or a map point
 * for feature f. With the same rules as O9.1, against the slot's occupant m:
 *   q bad or m == q -> nothing; m == -1 -> ADD(cur_kf, f, q); m bad -> nothing;
 *   m in LoopSet -> nothing (loop-victim-skipped, keeps the result chain-free);
 *   else m is a victim with survivor q (key (0, q): m sits in one slot of cur_kf).
 * The tables are applied (O9.3) before the search, which sees the updated map. */
static void forced_step(orc_map *m, int32_t cur_kf, const int32_t *forced_mp, int32_t n_w,
                        const int32_t *window, const int64_t *woff, const uint8_t *loopset, int64_t *cnt) {
  int32_t pos = -1;
  for (int32_t i = 0; i < n_w; ++i) if (window[i] == cur_kf) pos = i;
  int64_t *win = (int64_t *)malloc(sizeof(int64_t) * (size_t)(woff[n_w] > 0 ? woff[n_w] : 1));
  int64_t *vic = (int64_t *)malloc(sizeof(int64_t) * (size_t)(m->n_mp > 0 ? m->n_mp : 1));
  for (int64_t j = 0; j < woff[n_w]; ++j) win[j] = ORC_NONE;
  for (int32_t q = 0; q < m->n_mp; ++q) vic[q] = ORC_NONE;
  int32_t f0 = m->kf_feat_begin[cur_kf], nf = m->kf_feat_begin[cur_kf + 1] - f0;
  for (int32_t f = 0; f < nf; ++f) {
    int32_t q = forced_mp[f];
    if (q < 0 || (m->mp_flags[q] & 1u)) continue;
    int32_t slot = m->feat_mp[f0 + f];
    if (slot == q) continue;
    if (slot < 0) { win[woff[pos] + f] = (int64_t)q; cnt[C_FORCED]++; }
    else if (m->mp_flags[slot] & 1u) continue;
    else if (loopset[slot]) continue;
    else { vic[slot] = (int64_t)q; cnt[C_FORCED]++; }
  }
  apply_tables(m, n_w, window, woff, win, vic, cnt);
  free(win);
  free(vic);
}

int orc_fuse(orc_map *m, int32_t phase, int32_t w_lo, int32_t w_hi, int32_t n_w,
             const int32_t *window, const double *window_S, const int32_t *win_list_begin,
             const int32_t *mp_list, int32_t n_list, const orc_params *prm,
             int32_t cur_kf, const int32_t *forced_mp,
             int64_t *io_winner, int64_t *io_victim, int8_t *out_action,
             int32_t *out_status, int64_t *out_best, double *out_uv, int32_t *out_ncand,
             uint8_t *out_edge, int64_t *cnt) {
  if (n_w <= 0 || w_lo < 0 || w_hi > n_w || w_lo > w_hi) return -1;
  if (forced_mp) {
    int in = 0;
    for (int32_t i = 0; i < n_w; ++i) in |= window[i] == cur_kf;
    if (!in) return -1;
  }
  double scale[64];
  orc_scale_table(m->n_levels, m->scale_factor, scale);
  int64_t *woff = (int64_t *)malloc(sizeof(int64_t) * (size_t)(n_w + 1));
  woff[0] = 0;
  for (int32_t i = 0; i < n_w; ++i)
    woff[i + 1] = woff[i] + (m->kf_feat_begin[window[i] + 1] - m->kf_feat_begin[window[i]]);
  int64_t *qoff = (int64_t *)malloc(sizeof(int64_t) * (size_t)(n_w + 1));
  qoff[0] = 0;
  for (int32_t i = 0; i < n_w; ++i) {
    const int32_t *l; int32_t n;
    list_of(i, win_list_begin, mp_list, n_list, &l, &n);
    qoff[i + 1] = qoff[i] + n;
  }

  if (phase & 1) {
    /* LoopSet = union of all window KFs' loop lists (A21) */
    uint8_t *loopset = (uint8_t *)calloc((size_t)(m->n_mp > 0 ? m->n_mp : 1), 1);
    for (int32_t i = 0; i < n_w; ++i) {
      const int32_t *l; int32_t n;
      list_of(i, win_list_begin, mp_list, n_list, &l, &n);
      for (int32_t j = 0; j < n; ++j) loopset[l[j]] = 1;
    }
    if (forced_mp) forced_step(m, cur_kf, forced_mp, n_w, window, woff, loopset, cnt);   /* O9.4 */
    for (int64_t j = 0; j < woff[n_w]; ++j) io_winner[j] = ORC_NONE;
    for (int32_t q = 0; q < m->n_mp; ++q) io_victim[q] = ORC_NONE;
    for (int32_t i = w_lo; i < w_hi; ++i) {
      int32_t k = window[i];
      const double *S = window_S ? window_S + 13 * (size_t)i : m->kf_S_corr + 13 * (size_t)k;
      int32_t nf = m->kf_feat_begin[k + 1] - m->kf_feat_begin[k];
      int32_t f0 = m->kf_feat_begin[k];
      int64_t *win = io_winner + woff[i];
      const int32_t *l; int32_t n;
      list_of(i, win_list_begin, mp_list, n_list, &l, &n);
      for (int32_t j = 0; j < n; ++j) {
        int32_t q = l[j];
        orc_qres r;
        cnt[C_QUERIES]++;
        query_one(m, k, S, q, prm, NULL, 0, scale, &r);
        int64_t qi = qoff[i] + j;
        if (r.edge) cnt[C_EDGE_AMB]++;
        if (out_status) out_status[qi] = r.status;
        if (out_uv) { out_uv[2 * qi] = r.u; out_uv[2 * qi + 1] = r.v; }
        if (out_ncand) out_ncand[qi] = r.ncand;
        if (out_edge) out_edge[qi] = (uint8_t)r.edge;
        if (out_best) out_best[qi] = r.status < 0 ? (int64_t)r.status
            : (((int64_t)r.best_h << 48) | ((int64_t)r.second_h << 32) | (uint32_t)r.best_f);
        switch (r.status) {
          case Q_BAD: cnt[C_SKIP_BAD]++; continue;
          case Q_FOUND: cnt[C_SKIP_FOUND]++; continue;
          case Q_DEPTH: cnt[C_CULL_DEPTH]++; continue;
          case Q_BOUNDS: cnt[C_CULL_BOUNDS]++; continue;
          case Q_DIST: cnt[C_CULL_DIST]++; continue;
          case Q_ANGLE: cnt[C_CULL_ANGLE]++; continue;
          default: break;
        }
        cnt[C_CANDIDATES] += r.ncand;
        if (!proposal_ok(&r, prm, cnt)) continue;
        int64_t key = ((int64_t)r.best_h << 32) | (int64_t)q;          /* O7, A17 */
        if (key < win[r.best_f]) win[r.best_f] = key;
      }
      for (int32_t f = 0; f < nf; ++f) if (win[f] != ORC_NONE) cnt[C_WINNERS]++;
      if (out_action) for (int32_t f = 0; f < nf; ++f) out_action[woff[i] + f] = 0;
      if (prm->check_orientation) {
        int64_t *before = (int64_t *)malloc(sizeof(int64_t) * (size_t)(nf > 0 ? nf : 1));
        memcpy(before, win, sizeof(int64_t) * (size_t)nf);
        orientation_filter(m, k, win, nf, cnt);
        if (out_action)
          for (int32_t f = 0; f < nf; ++f)
            if (before[f] != ORC_NONE && win[f] == ORC_NONE) out_action[woff[i] + f] = 4;
        free(before);
      }
      for (int32_t f = 0; f < nf; ++f) {                                /* O9.1 actions */
        if (win[f] == ORC_NONE) continue;
        int32_t slot = m->feat_mp[f0 + f];
        int8_t act;
        if (slot < 0) { act = 1; cnt[C_ADD]++; }
        else if (m->mp_flags[slot] & 1u) { act = 5; cnt[C_BAD_SLOT]++; }
        else if (loopset[slot]) { act = 3; cnt[C_LOOP_SKIP]++; }
        else {
          act = 2; cnt[C_VICTIM_PROP]++;
          if (win[f] < io_victim[slot]) io_victim[slot] = win[f];      /* A20, A21 */
        }
        if (out_action) out_action[woff[i] + f] = act;
      }
    }
    free(loopset);
  }

  if (phase & 2) apply_tables(m, n_w, window, woff, io_winner, io_victim, cnt);   /* O9.3 */
  free(woff);
  free(qoff);
  return 0;
}

/* ------------------------------------------------------------------------- */
/* Loop map-point lists ("Loop list = MPs of the matched pass-A KF */
/* and its top-10 covisibles, ascending unique"; C5 "each has its own list: MPs of   */
/* its 10 nearest pass-A KFs"; EXT LoopClosing: mvpLoopMapPoints = the map points of */
/* the matched keyframe and its covisibles). List l = the ascending unique map points */
/* (>= 0, bad ones included: the queries skip them, O4) held by the keyframes         */
/* src_kf[src_begin[l] .. src_begin[l+1]). out_begin [n+1]; out_list >= the total.    */
/* Returns the total, or -1 on bad arguments.                                         */
/* ------------------------------------------------------------------------- */
static int cmp_i32_asc(const void *a, const void *b) {
  int32_t x = *(const int32_t *)a, y = *(const int32_t *)b;
  return (x > y) - (x < y);
}

int64_t orc_loop_lists(const orc_map *m, int32_t n, const int32_t *src_begin, const int32_t *src_kf,
                       int32_t *out_begin, int32_t *out_list, int64_t capacity) {
  if (n < 0 || (n > 0 && src_begin[0] != 0)) return -1;
  int64_t total = 0;
  out_begin[0] = 0;
  for (int32_t l = 0; l < n; ++l) {
    int64_t cnt = 0;
    for (int32_t j = src_begin[l]; j < src_begin[l + 1]; ++j) {
      int32_t k = src_kf[j];
      if (k < 0 || k >= m->n_kf) return -1;
      cnt += m->kf_feat_begin[k + 1] - m->kf_feat_begin[k];
    }
    int32_t *tmp = (int32_t *)malloc(sizeof(int32_t) * (size_t)(cnt > 0 ? cnt : 1));
    int64_t t = 0;
    for (int32_t j = src_begin[l]; j < src_begin[l + 1]; ++j)
      for (int32_t f = m->kf_feat_begin[src_kf[j]]; f < m->kf_feat_begin[src_kf[j] + 1]; ++f)
        if (m->feat_mp[f] >= 0) tmp[t++] = m->feat_mp[f];
    qsort(tmp, (size_t)t, sizeof(int32_t), cmp_i32_asc);
    int64_t u = 0;
    for (int64_t i = 0; i < t; ++i)
      if (i == 0 || tmp[i] != tmp[i - 1]) {
        if (total + u < capacity) out_list[total + u] = tmp[i];
        ++u;
      }
    free(tmp);
    total += u;
    out_begin[l + 1] = (int32_t)total;
  }
  return total;
}

/* ------------------------------------------------------------------------- */
/* TIMING ONLY: orc_fuse_plan_grid, the fuse PLAN (O4-O8 + the O9.1 victim        */
/* proposals) with an ORB-SLAM-style cell grid (EXT GetFeaturesInArea) and the     */
/* window keyframes spread over POSIX threads. It is the CPU baseline bench.py     */
/* reports ("Grid mode is the timed baseline ... at T = all host  */
/* cores"); it is NOT the parity definition (orc_fuse is) and tests check that its */
/* tables and counters equal orc_fuse's. Cell ranges are supersets of the window   */
/* (floor of monotone fp64 cell coordinates), the per-candidate test is O5's.      */
/* ------------------------------------------------------------------------- */
typedef struct {
  int32_t cols, rows;
  int32_t *cell_beg;   /* [n_kf][cols*rows + 1] offsets into cell_f (per keyframe, local) */
  int32_t *cell_f;     /* [n_feat] keyframe-local feature indices, by (cell, f) */
} orc_grid;

static int grid_cell(double x, double lo, double hi, int32_t n) {
  int c = (int)floor((x - lo) * ((double)n / (hi - lo)));
  return c < 0 ? 0 : (c >= n ? n - 1 : c);
}

orc_grid *orc_grid_build(const orc_map *m, int32_t cols, int32_t rows) {
  orc_grid *g = (orc_grid *)calloc(1, sizeof(orc_grid));
  const int32_t G = cols * rows;
  g->cols = cols; g->rows = rows;
  g->cell_beg = (int32_t *)malloc(sizeof(int32_t) * ((size_t)m->n_kf * (G + 1) + 1));
  g->cell_f = (int32_t *)malloc(sizeof(int32_t) * (size_t)(m->n_feat > 0 ? m->n_feat : 1));
  int32_t *cell = (int32_t *)malloc(sizeof(int32_t) * (size_t)(m->n_feat > 0 ? m->n_feat : 1));
  for (int32_t k = 0; k < m->n_kf; ++k) {
    const orc_camera *cam = &m->cams[m->kf_cam[k]];
    int32_t f0 = m->kf_feat_begin[k], nf = m->kf_feat_begin[k + 1] - f0;
    int32_t *beg = g->cell_beg + (size_t)k * (G + 1);
    for (int c = 0; c <= G; ++c) beg[c] = 0;
    for (int32_t f = 0; f < nf; ++f) {
      int cx = grid_cell((double)m->feat_uv[2 * (f0 + f)], cam->min_x, cam->max_x, cols);
      int cy = grid_cell((double)m->feat_uv[2 * (f0 + f) + 1], cam->min_y, cam->max_y, rows);
      cell[f0 + f] = cy * cols + cx;
      beg[cell[f0 + f] + 1]++;
    }
    for (int c = 0; c < G; ++c) beg[c + 1] += beg[c];
    int32_t *cur = (int32_t *)malloc(sizeof(int32_t) * (size_t)(G + 1));
    memcpy(cur, beg, sizeof(int32_t) * (size_t)(G + 1));
    for (int32_t f = 0; f < nf; ++f) g->cell_f[f0 + cur[cell[f0 + f]]++] = f;
    free(cur);
  }
  free(cell);
  return g;
}

void orc_grid_free(orc_grid *g) {
  if (!g) return;
  free(g->cell_beg);
  free(g->cell_f);
  free(g);
}

typedef struct { int32_t m; int64_t key; } orc_vprop;

typedef struct {
  orc_map *m;
  const orc_grid *g;
  int32_t n_w;
  const int32_t *window;
  const double *window_S;
  const int32_t *win_list_begin, *mp_list;
  int32_t n_list;
  const orc_params *prm;
  const int64_t *woff;
  const uint8_t *loopset;
  int64_t *io_winner;
  const double *scale;
  int32_t next;                 /* next window position (shared work counter) */
  pthread_mutex_t mu;
} grid_job;

typedef struct {
  grid_job *job;
  int64_t cnt[C_N];
  orc_vprop *vp;
  int64_t nvp, cap;
} grid_worker;

static int cmp_i32(const void *a, const void *b) {
  int32_t x = *(const int32_t *)a, y = *(const int32_t *)b;
  return (x > y) - (x < y);
}

static void grid_query(const orc_map *m, const orc_grid *g, int32_t k, const double *T, const double *Ow,
                       const int32_t *held, int32_t n_held, int32_t q, const orc_params *prm,
                       const double *scale, orc_qres *r) {
  memset(r, 0, sizeof(*r));
  r->best_f = -1; r->best_h = 256; r->second_h = 256; r->level = -1;
  if (m->mp_flags[q] & 1u) { r->status = Q_BAD; return; }
  if (n_held && bsearch(&q, held, (size_t)n_held, sizeof(int32_t), cmp_i32)) { r->status = Q_FOUND; return; }
  double p[3], pc[3];
  for (int i = 0; i < 3; ++i) p[i] = (double)m->mp_pos[3 * q + i];
  for (int i = 0; i < 3; ++i) pc[i] = row3(T + 3 * i, p) + T[9 + i];
  if (pc[2] <= 0.0) { r->status = Q_DEPTH; return; }
  const orc_camera *cam = &m->cams[m->kf_cam[k]];
  double uv[2];
  orc_project(cam, pc, uv);
  if (!(uv[0] >= cam->min_x && uv[0] < cam->max_x && uv[1] >= cam->min_y && uv[1] < cam->max_y)) {
    r->status = Q_BOUNDS; return;
  }
  double PO[3];
  for (int i = 0; i < 3; ++i) PO[i] = p[i] - Ow[i];
  double d = sqrt((PO[0] * PO[0] + PO[1] * PO[1]) + PO[2] * PO[2]);
  double dmax = (double)m->mp_max_dist[q];
  if (d < 0.8 * (dmax / scale[m->n_levels - 1]) || d > 1.2 * dmax) { r->status = Q_DIST; return; }
  double n[3];
  for (int i = 0; i < 3; ++i) n[i] = (double)m->mp_normal[3 * q + i];
  if (row3(PO, n) < 0.5 * d) { r->status = Q_ANGLE; return; }
  int lvl = orc_predict_level(d, dmax, scale, m->n_levels);
  double rad = (double)prm->th * scale[lvl];
  int32_t f0 = m->kf_feat_begin[k];
  const uint8_t *dq = m->mp_desc + 32 * (size_t)q;
  const int32_t G = g->cols * g->rows;
  const int32_t *beg = g->cell_beg + (size_t)k * (G + 1);
  int cx0 = grid_cell(uv[0] - rad, cam->min_x, cam->max_x, g->cols);
  int cx1 = grid_cell(uv[0] + rad, cam->min_x, cam->max_x, g->cols);
  int cy0 = grid_cell(uv[1] - rad, cam->min_y, cam->max_y, g->rows);
  int cy1 = grid_cell(uv[1] + rad, cam->min_y, cam->max_y, g->rows);
  for (int cy = cy0; cy <= cy1; ++cy)
    for (int cx = cx0; cx <= cx1; ++cx)
      for (int32_t j = beg[cy * g->cols + cx]; j < beg[cy * g->cols + cx + 1]; ++j) {
        int32_t f = g->cell_f[f0 + j];
        int oct = m->feat_octave[f0 + f];
        if (oct < lvl - 1 || oct > lvl) continue;
        double du = fabs((double)m->feat_uv[2 * (f0 + f)] - uv[0]);
        double dv = fabs((double)m->feat_uv[2 * (f0 + f) + 1] - uv[1]);
        if (!(du < rad && dv < rad)) continue;
        r->ncand++;
        int h = orc_hamming(dq, m->feat_desc + 32 * (size_t)(f0 + f));
        if (h < r->best_h || (h == r->best_h && f < r->best_f)) {
          if (r->best_f >= 0 && r->best_h < r->second_h) r->second_h = r->best_h;
          r->best_h = h; r->best_f = f;
        } else if (h < r->second_h) {
          r->second_h = h;
        }
      }
  r->status = Q_MATCHED_STAGE;
}

static void *grid_worker_main(void *arg) {
  grid_worker *wk = (grid_worker *)arg;
  grid_job *jb = wk->job;
  orc_map *m = jb->m;
  int32_t *held = NULL;
  int32_t held_cap = 0;
  for (;;) {
    pthread_mutex_lock(&jb->mu);
    int32_t i = jb->next++;
    pthread_mutex_unlock(&jb->mu);
    if (i >= jb->n_w) break;
    int32_t k = jb->window[i];
    const double *S = jb->window_S ? jb->window_S + 13 * (size_t)i : m->kf_S_corr + 13 * (size_t)k;
    double T[13], Ow[3];
    orc_sim3_se3(S, T);
    for (int j = 0; j < 3; ++j) Ow[j] = -col3(T, j, T + 9);
    int32_t f0 = m->kf_feat_begin[k], nf = m->kf_feat_begin[k + 1] - f0;
    if (nf > held_cap) { held_cap = nf; held = (int32_t *)realloc(held, sizeof(int32_t) * (size_t)held_cap); }
    int32_t n_held = 0;
    for (int32_t f = 0; f < nf; ++f) if (m->feat_mp[f0 + f] >= 0) held[n_held++] = m->feat_mp[f0 + f];
    qsort(held, (size_t)n_held, sizeof(int32_t), cmp_i32);
    int64_t *win = jb->io_winner + jb->woff[i];
    const int32_t *l; int32_t n;
    list_of(i, jb->win_list_begin, jb->mp_list, jb->n_list, &l, &n);
    int64_t *cnt = wk->cnt;
    for (int32_t j = 0; j < n; ++j) {
      int32_t q = l[j];
      orc_qres r;
      cnt[C_QUERIES]++;
      grid_query(m, jb->g, k, T, Ow, held, n_held, q, jb->prm, jb->scale, &r);
      switch (r.status) {
        case Q_BAD: cnt[C_SKIP_BAD]++; continue;
        case Q_FOUND: cnt[C_SKIP_FOUND]++; continue;
        case Q_DEPTH: cnt[C_CULL_DEPTH]++; continue;
        case Q_BOUNDS: cnt[C_CULL_BOUNDS]++; continue;
        case Q_DIST: cnt[C_CULL_DIST]++; continue;
        case Q_ANGLE: cnt[C_CULL_ANGLE]++; continue;
        default: break;
      }
      cnt[C_CANDIDATES] += r.ncand;
      if (!proposal_ok(&r, jb->prm, cnt)) continue;
      int64_t key = ((int64_t)r.best_h << 32) | (int64_t)q;
      if (key < win[r.best_f]) win[r.best_f] = key;
    }
    for (int32_t f = 0; f < nf; ++f) if (win[f] != ORC_NONE) cnt[C_WINNERS]++;
    if (jb->prm->check_orientation) orientation_filter(m, k, win, nf, cnt);
    for (int32_t f = 0; f < nf; ++f) {
      if (win[f] == ORC_NONE) continue;
      int32_t slot = m->feat_mp[f0 + f];
      if (slot < 0) cnt[C_ADD]++;
      else if (m->mp_flags[slot] & 1u) cnt[C_BAD_SLOT]++;
      else if (jb->loopset[slot]) cnt[C_LOOP_SKIP]++;
      else {
        cnt[C_VICTIM_PROP]++;
        if (wk->nvp == wk->cap) {
          wk->cap = wk->cap ? 2 * wk->cap : 1024;
          wk->vp = (orc_vprop *)realloc(wk->vp, sizeof(orc_vprop) * (size_t)wk->cap);
        }
        wk->vp[wk->nvp].m = slot;
        wk->vp[wk->nvp].key = win[f];
        wk->nvp++;
      }
    }
  }
  free(held);
  return NULL;
}

/* PLAN over the whole window with n_threads threads; io_winner / io_victim / cnt as
 * orc_fuse(phase = PLAN) (no forced matches, no debug outputs). */
int orc_fuse_plan_grid(orc_map *m, const orc_grid *g, int32_t n_threads, int32_t n_w,
                       const int32_t *window, const double *window_S, const int32_t *win_list_begin,
                       const int32_t *mp_list, int32_t n_list, const orc_params *prm,
                       int64_t *io_winner, int64_t *io_victim, int64_t *cnt) {
  if (n_w <= 0 || n_threads < 1 || !g) return -1;
  double scale[64];
  orc_scale_table(m->n_levels, m->scale_factor, scale);
  int64_t *woff = (int64_t *)malloc(sizeof(int64_t) * (size_t)(n_w + 1));
  woff[0] = 0;
  for (int32_t i = 0; i < n_w; ++i)
    woff[i + 1] = woff[i] + (m->kf_feat_begin[window[i] + 1] - m->kf_feat_begin[window[i]]);
  uint8_t *loopset = (uint8_t *)calloc((size_t)(m->n_mp > 0 ? m->n_mp : 1), 1);
  for (int32_t i = 0; i < n_w; ++i) {
    const int32_t *l; int32_t n;
    list_of(i, win_list_begin, mp_list, n_list, &l, &n);
    for (int32_t j = 0; j < n; ++j) loopset[l[j]] = 1;
  }
  for (int64_t j = 0; j < woff[n_w]; ++j) io_winner[j] = ORC_NONE;
  for (int32_t q = 0; q < m->n_mp; ++q) io_victim[q] = ORC_NONE;
  grid_job jb;
  memset(&jb, 0, sizeof(jb));
  jb.m = m; jb.g = g; jb.n_w = n_w; jb.window = window; jb.window_S = window_S;
  jb.win_list_begin = win_list_begin; jb.mp_list = mp_list; jb.n_list = n_list; jb.prm = prm;
  jb.woff = woff; jb.loopset = loopset; jb.io_winner = io_winner; jb.scale = scale; jb.next = 0;
  pthread_mutex_init(&jb.mu, NULL);
  grid_worker *wk = (grid_worker *)calloc((size_t)n_threads, sizeof(grid_worker));
  pthread_t *th = (pthread_t *)malloc(sizeof(pthread_t) * (size_t)n_threads);
  for (int32_t t = 0; t < n_threads; ++t) {
    wk[t].job = &jb;
    if (t > 0) pthread_create(&th[t], NULL, grid_worker_main, &wk[t]);
  }
  grid_worker_main(&wk[0]);
  for (int32_t t = 1; t < n_threads; ++t) pthread_join(th[t], NULL);
  for (int32_t t = 0; t < n_threads; ++t) {
    for (int c = 0; c < C_N; ++c) cnt[c] += wk[t].cnt[c];
    for (int64_t j = 0; j < wk[t].nvp; ++j)
      if (wk[t].vp[j].key < io_victim[wk[t].vp[j].m]) io_victim[wk[t].vp[j].m] = wk[t].vp[j].key;
    free(wk[t].vp);
  }
  pthread_mutex_destroy(&jb.mu);
  free(wk); free(th); free(loopset); free(woff);
  return 0;
}

/* ------------------------------------------------------------------------- */
/* Projection search over (keyframe, Sim3, parameter set, MP list) pairs:    */
/* PS1, PS2a||PS2b, PS3a-c. Read-only.      */
/* ------------------------------------------------------------------------- */
int orc_search_by_projection(const orc_map *m, int32_t n_pairs, const int32_t *pair_kf,
                             const double *pair_S, const int32_t *pair_param,
                             const orc_params *params, const int32_t *pair_list_begin,
                             const int32_t *mp_list, const int32_t *pair_taken,
                             int32_t *out_feat_mp, int32_t *out_feat_dist, int64_t *out_best,
                             double *out_uv, int32_t *out_ncand, uint8_t *out_edge,
                             int64_t *cnt /* [n_pairs][C_N] */) {
  double scale[64];
  orc_scale_table(m->n_levels, m->scale_factor, scale);
  int64_t off = 0;
  for (int32_t p = 0; p < n_pairs; ++p) {
    int32_t k = pair_kf[p];
    int32_t nf = m->kf_feat_begin[k + 1] - m->kf_feat_begin[k];
    const orc_params *prm = &params[pair_param[p]];
    const int32_t *taken = pair_taken ? pair_taken + off : NULL;
    int64_t *c = cnt + (size_t)C_N * p;
    int64_t *win = (int64_t *)malloc(sizeof(int64_t) * (size_t)(nf > 0 ? nf : 1));
    for (int32_t f = 0; f < nf; ++f) win[f] = ORC_NONE;
    for (int32_t j = pair_list_begin[p]; j < pair_list_begin[p + 1]; ++j) {
      int32_t q = mp_list[j];
      orc_qres r;
      c[C_QUERIES]++;
      query_one(m, k, pair_S + 13 * (size_t)p, q, prm, taken, 1, scale, &r);
      if (out_uv) { out_uv[2 * j] = r.u; out_uv[2 * j + 1] = r.v; }
      if (out_ncand) out_ncand[j] = r.ncand;
      if (out_edge) out_edge[j] = (uint8_t)r.edge;
      if (r.edge) c[C_EDGE_AMB]++;
      if (out_best) out_best[j] = r.status < 0 ? (int64_t)r.status
          : (((int64_t)r.best_h << 48) | ((int64_t)r.second_h << 32) | (uint32_t)r.best_f);
      switch (r.status) {
        case Q_BAD: c[C_SKIP_BAD]++; continue;
        case Q_FOUND: c[C_SKIP_FOUND]++; continue;
        case Q_DEPTH: c[C_CULL_DEPTH]++; continue;
        case Q_BOUNDS: c[C_CULL_BOUNDS]++; continue;
        case Q_DIST: c[C_CULL_DIST]++; continue;
        case Q_ANGLE: c[C_CULL_ANGLE]++; continue;
        default: break;
      }
      c[C_CANDIDATES] += r.ncand;
      if (!proposal_ok(&r, prm, c)) continue;
      int64_t key = ((int64_t)r.best_h << 32) | (int64_t)q;
      if (key < win[r.best_f]) win[r.best_f] = key;
    }
    for (int32_t f = 0; f < nf; ++f) if (win[f] != ORC_NONE) c[C_WINNERS]++;
    if (prm->check_orientation) orientation_filter(m, k, win, nf, c);
    for (int32_t f = 0; f < nf; ++f) {
      int32_t t = taken ? taken[f] : -1;
      if (t >= 0) { out_feat_mp[off + f] = t; out_feat_dist[off + f] = -1; }
      else if (win[f] != ORC_NONE) {
        out_feat_mp[off + f] = (int32_t)(win[f] & 0xffffffff);
        out_feat_dist[off + f] = (int32_t)(win[f] >> 32);
      } else { out_feat_mp[off + f] = -1; out_feat_dist[off + f] = -1; }
    }
    free(win);
    off += nf;
  }
  return 0;
}

/* ------------------------------------------------------------------------- */
/* O11 map-point refresh (readings A33-A37).              */
/*  what & 1: distinctive descriptor (EXT ComputeDistinctiveDescriptors)      */
/*  what & 2: normal + depth range   (EXT UpdateNormalAndDepth)               */
/* ------------------------------------------------------------------------- */
static int cmp_int(const void *a, const void *b) {
  int x = *(const int *)a, y = *(const int *)b;
  return (x > y) - (x < y);
}

/* camera centre of keyframe k: Ow = -R^T (t/s) of its pose (reading A2) */
static void kf_centre(const orc_map *m, int32_t k, double *O) {
  double T[13];
  orc_sim3_se3(m->kf_pose + 13 * (size_t)k, T);
  for (int i = 0; i < 3; ++i) O[i] = -col3(T, i, T + 9);
}

int orc_refresh(orc_map *m, int32_t n, const int32_t *idx, int32_t what, int64_t *cnt) {
  if (n < 0) return -1;
  /* A34: observations of every map point in ascending global feature order
   * (one counting pass over the associations, then an ordered fill) */
  int32_t *kf_of = (int32_t *)malloc(sizeof(int32_t) * (size_t)(m->n_feat > 0 ? m->n_feat : 1));
  int64_t *obeg = (int64_t *)calloc((size_t)m->n_mp + 1, sizeof(int64_t));
  for (int32_t k = 0; k < m->n_kf; ++k)
    for (int32_t f = m->kf_feat_begin[k]; f < m->kf_feat_begin[k + 1]; ++f) kf_of[f] = k;
  for (int32_t f = 0; f < m->n_feat; ++f)
    if (m->feat_mp[f] >= 0) obeg[m->feat_mp[f] + 1]++;
  for (int32_t q = 0; q < m->n_mp; ++q) obeg[q + 1] += obeg[q];
  int32_t *obs = (int32_t *)malloc(sizeof(int32_t) * (size_t)(obeg[m->n_mp] > 0 ? obeg[m->n_mp] : 1));
  int64_t *fill = (int64_t *)malloc(sizeof(int64_t) * (size_t)(m->n_mp > 0 ? m->n_mp : 1));
  for (int32_t q = 0; q < m->n_mp; ++q) fill[q] = obeg[q];
  for (int32_t f = 0; f < m->n_feat; ++f)
    if (m->feat_mp[f] >= 0) obs[fill[m->feat_mp[f]]++] = f;
  double scale[64];
  orc_scale_table(m->n_levels, m->scale_factor, scale);
  int64_t *c = cnt;
  const int32_t total = idx ? n : m->n_mp;
  for (int32_t t = 0; t < total; ++t) {
    const int32_t q = idx ? idx[t] : t;
    if (q < 0 || q >= m->n_mp) continue;
    if (m->mp_flags[q] & 1u) continue;                      /* A33: bad points are skipped */
    const int32_t *o = obs + obeg[q];
    const int32_t N = (int32_t)(obeg[q + 1] - obeg[q]);
    if (N == 0) continue;
    c[C_REFRESH_MP]++;
    c[C_REFRESH_OBS] += N;
    if (what & 1) {
      /* A35: least median Hamming distance to the other observation descriptors;
       * median = sorted row [floor((N-1)/2)]; the first such observation wins */
      int *row = (int *)malloc(sizeof(int) * (size_t)N);
      int best_med = 1 << 30, best_i = 0;
      for (int32_t i = 0; i < N; ++i) {
        for (int32_t j = 0; j < N; ++j)
          row[j] = orc_hamming(m->feat_desc + 32 * (size_t)o[i], m->feat_desc + 32 * (size_t)o[j]);
        qsort(row, (size_t)N, sizeof(int), cmp_int);
        const int med = row[(N - 1) / 2];
        if (med < best_med) { best_med = med; best_i = i; }
      }
      memcpy(m->mp_desc + 32 * (size_t)q, m->feat_desc + 32 * (size_t)o[best_i], 32);
      free(row);
    }
    if (what & 2) {
      /* A36: normal = (sum of unit vectors from the observing cameras) / N, in
       * observation order; zero-length vectors are skipped and not counted */
      const double p[3] = {(double)m->mp_pos[3 * (size_t)q], (double)m->mp_pos[3 * (size_t)q + 1],
                           (double)m->mp_pos[3 * (size_t)q + 2]};
      double acc[3] = {0.0, 0.0, 0.0};
      int32_t nn = 0;
      for (int32_t i = 0; i < N; ++i) {
        double O[3], v[3];
        kf_centre(m, kf_of[o[i]], O);
        for (int j = 0; j < 3; ++j) v[j] = p[j] - O[j];
        const double len = sqrt((v[0] * v[0] + v[1] * v[1]) + v[2] * v[2]);
        if (len == 0.0) continue;
        for (int j = 0; j < 3; ++j) acc[j] = acc[j] + v[j] / len;
        ++nn;
      }
      if (nn > 0)
        for (int j = 0; j < 3; ++j) m->mp_normal[3 * (size_t)q + j] = (float)(acc[j] / (double)nn);
      /* A37: dmax = |p - O_ref| * s_level, level = octave of the reference
       * keyframe's (first) observation; unchanged if it does not observe q */
      const int32_t ref = m->mp_ref_kf[q];
      for (int32_t i = 0; i < N; ++i) {
        if (kf_of[o[i]] != ref) continue;
        double O[3], v[3];
        kf_centre(m, ref, O);
        for (int j = 0; j < 3; ++j) v[j] = p[j] - O[j];
        const double dist = sqrt((v[0] * v[0] + v[1] * v[1]) + v[2] * v[2]);
        int lvl = m->feat_octave[o[i]];
        if (lvl >= m->n_levels) lvl = m->n_levels - 1;
        m->mp_max_dist[q] = (float)(dist * scale[lvl]);
        break;
      }
    }
  }
  free(kf_of); free(obeg); free(obs); free(fill);
  return 0;
}

/* ------------------------------------------------------------------------- */
/* O12 covisibility recount (readings A38-A40).           */
/* For each selected keyframe k: weight(k, k2) = number of distinct non-bad   */
/* map points held by k that k2 (!= k) also holds; edges with weight >= th,   */
/* or the single strongest one if none reaches th; ordered by weight desc,   */
/* then keyframe id asc. out_n[i] = number of edges (may exceed max_edges;    */
/* only the first max_edges are written to out_kf / out_w [i*max_edges...]).  */
/* ------------------------------------------------------------------------- */
int orc_update_connections(orc_map *m, int32_t n, const int32_t *idx, int32_t th, int32_t max_edges,
                           int32_t *out_n, int32_t *out_kf, int32_t *out_w, int64_t *cnt) {
  if (n < 0 || max_edges < 0) return -1;
  int32_t *kf_of = (int32_t *)malloc(sizeof(int32_t) * (size_t)(m->n_feat > 0 ? m->n_feat : 1));
  for (int32_t k = 0; k < m->n_kf; ++k)
    for (int32_t f = m->kf_feat_begin[k]; f < m->kf_feat_begin[k + 1]; ++f) kf_of[f] = k;
  /* holds[q] lists, per map point, the keyframes holding it (ascending, distinct) */
  int64_t *hbeg = (int64_t *)calloc((size_t)m->n_mp + 1, sizeof(int64_t));
  for (int32_t f = 0; f < m->n_feat; ++f)
    if (m->feat_mp[f] >= 0) hbeg[m->feat_mp[f] + 1]++;
  for (int32_t q = 0; q < m->n_mp; ++q) hbeg[q + 1] += hbeg[q];
  int32_t *holds = (int32_t *)malloc(sizeof(int32_t) * (size_t)(hbeg[m->n_mp] > 0 ? hbeg[m->n_mp] : 1));
  int64_t *hn = (int64_t *)calloc((size_t)(m->n_mp > 0 ? m->n_mp : 1), sizeof(int64_t));
  for (int32_t f = 0; f < m->n_feat; ++f) {   /* features ascending -> keyframes ascending */
    const int32_t q = m->feat_mp[f];
    if (q < 0) continue;
    const int32_t k = kf_of[f];
    if (hn[q] > 0 && holds[hbeg[q] + hn[q] - 1] == k) continue;   /* k holds q twice: once */
    holds[hbeg[q] + hn[q]++] = k;
  }
  int32_t *w = (int32_t *)calloc((size_t)(m->n_kf > 0 ? m->n_kf : 1), sizeof(int32_t));
  uint8_t *seen = (uint8_t *)calloc((size_t)(m->n_mp > 0 ? m->n_mp : 1), 1);
  const int32_t total = idx ? n : m->n_kf;
  for (int32_t t = 0; t < total; ++t) {
    const int32_t k = idx ? idx[t] : t;
    if (out_n) out_n[t] = 0;
    if (k < 0 || k >= m->n_kf) continue;
    memset(w, 0, sizeof(int32_t) * (size_t)m->n_kf);
    for (int32_t f = m->kf_feat_begin[k]; f < m->kf_feat_begin[k + 1]; ++f) {
      const int32_t q = m->feat_mp[f];
      if (q < 0 || (m->mp_flags[q] & 1u) || seen[q]) continue;   /* A38: distinct, not bad */
      seen[q] = 1;
      for (int64_t h = hbeg[q]; h < hbeg[q] + hn[q]; ++h)
        if (holds[h] != k) w[holds[h]]++;
    }
    for (int32_t f = m->kf_feat_begin[k]; f < m->kf_feat_begin[k + 1]; ++f)
      if (m->feat_mp[f] >= 0) seen[m->feat_mp[f]] = 0;
    /* A39 + A40: edges >= th by (weight desc, id asc); else the strongest one */
    int32_t ne = 0;
    for (int32_t k2 = 0; k2 < m->n_kf; ++k2) ne += w[k2] >= th && w[k2] > 0;
    int32_t wr = 0;
    if (ne == 0) {
      int32_t best = -1;
      for (int32_t k2 = 0; k2 < m->n_kf; ++k2)
        if (w[k2] > 0 && (best < 0 || w[k2] > w[best])) best = k2;
      if (best >= 0) {
        ne = 1;
        if (max_edges > 0 && out_kf) { out_kf[(size_t)t * max_edges] = best; out_w[(size_t)t * max_edges] = w[best]; }
      }
    } else {
      int32_t last_w = 1 << 30, last_k = -1;   /* selection in (weight desc, id asc) order */
      for (int32_t e = 0; e < ne; ++e) {
        int32_t bk = -1;
        for (int32_t k2 = 0; k2 < m->n_kf; ++k2) {
          if (!(w[k2] >= th && w[k2] > 0)) continue;
          const int after = w[k2] < last_w || (w[k2] == last_w && k2 > last_k);
          if (!after) continue;
          if (bk < 0 || w[k2] > w[bk] || (w[k2] == w[bk] && k2 < bk)) bk = k2;
        }
        last_w = w[bk]; last_k = bk;
        if (wr < max_edges && out_kf) {
          out_kf[(size_t)t * max_edges + wr] = bk;
          out_w[(size_t)t * max_edges + wr] = w[bk];
          ++wr;
        }
      }
    }
    if (out_n) out_n[t] = ne;
    cnt[C_CONN_KF]++;
    cnt[C_CONN_EDGES] += ne;
  }
  free(kf_of); free(hbeg); free(holds); free(hn); free(w); free(seen);
  return 0;
}

/* ------------------------------------------------------------------------- */
/* O13 Sim3 RANSAC (readings A41-A44).                    */
/* ------------------------------------------------------------------------- */
/* A42: eigen-decomposition of a symmetric 4x4 by cyclic Jacobi rotations in  */
/* the fixed order (0,1),(0,2),(0,3),(1,2),(1,3),(2,3); at most 50 sweeps,    */
/* stop when the off-diagonal sum of squares is 0 or <= 1e-300.               */
void orc_jacobi4(const double *A_in, double *evals, double *evecs /* [4][4] columns */) {
  double A[16], V[16];
  memcpy(A, A_in, sizeof(A));
  for (int i = 0; i < 16; ++i) V[i] = (i % 5 == 0) ? 1.0 : 0.0;
  for (int sweep = 0; sweep < 50; ++sweep) {
    double off = 0.0;
    for (int p = 0; p < 4; ++p)
      for (int q = p + 1; q < 4; ++q) off = off + A[4 * p + q] * A[4 * p + q];
    if (off <= 1e-300) break;
    for (int p = 0; p < 4; ++p)
      for (int q = p + 1; q < 4; ++q) {
        const double apq = A[4 * p + q];
        if (apq == 0.0) continue;
        const double theta = (A[4 * q + q] - A[4 * p + p]) / (2.0 * apq);
        const double t = (theta >= 0.0 ? 1.0 : -1.0) / (fabs(theta) + sqrt(theta * theta + 1.0));
        const double c = 1.0 / sqrt(t * t + 1.0), sn = t * c;
        for (int k = 0; k < 4; ++k) {   /* columns p, q of A */
          const double akp = A[4 * k + p], akq = A[4 * k + q];
          A[4 * k + p] = c * akp - sn * akq;
          A[4 * k + q] = sn * akp + c * akq;
        }
        for (int k = 0; k < 4; ++k) {   /* rows p, q of A */
          const double apk = A[4 * p + k], aqk = A[4 * q + k];
          A[4 * p + k] = c * apk - sn * aqk;
          A[4 * q + k] = sn * apk + c * aqk;
        }
        for (int k = 0; k < 4; ++k) {   /* eigenvector columns */
          const double vkp = V[4 * k + p], vkq = V[4 * k + q];
          V[4 * k + p] = c * vkp - sn * vkq;
          V[4 * k + q] = sn * vkp + c * vkq;
        }
      }
  }
  for (int i = 0; i < 4; ++i) evals[i] = A[4 * i + i];
  memcpy(evecs, V, sizeof(V));
}

/* A42: closed-form similarity S12 (p1 ~ s R p2 + t) from n >= 3 correspondences:
 * centroids, M = sum (p2-c2)(p1-c1)^T (EXT M = Pr2 Pr1^T), Horn's N, quaternion = eigenvector of the
 * largest eigenvalue (first on ties; sign so that w > 0, else the first non-zero
 * component > 0), R from the quaternion, s = sum (p1-c1).(R(p2-c2)) / sum |R(p2-c2)|^2
 * (1 when fix_scale), t = c1 - s R c2. Sums run in index order. Output 13-vector. */
void orc_horn(int32_t n, const int32_t *sel, const double *P1, const double *P2, int32_t fix_scale,
              double *S) {
  double c1[3] = {0, 0, 0}, c2[3] = {0, 0, 0};
  for (int32_t i = 0; i < n; ++i)
    for (int j = 0; j < 3; ++j) {
      c1[j] = c1[j] + P1[3 * (size_t)sel[i] + j];
      c2[j] = c2[j] + P2[3 * (size_t)sel[i] + j];
    }
  for (int j = 0; j < 3; ++j) { c1[j] = c1[j] / (double)n; c2[j] = c2[j] / (double)n; }
  double M[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
  for (int32_t i = 0; i < n; ++i) {
    double a[3], b[3];
    for (int j = 0; j < 3; ++j) { a[j] = P1[3 * (size_t)sel[i] + j] - c1[j]; b[j] = P2[3 * (size_t)sel[i] + j] - c2[j]; }
    for (int r = 0; r < 3; ++r)   /* M = sum (p2 - c2)(p1 - c1)^T: R maps frame 2 into 1 */
      for (int cc = 0; cc < 3; ++cc) M[3 * r + cc] = M[3 * r + cc] + b[r] * a[cc];
  }
  double N[16];
  N[0] = (M[0] + M[4]) + M[8];  N[1] = M[5] - M[7];          N[2] = M[6] - M[2];          N[3] = M[1] - M[3];
  N[5] = (M[0] - M[4]) - M[8];  N[6] = M[1] + M[3];          N[7] = M[6] + M[2];
  N[10] = (-M[0] + M[4]) - M[8]; N[11] = M[5] + M[7];
  N[15] = (-M[0] - M[4]) + M[8];
  N[4] = N[1]; N[8] = N[2]; N[12] = N[3]; N[9] = N[6]; N[13] = N[7]; N[14] = N[11];
  double ev[4], V[16];
  orc_jacobi4(N, ev, V);
  int best = 0;
  for (int i = 1; i < 4; ++i) if (ev[i] > ev[best]) best = i;
  double q[4] = {V[best], V[4 + best], V[8 + best], V[12 + best]};   /* (w, x, y, z) */
  int lead = 0;
  while (lead < 3 && q[lead] == 0.0) ++lead;
  if (q[lead] < 0.0) for (int i = 0; i < 4; ++i) q[i] = -q[i];
  const double w = q[0], x = q[1], y = q[2], z = q[3];
  double R[9];
  R[0] = ((w * w + x * x) - y * y) - z * z; R[1] = 2.0 * (x * y - w * z);         R[2] = 2.0 * (x * z + w * y);
  R[3] = 2.0 * (x * y + w * z);         R[4] = ((w * w - x * x) + y * y) - z * z; R[5] = 2.0 * (y * z - w * x);
  R[6] = 2.0 * (x * z - w * y);         R[7] = 2.0 * (y * z + w * x);         R[8] = ((w * w - x * x) - y * y) + z * z;
  double nom = 0.0, den = 0.0;
  for (int32_t i = 0; i < n; ++i) {
    double a[3], b[3], rb[3];
    for (int j = 0; j < 3; ++j) { a[j] = P1[3 * (size_t)sel[i] + j] - c1[j]; b[j] = P2[3 * (size_t)sel[i] + j] - c2[j]; }
    for (int j = 0; j < 3; ++j) rb[j] = row3(R + 3 * j, b);
    nom = nom + ((a[0] * rb[0] + a[1] * rb[1]) + a[2] * rb[2]);
    den = den + ((rb[0] * rb[0] + rb[1] * rb[1]) + rb[2] * rb[2]);
  }
  const double sc = fix_scale ? 1.0 : nom / den;
  memcpy(S, R, sizeof(R));
  for (int j = 0; j < 3; ++j) S[9 + j] = c1[j] - sc * row3(R + 3 * j, c2);
  S[12] = sc;
}

/* A43: both reprojection errors below chi2 * sigma^2; behind a camera = outlier */
static int ransac_inlier(const orc_camera *cam1, const orc_camera *cam2, const double *S12,
                         const double *S21, const double *p1, const double *p2, const float *uv1,
                         const float *uv2, float s1, float s2, double chi2) {
  double a[3], b[3], uv[2];
  orc_sim3_apply(S12, p2, a);                 /* P2 in camera 1 */
  if (a[2] <= 0.0) return 0;
  orc_project(cam1, a, uv);
  double du = uv[0] - (double)uv1[0], dv = uv[1] - (double)uv1[1];
  if (!(du * du + dv * dv < chi2 * (double)s1)) return 0;
  orc_sim3_apply(S21, p1, b);                 /* P1 in camera 2 */
  if (b[2] <= 0.0) return 0;
  orc_project(cam2, b, uv);
  du = uv[0] - (double)uv2[0]; dv = uv[1] - (double)uv2[1];
  return du * du + dv * dv < chi2 * (double)s2;
}

int orc_sim3_ransac(const orc_map *m, int32_t n_prob, const int32_t *pbeg, const double *P1,
                    const double *P2, const float *uv1, const float *uv2, const float *sig1,
                    const float *sig2, const int32_t *cam1, const int32_t *cam2, const int32_t *samples,
                    int32_t n_iter, double chi2, int32_t fix_scale, int32_t refit, double *out_S,
                    int32_t *out_inl, uint8_t *out_mask, int64_t *cnt) {
  for (int32_t b = 0; b < n_prob; ++b) {
    const int32_t c0 = pbeg[b], nc = pbeg[b + 1] - pbeg[b];
    const orc_camera *k1 = m->cams + cam1[b], *k2 = m->cams + cam2[b];
    int32_t best_inl = -1, best_it = -1;
    double bestS[13];
    for (int32_t it = 0; it < n_iter; ++it) {
      const int32_t *t = samples + 3 * ((size_t)b * n_iter + it);
      if (t[0] < 0 || t[1] < 0 || t[2] < 0 || t[0] >= nc || t[1] >= nc || t[2] >= nc ||
          t[0] == t[1] || t[0] == t[2] || t[1] == t[2]) continue;   /* A41 */
      int32_t sel[3] = {c0 + t[0], c0 + t[1], c0 + t[2]};
      double S[13], Si[13];
      orc_horn(3, sel, P1, P2, fix_scale, S);
      orc_sim3_inverse(S, Si);
      cnt[C_RANSAC_HYP]++;
      int32_t ninl = 0;
      for (int32_t i = 0; i < nc; ++i)
        ninl += ransac_inlier(k1, k2, S, Si, P1 + 3 * (size_t)(c0 + i), P2 + 3 * (size_t)(c0 + i),
                              uv1 + 2 * (size_t)(c0 + i), uv2 + 2 * (size_t)(c0 + i), sig1[c0 + i],
                              sig2[c0 + i], chi2);
      if (ninl > best_inl) { best_inl = ninl; best_it = it; memcpy(bestS, S, sizeof(S)); }   /* A44 */
    }
    if (best_it < 0) {   /* no valid sample */
      for (int i = 0; i < 13; ++i) out_S[13 * (size_t)b + i] = 0.0;
      out_inl[b] = 0;
      for (int32_t i = 0; i < nc; ++i) out_mask[c0 + i] = 0;
      continue;
    }
    double Si[13];
    orc_sim3_inverse(bestS, Si);
    int32_t *sel = (int32_t *)malloc(sizeof(int32_t) * (size_t)(nc > 0 ? nc : 1));
    int32_t ns = 0;
    for (int32_t i = 0; i < nc; ++i) {
      const int in = ransac_inlier(k1, k2, bestS, Si, P1 + 3 * (size_t)(c0 + i), P2 + 3 * (size_t)(c0 + i),
                                   uv1 + 2 * (size_t)(c0 + i), uv2 + 2 * (size_t)(c0 + i), sig1[c0 + i],
                                   sig2[c0 + i], chi2);
      out_mask[c0 + i] = (uint8_t)in;
      if (in) sel[ns++] = c0 + i;
    }
    out_inl[b] = ns;
    cnt[C_RANSAC_INLIERS] += ns;
    if (refit && ns >= 3) orc_horn(ns, sel, P1, P2, fix_scale, bestS);   /* A44 */
    memcpy(out_S + 13 * (size_t)b, bestS, sizeof(bestS));
    free(sel);
  }
  return 0;
}

/* ------------------------------------------------------------------------- */
/* O14 Sim3 refinement (readings A45-A48).                */
/* ------------------------------------------------------------------------- */
/* A45: retraction S <- D(d) o S, D(d) = (Cayley(w), tau, 1 + sig) for the      */
/* 7-vector d = (w0..2, tau0..2, sig): Cayley(w) = (I - [w]x)^-1 (I + [w]x) in  */
/* closed form (rational: identical in any IEEE implementation).              */
void orc_sim3_retract(const double *d, const double *S, double *out) {
  const double a = d[0], b = d[1], c = d[2];
  const double n2 = (a * a + b * b) + c * c;
  const double k = 1.0 / (1.0 + n2);
  double D[13];
  D[0] = ((1.0 + a * a) - b * b - c * c) * k;  D[1] = 2.0 * (a * b - c) * k;          D[2] = 2.0 * (a * c + b) * k;
  D[3] = 2.0 * (a * b + c) * k;          D[4] = ((1.0 - a * a) + b * b - c * c) * k;  D[5] = 2.0 * (b * c - a) * k;
  D[6] = 2.0 * (a * c - b) * k;          D[7] = 2.0 * (b * c + a) * k;          D[8] = ((1.0 - a * a) - b * b + c * c) * k;
  D[9] = d[3]; D[10] = d[4]; D[11] = d[5]; D[12] = 1.0 + d[6];
  orc_sim3_compose(D, S, out);
}

/* residuals of correspondence i under S (S21 = inverse(S)): r[0..1] = pi1(S p2) - uv1,
 * r[2..3] = pi2(S21 p1) - uv2; returns 0 if a point is behind a camera */
static int refine_res(const orc_camera *k1, const orc_camera *k2, const double *S, const double *p1,
                      const double *p2, const float *uv1, const float *uv2, double *r) {
  double Si[13], a[3], b[3], uv[2];
  orc_sim3_inverse(S, Si);
  orc_sim3_apply(S, p2, a);
  orc_sim3_apply(Si, p1, b);
  if (a[2] <= 0.0 || b[2] <= 0.0) return 0;
  orc_project(k1, a, uv);
  r[0] = uv[0] - (double)uv1[0]; r[1] = uv[1] - (double)uv1[1];
  orc_project(k2, b, uv);
  r[2] = uv[0] - (double)uv2[0]; r[3] = uv[1] - (double)uv2[1];
  return 1;
}

/* Huber weight of a chi2 value e2 = |r|^2 / sigma2 (A47): 1 if sqrt(e2) <= delta,
 * else delta / sqrt(e2) */
static double huber_w(double e2, double delta) {
  const double e = sqrt(e2);
  return e <= delta ? 1.0 : delta / e;
}

/* A46/A47: Gauss-Newton with central-difference Jacobians (h = 1e-6), Huber-weighted
 * normal equations accumulated in correspondence order, H + lambda*diag(H) solved by
 * the 7x7 Cholesky in fixed order; stop when |d|^2 < 1e-20 or after max_iter; A48:
 * inliers = both chi2 < th2 under the final model. Correspondences behind a camera
 * at the current model contribute nothing. */
/* chi2 of both residuals of correspondence i under S; 0 if behind a camera */
static int refine_chi2(const orc_camera *k1, const orc_camera *k2, const double *S, const double *p1,
                       const double *p2, const float *u1, const float *u2, float s1, float s2,
                       double *e1, double *e2) {
  double r[4];
  if (!refine_res(k1, k2, S, p1, p2, u1, u2, r)) return 0;
  *e1 = (r[0] * r[0] + r[1] * r[1]) / (double)s1;
  *e2 = (r[2] * r[2] + r[3] * r[3]) / (double)s2;
  return 1;
}

/* one Gauss-Newton step over the active correspondences; returns 0 if H is not SPD */
static int refine_step(const orc_camera *k1, const orc_camera *k2, int32_t c0, int32_t nc,
                       const uint8_t *act, const double *P1, const double *P2, const float *uv1,
                       const float *uv2, const float *sig1, const float *sig2, double delta,
                       double lambda, double *S, double *dn_out) {
  const double h = 1e-6;
  double H[49], g[7];
  for (int i = 0; i < 49; ++i) H[i] = 0.0;
  for (int i = 0; i < 7; ++i) g[i] = 0.0;
  for (int32_t i = 0; i < nc; ++i) {
    if (!act[i]) continue;
    const double *p1 = P1 + 3 * (size_t)(c0 + i), *p2 = P2 + 3 * (size_t)(c0 + i);
    const float *u1 = uv1 + 2 * (size_t)(c0 + i), *u2 = uv2 + 2 * (size_t)(c0 + i);
    double r[4], J[4][7];
    if (!refine_res(k1, k2, S, p1, p2, u1, u2, r)) continue;
    int ok = 1;
    for (int j = 0; j < 7 && ok; ++j) {
      double dp[7] = {0, 0, 0, 0, 0, 0, 0}, dm[7] = {0, 0, 0, 0, 0, 0, 0};
      dp[j] = h; dm[j] = -h;
      double Sp[13], Sm[13], rp[4], rm[4];
      orc_sim3_retract(dp, S, Sp);
      orc_sim3_retract(dm, S, Sm);
      ok = refine_res(k1, k2, Sp, p1, p2, u1, u2, rp) && refine_res(k1, k2, Sm, p1, p2, u1, u2, rm);
      for (int q = 0; q < 4; ++q) J[q][j] = (rp[q] - rm[q]) / (2.0 * h);
    }
    if (!ok) continue;
    const double s1 = (double)sig1[c0 + i], s2 = (double)sig2[c0 + i];
    const double e1 = (r[0] * r[0] + r[1] * r[1]) / s1, e2 = (r[2] * r[2] + r[3] * r[3]) / s2;
    const double w1 = huber_w(e1, delta) / s1, w2 = huber_w(e2, delta) / s2;
    for (int q = 0; q < 4; ++q) {
      const double wq = q < 2 ? w1 : w2;
      for (int x = 0; x < 7; ++x) {
        g[x] = g[x] + wq * J[q][x] * r[q];
        for (int y = 0; y <= x; ++y) H[7 * x + y] = H[7 * x + y] + wq * J[q][x] * J[q][y];
      }
    }
  }
  double L[49];   /* Cholesky of H + lambda * diag(H) (lower), then H d = -g */
  for (int x = 0; x < 7; ++x)
    for (int y = 0; y <= x; ++y) L[7 * x + y] = H[7 * x + y] + (x == y ? lambda * H[7 * x + x] : 0.0);
  for (int x = 0; x < 7; ++x)
    for (int y = 0; y <= x; ++y) {
      double acc = L[7 * x + y];
      for (int k = 0; k < y; ++k) acc = acc - L[7 * x + k] * L[7 * y + k];
      if (x == y) {
        if (!(acc > 0.0)) return 0;
        L[7 * x + x] = sqrt(acc);
      } else {
        L[7 * x + y] = acc / L[7 * y + y];
      }
    }
  double z[7], d[7];
  for (int x = 0; x < 7; ++x) {
    double acc = -g[x];
    for (int k = 0; k < x; ++k) acc = acc - L[7 * x + k] * z[k];
    z[x] = acc / L[7 * x + x];
  }
  for (int x = 6; x >= 0; --x) {
    double acc = z[x];
    for (int k = x + 1; k < 7; ++k) acc = acc - L[7 * k + x] * d[k];
    d[x] = acc / L[7 * x + x];
  }
  double S2[13];
  orc_sim3_retract(d, S, S2);
  memcpy(S, S2, sizeof(S2));
  double dn = 0.0;
  for (int x = 0; x < 7; ++x) dn = dn + d[x] * d[x];
  *dn_out = dn;
  return 1;
}

/* A46-A48: Gauss-Newton with central-difference Jacobians (h = 1e-6) and Huber
 * weights (delta = sqrt(th2)), normal equations accumulated in correspondence order,
 * H + lambda diag(H) solved by the fixed-order 7x7 Cholesky; phase 1 (<= 5 steps) on
 * all correspondences, then those with a chi2 >= th2 (or behind a camera) are dropped
 * (EXT OptimizeSim3), phase 2 (<= max_iter steps) on the rest; a phase stops when
 * |d|^2 < 1e-20 or H is not positive definite. Inliers: both chi2 < th2 under the
 * final model. */
int orc_sim3_refine(const orc_map *m, int32_t n_prob, const int32_t *pbeg, const double *P1,
                    const double *P2, const float *uv1, const float *uv2, const float *sig1,
                    const float *sig2, const int32_t *cam1, const int32_t *cam2, const double *S_in,
                    int32_t max_iter, double th2, double lambda, double *out_S, int32_t *out_inl,
                    uint8_t *out_mask, int64_t *cnt) {
  const double delta = sqrt(th2);
  for (int32_t b = 0; b < n_prob; ++b) {
    const int32_t c0 = pbeg[b], nc = pbeg[b + 1] - pbeg[b];
    const orc_camera *k1 = m->cams + cam1[b], *k2 = m->cams + cam2[b];
    double S[13];
    memcpy(S, S_in + 13 * (size_t)b, sizeof(S));
    uint8_t *act = (uint8_t *)malloc((size_t)(nc > 0 ? nc : 1));
    for (int32_t i = 0; i < nc; ++i) act[i] = 1;
    for (int phase = 0; phase < 2; ++phase) {
      const int32_t n_it = phase == 0 ? (max_iter < 5 ? max_iter : 5) : max_iter;
      for (int32_t it = 0; it < n_it; ++it) {
        double dn = 0.0;
        if (!refine_step(k1, k2, c0, nc, act, P1, P2, uv1, uv2, sig1, sig2, delta, lambda, S, &dn)) break;
        cnt[C_REFINE_ITERS]++;
        if (dn < 1e-20) break;
      }
      if (phase == 0)
        for (int32_t i = 0; i < nc; ++i) {
          double e1, e2;
          act[i] = refine_chi2(k1, k2, S, P1 + 3 * (size_t)(c0 + i), P2 + 3 * (size_t)(c0 + i),
                               uv1 + 2 * (size_t)(c0 + i), uv2 + 2 * (size_t)(c0 + i), sig1[c0 + i],
                               sig2[c0 + i], &e1, &e2) && e1 < th2 && e2 < th2;
        }
    }
    int32_t ninl = 0;
    for (int32_t i = 0; i < nc; ++i) {
      double e1, e2;
      const int in = refine_chi2(k1, k2, S, P1 + 3 * (size_t)(c0 + i), P2 + 3 * (size_t)(c0 + i),
                                 uv1 + 2 * (size_t)(c0 + i), uv2 + 2 * (size_t)(c0 + i), sig1[c0 + i],
                                 sig2[c0 + i], &e1, &e2) && e1 < th2 && e2 < th2;
      out_mask[c0 + i] = (uint8_t)in;
      ninl += in;
    }
    out_inl[b] = ninl;
    cnt[C_REFINE_INLIERS] += ninl;
    memcpy(out_S + 13 * (size_t)b, S, sizeof(S));
    free(act);
  }
  return 0;
}

/* ------------------------------------------------------------------------- */
/* O15 Essential-graph Sim3 pose-graph optimisation.     */
/* PAPER.md:244-248 §IV.F: "an essential (pose) graph optimization to          */
/* propagate the loop correction", Jacobians by "automatic differentiation",   */
/* "Eigen LDLT for the linear solver"; "Levenberg-Marquardt pose optimization  */
/* scheme" (Conclusion). The paper gives no formulas: the residual, tangent     */
/* order, exp/log branches, damping and stopping rules are readings A49-A53.    */
/* ------------------------------------------------------------------------- */
/* Forward-mode dual numbers with 7 partials (SPEC.md DualNumber7): a value and
 * its derivatives w.r.t. the 7 tangent coordinates of one vertex. */
typedef struct { double v; double d[7]; } d7;

static d7 d7c(double x) { d7 r; r.v = x; for (int k = 0; k < 7; ++k) r.d[k] = 0.0; return r; }
static d7 d7add(d7 a, d7 b) { d7 r; r.v = a.v + b.v; for (int k = 0; k < 7; ++k) r.d[k] = a.d[k] + b.d[k]; return r; }
static d7 d7sub(d7 a, d7 b) { d7 r; r.v = a.v - b.v; for (int k = 0; k < 7; ++k) r.d[k] = a.d[k] - b.d[k]; return r; }
static d7 d7mul(d7 a, d7 b) {
  d7 r; r.v = a.v * b.v;
  for (int k = 0; k < 7; ++k) r.d[k] = a.d[k] * b.v + a.v * b.d[k];
  return r;
}
static d7 d7div(d7 a, d7 b) {
  d7 r; r.v = a.v / b.v;
  for (int k = 0; k < 7; ++k) r.d[k] = (a.d[k] * b.v - a.v * b.d[k]) / (b.v * b.v);
  return r;
}
static d7 d7scl(d7 a, double c) { d7 r; r.v = a.v * c; for (int k = 0; k < 7; ++k) r.d[k] = a.d[k] * c; return r; }
static d7 d7addc(d7 a, double c) { a.v += c; return a; }
/* chain rule: f(a) with f' = df at a.v */
static d7 d7fn(d7 a, double f, double df) { d7 r; r.v = f; for (int k = 0; k < 7; ++k) r.d[k] = df * a.d[k]; return r; }
static d7 d7sqrt(d7 a) { const double s = sqrt(a.v); return d7fn(a, s, 0.5 / s); }
static d7 d7sin(d7 a) { return d7fn(a, sin(a.v), cos(a.v)); }
static d7 d7cos(d7 a) { return d7fn(a, cos(a.v), -sin(a.v)); }
static d7 d7exp(d7 a) { const double e = exp(a.v); return d7fn(a, e, e); }
static d7 d7expm1(d7 a) { return d7fn(a, expm1(a.v), exp(a.v)); }
static d7 d7log(d7 a) { return d7fn(a, log(a.v), 1.0 / a.v); }
static d7 d7atan2(d7 y, d7 x) {
  d7 r; r.v = atan2(y.v, x.v);
  const double den = x.v * x.v + y.v * y.v;
  for (int k = 0; k < 7; ++k) r.d[k] = (x.v * y.d[k] - y.v * x.d[k]) / den;
  return r;
}
static d7 d7dot3(const d7 *a, const d7 *b) { return d7add(d7add(d7mul(a[0], b[0]), d7mul(a[1], b[1])), d7mul(a[2], b[2])); }
static void d7cross(const d7 *a, const d7 *b, d7 *o) {
  d7 r[3];
  r[0] = d7sub(d7mul(a[1], b[2]), d7mul(a[2], b[1]));
  r[1] = d7sub(d7mul(a[2], b[0]), d7mul(a[0], b[2]));
  r[2] = d7sub(d7mul(a[0], b[1]), d7mul(a[1], b[0]));
  o[0] = r[0]; o[1] = r[1]; o[2] = r[2];
}

/* Sim3 with dual entries: p' = s R p + t (reading A1 layout) */
typedef struct { d7 R[9]; d7 t[3]; d7 s; } s7;

static s7 s7c(const double *S) {
  s7 r;
  for (int i = 0; i < 9; ++i) r.R[i] = d7c(S[i]);
  for (int i = 0; i < 3; ++i) r.t[i] = d7c(S[9 + i]);
  r.s = d7c(S[12]);
  return r;
}
/* A o B: R = R_A R_B, t = s_A R_A t_B + t_A, s = s_A s_B (same as orc_sim3_compose) */
static s7 s7compose(const s7 *A, const s7 *B) {
  s7 r;
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j)
      r.R[3 * i + j] = d7add(d7add(d7mul(A->R[3 * i + 0], B->R[0 + j]), d7mul(A->R[3 * i + 1], B->R[3 + j])),
                             d7mul(A->R[3 * i + 2], B->R[6 + j]));
  for (int i = 0; i < 3; ++i)
    r.t[i] = d7add(d7mul(A->s, d7dot3(A->R + 3 * i, B->t)), A->t[i]);
  r.s = d7mul(A->s, B->s);
  return r;
}
/* inverse: R^T, -R^T t / s, 1/s */
static s7 s7inverse(const s7 *S) {
  s7 r;
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) r.R[3 * i + j] = S->R[3 * j + i];
  for (int i = 0; i < 3; ++i) {
    d7 c = d7add(d7add(d7mul(S->R[0 + i], S->t[0]), d7mul(S->R[3 + i], S->t[1])), d7mul(S->R[6 + i], S->t[2]));
    r.t[i] = d7scl(d7div(c, S->s), -1.0);
  }
  r.s = d7div(d7c(1.0), S->s);
  return r;
}

/* A49: coefficients of W(omega, sigma) = A I + B Omega + C Omega^2, the integral
 * int_0^1 e^(sigma tau) exp(tau Omega) dtau, with th2 = |omega|^2:
 *   A = expm1(s)/s; B = (e^s s sin(th) + th (2 sin^2(th/2) - expm1(s) cos(th))) / (th (s^2 + th^2));
 *   C = (A - ((expm1(s) cos(th) - 2 sin^2(th/2)) s + e^s sin(th) th) / (s^2 + th^2)) / th^2;
 * for |s| < 1e-3 A is its Taylor series to s^3; for th < 1e-4 B, C are their th -> 0
 * limits B0(s) = int tau e^(s tau), C0(s) = int tau^2/2 e^(s tau) (Taylor series to s^3
 * when |s| < 1e-3, else closed form). */
static void pgo_coef(d7 th2, d7 sg, d7 *A, d7 *B, d7 *C) {
  const int ssmall = fabs(sg.v) < 1e-3;
  if (ssmall) {  /* 1 + s/2 + s^2/6 + s^3/24 */
    *A = d7addc(d7mul(sg, d7addc(d7mul(sg, d7addc(d7scl(sg, 1.0 / 24.0), 1.0 / 6.0)), 0.5)), 1.0);
  } else {
    *A = d7div(d7expm1(sg), sg);
  }
  if (th2.v < 1e-8) {
    if (ssmall) {  /* B0 = 1/2 + s/3 + s^2/8 + s^3/30; C0 = 1/6 + s/8 + s^2/20 + s^3/72 */
      *B = d7addc(d7mul(sg, d7addc(d7mul(sg, d7addc(d7scl(sg, 1.0 / 30.0), 1.0 / 8.0)), 1.0 / 3.0)), 0.5);
      *C = d7addc(d7mul(sg, d7addc(d7mul(sg, d7addc(d7scl(sg, 1.0 / 72.0), 1.0 / 20.0)), 1.0 / 8.0)), 1.0 / 6.0);
    } else {       /* B0 = ((s - 1) e^s + 1) / s^2; C0 = ((s^2 - 2 s + 2) e^s - 2) / (2 s^3) */
      const d7 es = d7exp(sg), s2 = d7mul(sg, sg);
      *B = d7div(d7addc(d7mul(d7addc(sg, -1.0), es), 1.0), s2);
      *C = d7div(d7addc(d7mul(d7addc(d7sub(s2, d7scl(sg, 2.0)), 2.0), es), -2.0), d7scl(d7mul(s2, sg), 2.0));
    }
    return;
  }
  const d7 th = d7sqrt(th2), sn = d7sin(th), cs = d7cos(th), h = d7sin(d7scl(th, 0.5));
  const d7 es = d7exp(sg), em = d7expm1(sg);
  const d7 h2 = d7scl(d7mul(h, h), 2.0);              /* 2 sin^2(th/2) = 1 - cos(th) */
  const d7 den = d7add(d7mul(sg, sg), th2);
  const d7 nb = d7add(d7mul(d7mul(es, sg), sn), d7mul(th, d7sub(h2, d7mul(em, cs))));
  *B = d7div(nb, d7mul(th, den));
  const d7 nc = d7add(d7mul(d7sub(d7mul(em, cs), h2), sg), d7mul(d7mul(es, sn), th));
  *C = d7div(d7sub(*A, d7div(nc, den)), th2);
}

/* A49: x = (omega0..2, upsilon0..2, sigma). exp(x) = (R, W upsilon, e^sigma),
 * R = I + a Omega + b Omega^2, a = sin(th)/th, b = 2 sin^2(th/2)/th^2 (th < 1e-4:
 * a = 1 - th^2/6, b = 1/2 - th^2/24). */
static s7 pgo_exp(const d7 *x) {
  const d7 *w = x, *u = x + 3;
  const d7 th2 = d7dot3(w, w);
  d7 a, b;
  if (th2.v < 1e-8) {
    a = d7addc(d7scl(th2, -1.0 / 6.0), 1.0);
    b = d7addc(d7scl(th2, -1.0 / 24.0), 0.5);
  } else {
    const d7 th = d7sqrt(th2), hh = d7sin(d7scl(th, 0.5));
    a = d7div(d7sin(th), th);
    b = d7div(d7scl(d7mul(hh, hh), 2.0), th2);
  }
  /* Omega = [w]x, Omega^2 = w w^T - th2 I */
  const d7 O[9] = {d7c(0.0), d7scl(w[2], -1.0), w[1], w[2], d7c(0.0), d7scl(w[0], -1.0),
                   d7scl(w[1], -1.0), w[0], d7c(0.0)};
  s7 r;
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) {
      d7 o2 = d7mul(w[i], w[j]);
      if (i == j) o2 = d7sub(o2, th2);
      d7 e = d7add(d7mul(a, O[3 * i + j]), d7mul(b, o2));
      if (i == j) e = d7addc(e, 1.0);
      r.R[3 * i + j] = e;
    }
  d7 A, B, C, wu[3], wwu[3];
  pgo_coef(th2, x[6], &A, &B, &C);
  d7cross(w, u, wu);
  d7cross(w, wu, wwu);
  for (int i = 0; i < 3; ++i) r.t[i] = d7add(d7add(d7mul(A, u[i]), d7mul(B, wu[i])), d7mul(C, wwu[i]));
  r.s = d7exp(x[6]);
  return r;
}

/* A49: log(S) = (omega, W^-1 t, ln s): v = vee(R - R^T), c = (tr R - 1)/2; if
 * |v|^2 < 4e-8 and c > 0, omega = (1/2 + |v|^2/48) v (theta/(2 sin theta) to second
 * order with sin^2 theta = |v|^2/4); else theta = atan2(|v|/2, c), omega = theta v / |v|.
 * upsilon solves W upsilon = t by Cramer's rule. Rotation angles near pi are outside
 * the reading (the residuals of an essential graph are small rotations). */
static void pgo_log(const s7 *S, d7 *x) {
  const d7 *R = S->R;
  const d7 v[3] = {d7sub(R[7], R[5]), d7sub(R[2], R[6]), d7sub(R[3], R[1])};
  const d7 c = d7scl(d7addc(d7add(d7add(R[0], R[4]), R[8]), -1.0), 0.5);
  const d7 n2 = d7dot3(v, v);
  d7 w[3];
  if (n2.v < 4e-8 && c.v > 0.0) {
    const d7 f = d7addc(d7scl(n2, 1.0 / 48.0), 0.5);
    for (int i = 0; i < 3; ++i) w[i] = d7mul(f, v[i]);
  } else {
    const d7 nv = d7sqrt(n2);
    const d7 th = d7atan2(d7scl(nv, 0.5), c);
    const d7 f = d7div(th, nv);
    for (int i = 0; i < 3; ++i) w[i] = d7mul(f, v[i]);
  }
  const d7 sg = d7log(S->s);
  const d7 th2 = d7dot3(w, w);
  d7 A, B, C;
  pgo_coef(th2, sg, &A, &B, &C);
  const d7 O[9] = {d7c(0.0), d7scl(w[2], -1.0), w[1], w[2], d7c(0.0), d7scl(w[0], -1.0),
                   d7scl(w[1], -1.0), w[0], d7c(0.0)};
  d7 W[9];
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) {
      d7 o2 = d7mul(w[i], w[j]);
      if (i == j) o2 = d7sub(o2, th2);
      d7 e = d7add(d7mul(B, O[3 * i + j]), d7mul(C, o2));
      if (i == j) e = d7add(e, A);
      W[3 * i + j] = e;
    }
  /* Cramer: u_k = det(W with column k := t) / det(W) */
  d7 det = d7c(0.0);
  {
    const d7 m0 = d7sub(d7mul(W[4], W[8]), d7mul(W[5], W[7]));
    const d7 m1 = d7sub(d7mul(W[3], W[8]), d7mul(W[5], W[6]));
    const d7 m2 = d7sub(d7mul(W[3], W[7]), d7mul(W[4], W[6]));
    det = d7add(d7sub(d7mul(W[0], m0), d7mul(W[1], m1)), d7mul(W[2], m2));
  }
  for (int k = 0; k < 3; ++k) {
    d7 Wk[9];
    for (int i = 0; i < 9; ++i) Wk[i] = W[i];
    for (int i = 0; i < 3; ++i) Wk[3 * i + k] = S->t[i];
    const d7 m0 = d7sub(d7mul(Wk[4], Wk[8]), d7mul(Wk[5], Wk[7]));
    const d7 m1 = d7sub(d7mul(Wk[3], Wk[8]), d7mul(Wk[5], Wk[6]));
    const d7 m2 = d7sub(d7mul(Wk[3], Wk[7]), d7mul(Wk[4], Wk[6]));
    const d7 dk = d7add(d7sub(d7mul(Wk[0], m0), d7mul(Wk[1], m1)), d7mul(Wk[2], m2));
    x[3 + k] = d7div(dk, det);
  }
  x[0] = w[0]; x[1] = w[1]; x[2] = w[2];
  x[6] = sg;
}

static void s7out(const s7 *S, double *o) {
  for (int i = 0; i < 9; ++i) o[i] = S->R[i].v;
  for (int i = 0; i < 3; ++i) o[9 + i] = S->t[i].v;
  o[12] = S->s.v;
}

/* plain-value exp / log (pins) */
void orc_pgo_exp(const double *x, double *S) {
  d7 xd[7];
  for (int k = 0; k < 7; ++k) xd[k] = d7c(x[k]);
  const s7 r = pgo_exp(xd);
  s7out(&r, S);
}
void orc_pgo_log(const double *S, double *x) {
  const s7 Sd = s7c(S);
  d7 xd[7];
  pgo_log(&Sd, xd);
  for (int k = 0; k < 7; ++k) x[k] = xd[k].v;
}

/* A50: residual of edge (i, j) with measurement M (= S_j S_i^-1 when the edge was
 * made): e = log(M o S_i o S_j^-1), identity information; left-multiplicative
 * updates S <- exp(delta) o S. which = 0 seeds delta_i, 1 seeds delta_j (seven unit
 * seed directions, evaluated at delta = 0). */
static void pgo_edge_dual(const double *M, const double *Si, const double *Sj, int which, d7 *e) {
  d7 x[7];
  for (int k = 0; k < 7; ++k) { x[k] = d7c(0.0); x[k].d[k] = 1.0; }
  const s7 E = pgo_exp(x);
  const s7 Md = s7c(M);
  s7 SI = s7c(Si), SJ = s7c(Sj);
  if (which == 0) SI = s7compose(&E, &SI);
  else SJ = s7compose(&E, &SJ);
  const s7 SJi = s7inverse(&SJ);
  const s7 T1 = s7compose(&Md, &SI);
  const s7 T = s7compose(&T1, &SJi);
  pgo_log(&T, e);
}

/* e[7], Ji[7][7], Jj[7][7] row-major: J[r][k] = d e_r / d delta_k */
void orc_pgo_edge(const double *M, const double *Si, const double *Sj, double *e, double *Ji, double *Jj) {
  d7 ea[7], eb[7];
  pgo_edge_dual(M, Si, Sj, 0, ea);
  pgo_edge_dual(M, Si, Sj, 1, eb);
  for (int r = 0; r < 7; ++r) {
    e[r] = ea[r].v;
    for (int k = 0; k < 7; ++k) {
      Ji[7 * r + k] = ea[r].d[k];
      Jj[7 * r + k] = eb[r].d[k];
    }
  }
}

typedef struct {
  int32_t max_iter, cg_max_iter;
  double lambda0, eps_dx, eps_chi2, cg_tol;
} orc_pgo_params;

/* chi2 = sum over edges (ascending) of e^T e (r ascending) */
static double pgo_chi2(int32_t n_e, const int32_t *eij, const double *M, const double *S) {
  double chi2 = 0.0;
  for (int32_t k = 0; k < n_e; ++k) {
    const int32_t i = eij[2 * k], j = eij[2 * k + 1];
    const s7 Md = s7c(M + 13 * (size_t)k), SI = s7c(S + 13 * (size_t)i), SJ = s7c(S + 13 * (size_t)j);
    const s7 SJi = s7inverse(&SJ);
    const s7 T1 = s7compose(&Md, &SI);
    const s7 T = s7compose(&T1, &SJi);
    d7 e[7];
    pgo_log(&T, e);
    double c = 0.0;
    for (int r = 0; r < 7; ++r) c += e[r].v * e[r].v;
    chi2 += c;
  }
  return chi2;
}

/* A51: dense LDL^T of the N x N symmetric matrix A (lower triangle used), no pivoting;
 * fails (returns 0) when a pivot is not > 0 (not SPD). Solves A x = r. */
static int ldlt_solve(int64_t N, const double *A, const double *r, double *x) {
  double *L = (double *)calloc((size_t)(N * N > 0 ? N * N : 1), sizeof(double));
  double *D = (double *)calloc((size_t)(N > 0 ? N : 1), sizeof(double));
  int ok = 1;
  for (int64_t j = 0; j < N && ok; ++j) {
    double dj = A[j * N + j];
    for (int64_t k = 0; k < j; ++k) dj -= L[j * N + k] * L[j * N + k] * D[k];
    if (!(dj > 0.0)) { ok = 0; break; }
    D[j] = dj;
    L[j * N + j] = 1.0;
    for (int64_t i = j + 1; i < N; ++i) {
      double a = A[i * N + j];
      for (int64_t k = 0; k < j; ++k) a -= L[i * N + k] * L[j * N + k] * D[k];
      L[i * N + j] = a / dj;
    }
  }
  if (ok) {
    for (int64_t i = 0; i < N; ++i) {      /* L y = r */
      double y = r[i];
      for (int64_t k = 0; k < i; ++k) y -= L[i * N + k] * x[k];
      x[i] = y;
    }
    for (int64_t i = 0; i < N; ++i) x[i] /= D[i];
    for (int64_t i = N - 1; i >= 0; --i) { /* L^T x = z */
      double y = x[i];
      for (int64_t k = i + 1; k < N; ++k) y -= L[k * N + i] * x[k];
      x[i] = y;
    }
  }
  free(L);
  free(D);
  return ok;
}

/* A52/A53: Levenberg-Marquardt over the free vertices (fixed vertices are excluded
 * from the reduced system). Each iteration: (re)linearise after an accepted step --
 * H = sum_e J^T J, b = sum_e J^T e accumulated in ascending edge order --, solve
 * (H + lambda diag(H)) delta = -b by LDL^T; a failed factorisation multiplies lambda
 * by 4; |delta| < eps_dx stops; else the trial S_v' = exp(delta_v) o S_v is accepted
 * iff chi2' < chi2 (lambda <- max(lambda/2, 1e-12); stop when (chi2 - chi2')/chi2 <
 * eps_chi2), otherwise lambda <- 4 lambda. lambda > 1e8 stops; so does max_iter.
 * chi2 == 0 at the start stops before any solve. trace [max_iter][6]: chi2, lambda,
 * chi2 trial (-1: solve failed; chi2 when |delta| stopped), accepted, |delta|, solver
 * iterations (1 = one direct solve). stop codes: 1 |delta|, 2 chi2 change, 3 max_iter,
 * 4 lambda, 5 zero chi2. */
int orc_pgo(int32_t n_v, const double *S_in, const uint8_t *fixed, int32_t n_e, const int32_t *eij,
            const double *M, const orc_pgo_params *p, double *out_S, double *trace, double *chi2_out,
            int64_t *cnt) {
  int32_t *fidx = (int32_t *)malloc(sizeof(int32_t) * (size_t)(n_v > 0 ? n_v : 1));
  int64_t nf = 0;
  for (int32_t v = 0; v < n_v; ++v) fidx[v] = fixed[v] ? -1 : (int32_t)nf++;
  const int64_t N = 7 * nf;
  double *S = out_S;
  memcpy(S, S_in, sizeof(double) * 13 * (size_t)n_v);
  double *St = (double *)malloc(sizeof(double) * 13 * (size_t)(n_v > 0 ? n_v : 1));
  double *H = (double *)calloc((size_t)(N * N > 0 ? N * N : 1), sizeof(double));
  double *A = (double *)malloc(sizeof(double) * (size_t)(N * N > 0 ? N * N : 1));
  double *b = (double *)calloc((size_t)(N > 0 ? N : 1), sizeof(double));
  double *nb = (double *)malloc(sizeof(double) * (size_t)(N > 0 ? N : 1));
  double *dx = (double *)malloc(sizeof(double) * (size_t)(N > 0 ? N : 1));
  double chi2 = pgo_chi2(n_e, eij, M, S);
  if (chi2_out) chi2_out[0] = chi2;
  double lambda = p->lambda0;
  int stop = chi2 == 0.0 ? 5 : 0, relin = 1;
  int32_t it = 0;
  while (!stop) {
    if (it >= p->max_iter) { stop = 3; break; }
    if (relin) {
      memset(H, 0, sizeof(double) * (size_t)(N * N));
      memset(b, 0, sizeof(double) * (size_t)N);
      for (int32_t k = 0; k < n_e; ++k) {
        const int32_t i = eij[2 * k], j = eij[2 * k + 1];
        double e[7], J[2][49];
        orc_pgo_edge(M + 13 * (size_t)k, S + 13 * (size_t)i, S + 13 * (size_t)j, e, J[0], J[1]);
        const int32_t vv[2] = {i, j};
        for (int a = 0; a < 2; ++a) {
          if (fidx[vv[a]] < 0) continue;
          const int64_t ra = 7 * (int64_t)fidx[vv[a]];
          for (int r = 0; r < 7; ++r) {
            double g = 0.0;
            for (int q = 0; q < 7; ++q) g += J[a][7 * q + r] * e[q];
            b[ra + r] += g;
          }
          for (int c2 = 0; c2 < 2; ++c2) {
            if (fidx[vv[c2]] < 0) continue;
            const int64_t rc = 7 * (int64_t)fidx[vv[c2]];
            for (int r = 0; r < 7; ++r)
              for (int cc = 0; cc < 7; ++cc) {
                double h = 0.0;
                for (int q = 0; q < 7; ++q) h += J[a][7 * q + r] * J[c2][7 * q + cc];
                H[(ra + r) * N + rc + cc] += h;
              }
          }
        }
      }
      relin = 0;
    }
    memcpy(A, H, sizeof(double) * (size_t)(N * N));
    for (int64_t k = 0; k < N; ++k) A[k * N + k] = H[k * N + k] + lambda * H[k * N + k];
    for (int64_t k = 0; k < N; ++k) nb[k] = -b[k];
    const int ok = ldlt_solve(N, A, nb, dx);
    double *row = trace ? trace + 6 * (size_t)it : NULL;
    ++it;
    cnt[C_PGO_ITERS]++;
    if (row) { row[0] = chi2; row[1] = lambda; row[2] = -1.0; row[3] = 0.0; row[4] = -1.0; row[5] = 1.0; }
    if (!ok) {
      lambda *= 4.0;
      if (lambda > 1e8) stop = 4;
      continue;
    }
    double dn = 0.0;
    for (int64_t k = 0; k < N; ++k) dn += dx[k] * dx[k];
    dn = sqrt(dn);
    if (row) row[4] = dn;
    if (dn < p->eps_dx) {
      if (row) row[2] = chi2;
      stop = 1;
      break;
    }
    for (int32_t v = 0; v < n_v; ++v) {
      if (fidx[v] < 0) { memcpy(St + 13 * (size_t)v, S + 13 * (size_t)v, sizeof(double) * 13); continue; }
      double E[13];
      orc_pgo_exp(dx + 7 * (int64_t)fidx[v], E);
      orc_sim3_compose(E, S + 13 * (size_t)v, St + 13 * (size_t)v);
    }
    const double chi2t = pgo_chi2(n_e, eij, M, St);
    if (row) row[2] = chi2t;
    if (chi2t < chi2) {
      if (row) row[3] = 1.0;
      cnt[C_PGO_ACCEPTED]++;
      const double rel = (chi2 - chi2t) / chi2;
      memcpy(S, St, sizeof(double) * 13 * (size_t)n_v);
      chi2 = chi2t;
      lambda = lambda * 0.5 < 1e-12 ? 1e-12 : lambda * 0.5;
      relin = 1;
      if (rel < p->eps_chi2) stop = 2;
    } else {
      lambda *= 4.0;
      if (lambda > 1e8) stop = 4;
    }
  }
  cnt[C_PGO_SOLVER_ITERS] += it;
  cnt[C_PGO_STOP] = stop;
  if (chi2_out) chi2_out[1] = chi2;
  free(fidx); free(St); free(H); free(A); free(b); free(nb); free(dx);
  return 0;
}

int32_t orc_ncount(void) { return C_N; }
