// k_match.cu -- projection + windowed Hamming matching, per-feature conflict
// resolution, orientation filter and fusion apply.
//
// PAPER.md:217 (§IV.D.1): "Each GPU thread handles the projection and matching
// operations for a single map point"; PAPER.md:228 (§IV.D.3): loop fusion over
// mutually independent connected keyframes. B200 design:
// one CTA per (keyframe, query chunk); the keyframe's cell-major keypoints,
// octaves and grid offsets are staged in shared memory once per CTA together
// with a hash of the map points the keyframe already holds; every thread owns
// one query (64-B map-point record gather, fp64 projection + culls, candidate
// scan over the staged cells, 2 x uint4 descriptor loads + 8 POPC per
// candidate); per-feature winners are resolved with a 64-bit atomicMin on
// (H << 32) | q, which is the lowest-(H, q) rule of reading A17.
#include <cuda_runtime.h>

#include <algorithm>

#include "lc_internal.cuh"

namespace {

constexpr unsigned long long NONE = 0x7FFFFFFFFFFFFFFFull;

// local per-thread counters of the matching kernel (subset of LC_COUNT_*)
enum { M_QUERIES, M_BAD, M_FOUND, M_DEPTH, M_BOUNDS, M_DIST, M_ANGLE, M_CAND, M_NOCAND,
       M_OVERTH, M_RATIO, M_PROP, M_N };
__device__ __constant__ int kProjSlot[8] = {
    LC_COUNT_QUERIES, LC_COUNT_SKIP_BAD, LC_COUNT_SKIP_FOUND, LC_COUNT_CULL_DEPTH,
    LC_COUNT_CULL_BOUNDS, LC_COUNT_CULL_DIST, LC_COUNT_CULL_ANGLE, LC_COUNT_EDGE_AMB};
__device__ __constant__ int kMatchSlot2[6] = {LC_COUNT_CANDIDATES, LC_COUNT_NO_CAND,
                                              LC_COUNT_OVER_TH, LC_COUNT_RATIO_REJ,
                                              LC_COUNT_PROPOSALS, LC_COUNT_EDGE_AMB};

// edge-ambiguity (the oracle's flag, same fp64 expressions): a bounds
// or window decision within 1e-4 px of the edge
constexpr double kEdgeEps = 1e-4;
constexpr uint32_t kSurvEdge = 1u << 30;   // Surv.jl bit: the query's bounds decision was
__device__ __forceinline__ bool bounds_edge(const DevCam& c, double u, double v) {
  return fabs(u - c.min_x) < kEdgeEps || fabs(u - c.max_x) < kEdgeEps || fabs(v - c.min_y) < kEdgeEps ||
         fabs(v - c.max_y) < kEdgeEps;
}
__device__ __forceinline__ bool window_edge(double du, double dv, double r) {
  return du < r + kEdgeEps && dv < r + kEdgeEps && (du > r - kEdgeEps || dv > r - kEdgeEps);
}


// Reduce per-thread counters over the block and add them to global memory.
template <int N>
__device__ __forceinline__ void block_add(const uint32_t (&loc)[N], const int* slots,
                                          unsigned long long* gdst) {
  __shared__ unsigned int s_acc[32];
  if (threadIdx.x < 32) s_acc[threadIdx.x] = 0;
  __syncthreads();
#pragma unroll
  for (int i = 0; i < N; ++i) {
    uint32_t v = loc[i];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
    if ((threadIdx.x & 31) == 0 && v) atomicAdd(&s_acc[i], v);
  }
  __syncthreads();
  if (threadIdx.x < N && s_acc[threadIdx.x])
    atomicAdd(&gdst[slots[threadIdx.x]], (unsigned long long)s_acc[threadIdx.x]);
}

__device__ __forceinline__ int popc_desc(const uint4& a0, const uint4& a1, const uint4& b0,
                                         const uint4& b1) {
  return __popc(a0.x ^ b0.x) + __popc(a0.y ^ b0.y) + __popc(a0.z ^ b0.z) + __popc(a0.w ^ b0.w) +
         __popc(a1.x ^ b1.x) + __popc(a1.y ^ b1.y) + __popc(a1.z ^ b1.z) + __popc(a1.w ^ b1.w);
}

// ---------------------------------------------------------------------------
// TMA (cp.async.bulk) + mbarrier helpers
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes) : "memory");
}
__device__ __forceinline__ void tma_load_1d(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_wait2() {   // all but the 2 newest groups
  asm volatile("cp.async.wait_group 2;" ::: "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() {
  asm volatile("cp.async.commit_group;\n cp.async.wait_group 0;" ::: "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
  uint32_t done = 0;
  while (!done) {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
        " selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(done)
        : "r"(smem_u32(bar)), "r"(phase)
        : "memory");
  }
}


// ---------------------------------------------------------------------------
// Loop fusion / projection search in two kernels over the same (unit, query chunk)
// blocks (unit = keyframe for fuse, (keyframe, Sim3, params) pair for SBP):
//
// k_project ("each GPU thread handles the projection ... for a single
//   map point"): thread per query. List entry -> {flags, first 32-B sector of the
//   64-B map-point record}; already-found test against a shared-memory hash of the
//   keyframe's associations; fp64 SE3 projection and culls in the order of the
//   definition (division-free conservative pre-tests decide the bounds and lower
//   distance culls when the value is farther from the bound than a margin >> fp64
//   rounding; the exact expression otherwise); level prediction (float guess,
//   exact fp64 adjustment). Survivors are warp-aggregated into the block's region
//   of a global survivor buffer (L2-resident between the two launches).
// k_match: CTA per block; one elected thread stages the keyframe's cell offsets,
//   keypoints and octave/index words with three 1-D TMA bulk copies on an mbarrier;
//   each warp takes 32 survivors at a time: (1) lane-serial scan of the window's
//   cells in shared memory (octave test + fp32-filtered exact square-window test)
//   recording candidate positions; (2) warp-wide Hamming distances of all recorded
//   candidates (one 32-B descriptor sector each, query words by shuffle);
//   (3) per-lane best = min (H << 16 | f), second = min H of the rest, proposal =
//   u64 atomicMin on (H << 32) | q. In sole mode (one block per unit) the CTA then
//   resolves its unit (orientation + fuse actions) without another launch.
// ---------------------------------------------------------------------------
template <int MODE>
__device__ void resolve_unit(const MatchArgs& a, int unit);

constexpr int NWARP = LC_NTHREADS / 32;
#ifndef LC_KM_MINB
#define LC_KM_MINB 3      // k_match CTAs per SM the register budget is cut for
#endif
#ifndef LC_KM_B
#define LC_KM_B 2         // k_match window scan: features per batch of shared-memory loads
#endif
#ifndef LC_KP_MINB
#define LC_KP_MINB 4      // k_project CTAs per SM the register budget is cut for
#endif
#ifndef LC_KM_PF
#define LC_KM_PF 0        // L1 prefetch of a candidate's descriptor when it is recorded
#endif
constexpr int CPL = 6;            // candidate slots per survivor (more -> serial fallback)

__device__ __forceinline__ uint32_t hslot(int32_t key, uint32_t size) {
  return (uint32_t)(((uint64_t)((uint32_t)key * 2654435769u) * size) >> 32);
}
__device__ __forceinline__ void hins(int32_t* tab, uint32_t size, int32_t key) {
  uint32_t h = hslot(key, size);
  while (true) {
    int32_t prev = atomicCAS(&tab[h], -1, key);
    if (prev == -1 || prev == key) return;
    h = (h + 1 == size) ? 0 : h + 1;
  }
}
__device__ __forceinline__ bool hhas(const int32_t* tab, uint32_t size, int32_t key) {
  uint32_t h = hslot(key, size);
  while (true) {
    int32_t v = tab[h];
    if (v == key) return true;
    if (v == -1) return false;
    h = (h + 1 == size) ? 0 : h + 1;
  }
}

// fp32 window-filter margin (px): |fuv - fu| in fp32 is within 2.5e-4 (rounding of the
// exact u to fp32) + 4.9e-4 (fp32 subtraction at |u| < 4096) px of the exact distance
constexpr float kWinTol = 1e-3f;

template <int FCAP>
struct HashSize {
  static constexpr int HS = ((2 * FCAP + 1) + 31) & ~31;   // load factor <= 0.5
};
// membership pre-filter over the keyframe's associations: 2^15 bits, one hash
// (a miss -- the common case -- costs one shared-memory load instead of a probe run)
constexpr int FILT_LOG2 = 15;
__device__ __forceinline__ uint32_t fslot(int32_t key) {
  return ((uint32_t)key * 0x85EBCA6Bu) >> (32 - FILT_LOG2);
}

// exact fp64 projection of a culled query only to decide its edge flag (rare)
__device__ __noinline__ bool edge_exact(const DevCam& cam, double x, double y, double z) {
  double u, v;
  lc_project(cam, x, y, z, u, v);
  return bounds_edge(cam, u, v);
}

// the definition's expressions (oracle O4 steps 5-8): d = sqrt(s), distance range, view
// angle, smallest n with d * s_n >= dmax
__device__ __noinline__ int dal_exact(double sq, double g, double dmax, double sLm1, const double* scale,
                                      int L, int& lvl) {
  const double d = sqrt(sq);
  if (d < 0.8 * (dmax / sLm1) || d > 1.2 * dmax) return LC_Q_DIST;
  if (g < 0.5 * d) return LC_Q_ANGLE;
  lvl = L - 1;
  for (int n = 0; n < L; ++n)
    if (d * scale[n] >= dmax) { lvl = n; break; }
  return 1;
}

// distance / angle / level from s = |PO|^2 and g = PO . n: 1 (kept, lvl set), LC_Q_DIST or
// LC_Q_ANGLE; identical decisions to dal_exact (which it calls inside the bands)
__device__ __forceinline__ int dist_angle_level(double sq, double g, double dmax, double c08, double sLm1,
                                                const double* scale, const double* scale2, int L, float inv_lsf,
                                                int& lvl) {
  const double hi = 1.2 * dmax, hi2 = hi * hi;
  const double lo = dmax * c08, lo2 = lo * lo;   // lo within a few ulp of 0.8 * (dmax / s_{L-1})
  if (sq > hi2 * (1.0 + 1e-12) || sq < lo2 * (1.0 - 1e-9)) return LC_Q_DIST;
  if (!(sq < hi2 * (1.0 - 1e-12)) || !(sq > lo2 * (1.0 + 1e-9))) return dal_exact(sq, g, dmax, sLm1, scale, L, lvl);
  if (g < 0.0) return LC_Q_ANGLE;   // 0.5 * d >= 0 > g
  const double g2 = g * g, q4 = 0.25 * sq;
  if (g2 < q4 * (1.0 - 1e-12)) return LC_Q_ANGLE;
  if (!(g2 > q4 * (1.0 + 1e-12))) return dal_exact(sq, g, dmax, sLm1, scale, L, lvl);
  // level: d * s_n >= dmax  <=>  s * s_n^2 >= dmax^2 outside the band
  const double dm2 = dmax * dmax, dm2h = dm2 * (1.0 + 1e-12), dm2l = dm2 * (1.0 - 1e-12);
  int n = (int)ceilf(0.5f * __logf((float)dm2 / (float)sq) * inv_lsf);
  n = min(max(n, 0), L - 1);
  auto cmp = [&](int k) -> int {   // 1 true, 0 false, -1 inside the band (scale2[k] = scale[k]^2)
    const double t = sq * scale2[k];
    if (t > dm2h) return 1;
    if (t < dm2l) return 0;
    return -1;
  };
  while (n > 0) {
    const int c = cmp(n - 1);
    if (c < 0) return dal_exact(sq, g, dmax, sLm1, scale, L, lvl);
    if (!c) break;
    --n;
  }
  while (n < L - 1) {
    const int c = cmp(n);
    if (c < 0) return dal_exact(sq, g, dmax, sLm1, scale, L, lvl);
    if (c) break;
    ++n;
  }
  lvl = n;
  return 1;
}

// ---- k_project ---------------------------------------------------------------
template <int MODE, int FCAP>
__global__ void __launch_bounds__(LC_NTHREADS, LC_KP_MINB) k_project(const MatchArgs a) {
  constexpr uint32_t HS = (uint32_t)HashSize<FCAP>::HS;
  extern __shared__ __align__(16) int32_t s_hash[];   // [HS] (dynamic: up to 64 KB)
  __shared__ __align__(16) uint32_t s_filt[1 << (FILT_LOG2 - 5)];
  __shared__ double s_T[12];
  __shared__ double s_Ow[3];
  __shared__ double s_scale[LC_MAX_LEVELS], s_scale2[LC_MAX_LEVELS];
  __shared__ DevCam s_cam;
  __shared__ double s_box[4];   // image centre x, half width, centre y, half height
  __shared__ int s_cnt;
  const int tid = threadIdx.x;
  const int lane = tid & 31;
  const unsigned ltmask = (1u << lane) - 1u;
  const int blk = a.blk_base + (int)blockIdx.x;
  const int unit = a.blk_unit[blk];
  const int k = a.unit_kf[unit];
  const int fb = a.kf_fbeg[k];
  const int F = a.kf_fbeg[k + 1] - fb;
  const int64_t toff = (MODE == 1 && a.taken) ? a.unit_toff[unit] : 0;
  if (tid == 0) {
    double S[13], T[13];
    const double* src = a.unit_S ? a.unit_S + 13 * (size_t)unit : a.kf_S_corr + 13 * (size_t)k;
    for (int i = 0; i < 13; ++i) S[i] = src[i];
    lc_sim3_se3(S, T);  // reading A2: project with (R, t/s)
    for (int i = 0; i < 12; ++i) s_T[i] = T[i];
    for (int i = 0; i < 3; ++i) s_Ow[i] = -lc_col3(T, i, T + 9);
    s_cam = a.cams[a.kf_cam[k]];
    s_box[0] = 0.5 * (s_cam.min_x + s_cam.max_x);
    s_box[1] = 0.5 * (s_cam.max_x - s_cam.min_x);
    s_box[2] = 0.5 * (s_cam.min_y + s_cam.max_y);
    s_box[3] = 0.5 * (s_cam.max_y - s_cam.min_y);
    s_cnt = 0;
  }
  // software pipeline: the 32-B record (geometry sector) of the query two steps ahead
  // is copied by cp.async into a per-thread 3-slot ring behind the hash (no registers
  // held), its flag and the list entry three steps ahead are in flight in registers.
  // The prologue is issued before the association hash is built, so the first records'
  // latency overlaps the setup (the ring does not alias the hash).
  const int64_t q0 = a.blk_q0[blk], q1 = a.blk_q1[blk];
  uint4* s_rec = reinterpret_cast<uint4*>(s_hash + HS);   // [3][LC_NTHREADS][2]
  auto list_at = [&](int64_t jj) -> int32_t { return jj < q1 ? __ldg(a.mp_list + jj) : -1; };
  auto flag_at = [&](int32_t qq) -> uint8_t {
    return (unsigned)qq < (unsigned)a.n_mp ? __ldg(a.mp_flags + qq) : (uint8_t)1;
  };
  auto issue = [&](int32_t qq, int slot) {
    if ((unsigned)qq < (unsigned)a.n_mp) {
      const uint4* rp = reinterpret_cast<const uint4*>(a.mp_rec + qq);
      uint4* d = s_rec + 2 * (slot * LC_NTHREADS + tid);
      cp_async16(d, rp);
      cp_async16(d + 1, rp + 1);
    }
    cp_async_commit();   // one group per step, empty or not
  };
  int32_t qa = list_at(q0 + tid), qb = list_at(q0 + tid + LC_NTHREADS);
  int32_t qc = list_at(q0 + tid + 2 * LC_NTHREADS);
  uint8_t fa = flag_at(qa), fbl = flag_at(qb);
  issue(qa, 0);
  issue(qb, 1);
  if (tid < LC_MAX_LEVELS) {
    s_scale[tid] = a.scale[tid];
    s_scale2[tid] = a.scale[tid] * a.scale[tid];
  }
  // (16-B stores: HS is a multiple of 32, the filter 1024 words)
  for (int i = tid; i < (int)HS / 4; i += LC_NTHREADS) reinterpret_cast<int4*>(s_hash)[i] = make_int4(-1, -1, -1, -1);
  for (int i = tid; i < (1 << (FILT_LOG2 - 5)) / 4; i += LC_NTHREADS)
    reinterpret_cast<uint4*>(s_filt)[i] = make_uint4(0u, 0u, 0u, 0u);
  __syncthreads();
  // the keyframe's associations: 8 loads per thread in flight, then the inserts
  const int32_t* assoc = (MODE == 0) ? a.feat_mp + fb : (a.taken ? a.taken + toff : nullptr);
  if (assoc) {
    for (int f0 = tid; f0 < F; f0 += 8 * LC_NTHREADS) {
      int32_t m[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int f = f0 + u * LC_NTHREADS;
        m[u] = f < F ? __ldg(assoc + f) : -1;
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        if (m[u] >= 0) {
          const uint32_t b = fslot(m[u]);
          atomicOr(&s_filt[b >> 5], 1u << (b & 31));
          hins(s_hash, HS, m[u]);
        }
      }
    }
  }
  __syncthreads();
  const int L = a.n_levels;
  const double sLm1 = a.scale[L - 1];
  const double c08 = 0.8 / sLm1;   // for the division-free pre-test only
  const bool pinhole = s_cam.model == 0;
  const float inv_lsf = 1.0f / logf((float)a.scale[1]);
  const int64_t qbase = a.unit_qoff[unit] + (q0 - a.unit_lbeg[unit]);
  Surv* out = a.surv + a.surv_off[blk];
  uint32_t cA = 0, cB = 0;   // packed 10-bit counters (<= 1023 queries per thread per block)
  uint32_t cE = 0;                   // edge-ambiguous culled queries (survivors: flag to k_match)
  const bool dbg_any = a.dbg_best || a.dbg_uv || a.dbg_ncand;
  int slot = 0;
  for (int64_t jb = q0; jb < q1; jb += LC_NTHREADS, slot = slot == 2 ? 0 : slot + 1) {
    const int64_t j = jb + tid;
    const bool valid = j < q1;
    const int32_t q = qa;
    const uint8_t flag = fa;
    issue(qc, slot == 0 ? 2 : slot - 1);   // slot of step + 2
    const uint8_t fc = flag_at(qc);
    const int32_t qd = list_at(j + 3 * LC_NTHREADS);
    cp_async_wait2();                      // this step's record is in
    const uint4 r0 = s_rec[2 * (slot * LC_NTHREADS + tid)];
    const uint4 r1 = s_rec[2 * (slot * LC_NTHREADS + tid) + 1];
    qa = qb; fa = fbl; qb = qc; fbl = fc; qc = qd;
    const bool in_range = valid && (unsigned)q < (unsigned)a.n_mp;
    // LoopSet stamp with the host-known epoch (eager calls; prep does not touch loop_ep
    // here and nothing reads it before k_match's wait)
    if (a.stamp_epoch && in_range) a.loop_ep_w[q] = a.stamp_epoch;
    int status = 0;
    float fu = 0.f, fv = 0.f;
    int lvl = 0;
    bool edge = false;
    if (valid) {
      do {
        if (!in_range || (flag & 1u)) { status = LC_Q_BAD; cA += 1u; break; }
        const uint32_t fb2 = fslot(q);
        if (((s_filt[fb2 >> 5] >> (fb2 & 31)) & 1u) && hhas(s_hash, HS, q)) {
          status = LC_Q_FOUND; cA += 1u << 10; break;
        }
        const double p0 = __uint_as_float(r0.x), p1 = __uint_as_float(r0.y), p2 = __uint_as_float(r0.z);
        double x, y, z;
        lc_se3_xyz(s_T, p0, p1, p2, x, y, z);
        if (z <= 0.0) { status = LC_Q_DEPTH; cA += 1u << 20; break; }
        bool exact = !pinhole || a.dbg_uv;
        if (!exact) {
          // conservative pre-test: |ua - u| <= 1e-6 |u| + tiny, margin 1e-2 px
          const double rz = (double)__frcp_rn((float)z);
          const double A = s_cam.fx * x, B = s_cam.fy * y;
          const double e = 1e-6 * (fabs(A * rz) + fabs(B * rz)) + 1e-2;
          const double ua = A * rz * (2.0 - z * rz) + s_cam.cx;   // one Newton step
          const double va = B * rz * (2.0 - z * rz) + s_cam.cy;
          const double e2 = e + kEdgeEps;
          // distances from the image centre against the half extents (s_box): the same
          // certain decisions as against each bound (up to an ulp, inside the margin e;
          // a value exactly on a shifted bound goes to the exact path)
          const double ax = fabs(ua - s_box[0]), ay = fabs(va - s_box[2]);
          if (ax > s_box[1] + e || ay > s_box[3] + e) {
            // certainly culled; edge-ambiguous only if u or v is within 1e-4 px of a
            // bound, which needs ua or va within e + 1e-4 of one: decide exactly then
            if (fabs(ax - s_box[1]) < e2 || fabs(ay - s_box[3]) < e2) cE += edge_exact(s_cam, x, y, z) ? 1u : 0u;
            status = LC_Q_BOUNDS; cB += 1u; break;
          }
          if (ax < s_box[1] - e2 && ay < s_box[3] - e2) {
            // certainly inside and no bound within 1e-4 px: the fp32 survivor pixel is
            // taken from the refined estimate (|ua - u| << the fp32 window tolerance)
            fu = (float)ua; fv = (float)va;
          } else {
            exact = true;
          }
        }
        if (exact) {
          double u, v;
          lc_project(s_cam, x, y, z, u, v);
          edge = bounds_edge(s_cam, u, v);   // SURVEY §8(c) edge-ambiguous (oracle: before the cull)
          if (a.dbg_uv) {   // (survivors: k_match writes the same exact values again)
            const int64_t qi = qbase + (j - q0);
            a.dbg_uv[2 * qi] = u; a.dbg_uv[2 * qi + 1] = v;
          }
          if (!(u >= s_cam.min_x && u < s_cam.max_x && v >= s_cam.min_y && v < s_cam.max_y)) {
            status = LC_Q_BOUNDS; cB += 1u; break;
          }
          fu = (float)u; fv = (float)v;
        }
        // distance range, view angle, level (readings A5-A7) decided on s = |PO|^2 with
        // relative bands (1e-12, 1e-9) far wider than any rounding; the definition's exact
        // expressions (with the square root) only when a value falls inside a band
        const double PO0 = p0 - s_Ow[0], PO1 = p1 - s_Ow[1], PO2 = p2 - s_Ow[2];
        const double sq = (PO0 * PO0 + PO1 * PO1) + PO2 * PO2;
        const double dmax = __uint_as_float(r0.w);
        const double n0 = __uint_as_float(r1.x), n1 = __uint_as_float(r1.y), n2 = __uint_as_float(r1.z);
        const double g = (PO0 * n0 + PO1 * n1) + PO2 * n2;
        const int st = dist_angle_level(sq, g, dmax, c08, sLm1, s_scale, s_scale2, L, inv_lsf, lvl);
        if (st == LC_Q_DIST) { status = LC_Q_DIST; cB += 1u << 10; break; }
        if (st == LC_Q_ANGLE) { status = LC_Q_ANGLE; cB += 1u << 20; break; }
        status = 1;
      } while (0);
    }
    const bool surv = status == 1;
    const unsigned m = __ballot_sync(0xffffffffu, surv);
    int wbase = 0;
    if (lane == 0 && m) wbase = atomicAdd(&s_cnt, __popc(m));
    wbase = __shfl_sync(0xffffffffu, wbase, 0);
    if (surv) {
      Surv e;
      e.q = q; e.jl = (uint32_t)(j - q0) | ((uint32_t)lvl << 27) | (edge ? kSurvEdge : 0u);
      e.fu = fu; e.fv = fv;
      out[wbase + __popc(m & ltmask)] = e;
    } else if (valid) {
      cE += edge ? 1u : 0u;
      if (dbg_any) {
        const int64_t qi = qbase + (j - q0);
        if (a.dbg_best) a.dbg_best[qi] = status;
        if (a.dbg_uv && status > LC_Q_BOUNDS) { a.dbg_uv[2 * qi] = 0.0; a.dbg_uv[2 * qi + 1] = 0.0; }
        if (a.dbg_ncand) a.dbg_ncand[qi] = 0;
      }
    }
  }
  __syncthreads();
  if (tid == 0) a.surv_cnt[blk] = s_cnt;
  pdl_trigger();
  uint32_t cnt[8];
  cnt[0] = tid == 0 ? (uint32_t)(q1 - q0) : 0u;   // the block's queries
  cnt[1] = cA & 1023u; cnt[2] = (cA >> 10) & 1023u; cnt[3] = (cA >> 20) & 1023u;
  cnt[4] = cB & 1023u; cnt[5] = (cB >> 10) & 1023u; cnt[6] = (cB >> 20) & 1023u; cnt[7] = cE;
  unsigned long long* cdst = a.counts + (MODE == 1 ? (size_t)unit * LC_NCOUNT : 0);
  pdl_wait();   // (PDL) k_fuse_prep zeroes the counters and publishes the epoch
  if (a.loop_ep_w && !a.stamp_epoch) {   // (graph capture: the replay's epoch is on the device)
    const uint32_t epoch = *a.epoch;
    for (int64_t j = q0 + tid; j < q1; j += LC_NTHREADS) {
      const int32_t q = __ldg(a.mp_list + j);
      if ((unsigned)q < (unsigned)a.n_mp) a.loop_ep_w[q] = epoch;
    }
  }
  block_add<8>(cnt, kProjSlot, cdst);
}

// ---- k_match ------------------------------------------------------------------
template <int FCAP>
struct MatchSmem {
  // per warp: candidate keys [32][CPL] u32, candidate positions [32][CPL] u16,
  // query descriptors [32][8] u32 (cp.async destination)
  static constexpr int WKEY = 0;
  static constexpr int WCAND = WKEY + 32 * CPL * 4;
  static constexpr int WOWN = WCAND + 32 * (CPL + 1) * 2;               // (+1: overflow sink)
  static constexpr int WQD = (WOWN + 32 * CPL * 2 + 15) & ~15;
  static constexpr int WB = WQD + 32 * 32;
  static constexpr int UV = 0;
  static constexpr int META = UV + ((FCAP * 8 + 15) & ~15);
  static constexpr int QUEUE = META + ((FCAP * 4 + 15) & ~15);
  static constexpr int CELL = QUEUE + NWARP * WB;   // runtime-size cell table last
};

// exact fp64 (u, v) of a survivor: the same expressions as k_project (same bits)
__device__ __noinline__ void exact_uv(const MatchArgs& a, const double* T, const DevCam& cam,
                                         int q, double& u, double& v) {
  const MpRec* r = a.mp_rec + q;
  double x, y, z;
  lc_se3_xyz(T, (double)__ldg(&r->pos[0]), (double)__ldg(&r->pos[1]), (double)__ldg(&r->pos[2]), x, y, z);
  lc_project(cam, x, y, z, u, v);
}

// Exact fp64 window scan of one survivor over its octave grids lvl-1, lvl (readings A8,
// A9): every feature of the conservative cell ranges is tested against the exact (u, v);
// take((H << 16) | f) per candidate, edge flags accumulated. Used when the fp32 filter
// was ambiguous or a survivor overflowed its candidate slots. dsc = the keyframe's
// cell-major descriptors (global or shared memory).
template <int MODE, typename Take>
__device__ __forceinline__ void scan_exact(const MatchArgs& a, const DevCam& cam, const uint16_t* s_cell,
                                           const float2* s_uv, const uint32_t* s_meta, const uint4* dsc,
                                           float fu, float fv, float fr, int lvl, double u, double v, double r,
                                           const uint4& d0, const uint4& d1, Take& take, int& nc, bool& wedge) {
  const float fminx = (float)cam.min_x, fminy = (float)cam.min_y;
  for (int o = max(lvl - 1, 0); o <= lvl; ++o) {
    const int oc = a.ocols[o], orr = a.orows[o], ob = a.obase[o];
    const float fsx = (float)cam.cell_sx[o], fsy = (float)cam.cell_sy[o];
    const int cx0 = max(0, (int)floorf((fu - fr - 0.01f - fminx) * fsx));
    const int cx1 = min(oc - 1, (int)floorf((fu + fr + 0.01f - fminx) * fsx));
    const int cy0 = max(0, (int)floorf((fv - fr - 0.01f - fminy) * fsy));
    const int cy1 = min(orr - 1, (int)floorf((fv + fr + 0.01f - fminy) * fsy));
    for (int cy = cy0; cy <= cy1; ++cy) {
      const int pe = s_cell[ob + cy * oc + cx1 + 1];
      for (int p = s_cell[ob + cy * oc + cx0]; p < pe; ++p) {
        const uint32_t meta = s_meta[p];
        if (MODE == 1 && (meta & 0x80000000u)) continue;
        const float2 fuv = s_uv[p];
        const double du = fabs((double)fuv.x - u), dv = fabs((double)fuv.y - v);
        wedge |= window_edge(du, dv, r);
        if (!(du < r && dv < r)) continue;
        take(((uint32_t)popc_desc(d0, d1, dsc[2 * p], dsc[2 * p + 1]) << 16) | (meta & 0xFFFFu));
        ++nc;
      }
    }
  }
}

template <int MODE, int FCAP>
__global__ void __launch_bounds__(LC_NTHREADS, LC_KM_MINB) k_match(const MatchArgs a) {
  using SM = MatchSmem<FCAP>;
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ __align__(8) uint64_t s_bar;
  __shared__ double s_T[12];
  __shared__ __align__(16) DevCam s_cam;
  __shared__ float s_fr[LC_MAX_LEVELS];
  // per octave: {cols, rows, first cell, fp32 cell scale x} + fp32 cell scale y (one
  // 16-B and one 4-B shared load per octave in the scan)
  __shared__ int4 s_og[LC_MAX_LEVELS];
  __shared__ float s_fsy[LC_MAX_LEVELS];
  const int tid = threadIdx.x;
  const int lane = tid & 31, warp = tid >> 5;
  const int blk = a.blk_base + (int)blockIdx.x;
  const int unit = a.blk_unit[blk];
  const int k = a.unit_kf[unit];
  const int fb = a.kf_fbeg[k];
  const int F = a.kf_fbeg[k + 1] - fb;
  const int fp = a.kf_fpad[k];
  uint16_t* s_cell = (uint16_t*)(smem + SM::CELL);
  float2* s_uv = (float2*)(smem + SM::UV);
  uint32_t* s_meta = (uint32_t*)(smem + SM::META);
  unsigned char* wb = smem + SM::QUEUE + warp * SM::WB;
  uint32_t* s_key = (uint32_t*)(wb + SM::WKEY);     // [32][CPL] candidate keys
  uint16_t* s_cand = (uint16_t*)(wb + SM::WCAND);   // [32][CPL + 1] candidate positions
  uint16_t* s_own = (uint16_t*)(wb + SM::WOWN);     // [32 CPL] owner map of the flattened candidates
  const bool dbg_any = a.dbg_best || a.dbg_uv || a.dbg_ncand;
  uint32_t* s_qd = (uint32_t*)(wb + SM::WQD);       // [32][8] query descriptors
  const int64_t toff = (MODE == 1 && a.taken) ? a.unit_toff[unit] : 0;
  if (tid == 0) {
    mbar_init(&s_bar, 1);
    const uint32_t b_cell = (uint32_t)a.Gs * 2u;
    const uint32_t b_uv = (uint32_t)((F + 1) & ~1) * 8u;
    const uint32_t b_meta = (uint32_t)((F + 3) & ~3) * 4u;
    mbar_expect_tx(&s_bar, b_cell + (F > 0 ? b_uv + b_meta : 0u));
    tma_load_1d(s_cell, a.kf_cell + (size_t)k * a.Gs, b_cell, &s_bar);
    if (F > 0) {
      tma_load_1d(s_uv, a.fc_uv + fp, b_uv, &s_bar);
      tma_load_1d(s_meta, a.fc_meta + fp, b_meta, &s_bar);
    }
  }
  if (tid >= 32 && tid < 44) {   // SE3 part (R, t/s) of the unit's Sim3 (reading A2)
    const double* src = a.unit_S ? a.unit_S + 13 * (size_t)unit : a.kf_S_corr + 13 * (size_t)k;
    const int i = tid - 32;
    s_T[i] = i < 9 ? src[i] : src[i] / src[12];
  }
  if (tid >= 64 && tid < 64 + (int)(sizeof(DevCam) / 16)) {
    static_assert(sizeof(DevCam) % 16 == 0, "DevCam copy granularity");
    reinterpret_cast<uint4*>(&s_cam)[tid - 64] =
        reinterpret_cast<const uint4*>(a.cams + a.kf_cam[k])[tid - 64];
  }
  if (tid >= 128 && tid < 128 + LC_MAX_LEVELS) {   // per-octave grid constants, fp32 radii
    const int o = tid - 128;
    const DevCam& c = a.cams[a.kf_cam[k]];
    const lc_match_params pp = a.params[(MODE == 1 && a.unit_param) ? a.unit_param[unit] : 0];
    s_fsy[o] = (float)c.cell_sy[o];
    s_fr[o] = (float)((double)pp.th * a.scale[o]);
    s_og[o] = make_int4(a.ocols[o], a.orows[o], a.obase[o], __float_as_int((float)c.cell_sx[o]));
  }
  if (a.sole) {  // this CTA owns the unit's winner words: initialise them here
    unsigned long long* w0 = a.winner + a.unit_woff[unit];
    for (int f = tid; f < F; f += LC_NTHREADS) w0[f] = NONE;
  }
  __syncthreads();
  mbar_wait(&s_bar, 0);
  if (MODE == 1 && a.taken) {  // taken features are not candidates (reading A19)
    for (int p = tid; p < F; p += LC_NTHREADS)
      if (a.taken[toff + (s_meta[p] & 0xFFFFu)] >= 0) s_meta[p] |= 0x80000000u;
  }
  __syncthreads();

  const lc_match_params prm = a.params[(MODE == 1 && a.unit_param) ? a.unit_param[unit] : 0];
  const bool f32ok = fmax(fabs(s_cam.min_x), fabs(s_cam.max_x)) < 4096.0 &&
                     fmax(fabs(s_cam.min_y), fabs(s_cam.max_y)) < 4096.0;
  const float fminx = (float)s_cam.min_x, fminy = (float)s_cam.min_y;
  unsigned long long* win = a.winner + a.unit_woff[unit];
  const int64_t q0 = a.blk_q0[blk];
  const int64_t qbase = a.unit_qoff[unit] + (q0 - a.unit_lbeg[unit]);
  pdl_wait();   // survivors of k_project from here on
  const Surv* sv = a.surv + a.surv_off[blk];
  const int ns_tot = a.surv_cnt[blk];
  uint32_t cC = 0, cP = 0, cE = 0;   // NOCAND | OVERTH << 10 | RATIO << 20; PROP; CAND
  uint32_t cW = 0;                   // edge-ambiguous survivors

  // strict square window |fuv - uv| < r (reading A8). fp32 filter: |(float)a - fu| is
  // within 2.5e-4 px of the exact |a - u| for |u| < 4096 px, so a decision farther
  // than 1e-3 px from the edge is exact; -1 = ambiguous (decide in fp64)
  // (frp = fr + tol, frm = fr - tol per survivor; tol = +inf when fp32 cannot decide:
  // every test is then ambiguous)
  auto win_f32 = [&](const float2 fuv, float fu, float fv, float frp, float frm) -> int {
    const float dm = fmaxf(fabsf(fuv.x - fu), fabsf(fuv.y - fv));
    if (dm > frp) return 0;   // du > fr + tol || dv > fr + tol
    if (dm < frm) return 1;   // du < fr - tol && dv < fr - tol
    return -1;
  };
  const float wtol = f32ok ? kWinTol : INFINITY;

  // the next step's survivor entries are in flight while the current step runs
  Surv e_nx;
  e_nx.q = 0; e_nx.jl = 0u; e_nx.fu = 0.f; e_nx.fv = 0.f;
  if (warp * 32 + lane < ns_tot) e_nx = sv[warp * 32 + lane];
  for (int i0 = warp * 32; i0 < ns_tot; i0 += NWARP * 32) {
    const bool act = i0 + lane < ns_tot;
    const Surv e = e_nx;
    if (i0 + NWARP * 32 + lane < ns_tot) e_nx = sv[i0 + NWARP * 32 + lane];
    const int lvl = (int)((e.jl >> 27) & 7u);
    int nc = 0;
    bool wedge = false;   // edge-ambiguous query (bounds flag from k_project, or a window decision)
    const float fr = s_fr[lvl];
    if (act) {
      // query descriptor -> shared memory, asynchronously, during the scan
      const uint4* rp = reinterpret_cast<const uint4*>(a.mp_rec + e.q);
      cp_async16(s_qd + lane * 8, rp + 2);
      cp_async16(s_qd + lane * 8 + 4, rp + 3);
      wedge = (e.jl & kSurvEdge) != 0u;
      // (1) window scan over the staged cells of the octave grids lvl-1 and lvl (reading A9:
      // octave in [lvl-1, lvl]; grid o holds exactly the octave-o features), conservative
      // (0.01 px) cell ranges; slots whose fp32 window test is ambiguous are marked and
      // settled in fp64 after the scan
      uint32_t amb = 0u;
      const float frp = fr + wtol, frm = fr - wtol;
      // the window's conservative pixel range (the same fp32 expressions per octave before)
      const float ulo = e.fu - fr - 0.01f - fminx, uhi = e.fu + fr + 0.01f - fminx;
      const float vlo = e.fv - fr - 0.01f - fminy, vhi = e.fv + fr + 0.01f - fminy;
      for (int o = max(lvl - 1, 0); o <= lvl; ++o) {
        const int4 og = s_og[o];
        const int oc = og.x, orr = og.y, ob = og.z;
        const float fsx = __int_as_float(og.w), fsy = s_fsy[o];
        const int cx0 = max(0, (int)floorf(ulo * fsx));
        const int cx1 = min(oc - 1, (int)floorf(uhi * fsx));
        const int cy0 = max(0, (int)floorf(vlo * fsy));
        const int cy1 = min(orr - 1, (int)floorf(vhi * fsy));
        // two rows at a time: their feature ranges [psA, peA) and [psB, peB) walked as one
        // index range (k < nA: row A), so a lane's loop trips do not depend on whether its
        // window spans one row or two (the common cases)
        for (int cy = cy0; cy <= cy1; cy += 2) {
          const int rb = ob + cy * oc;
          const int psA = s_cell[rb + cx0], peA = s_cell[rb + cx1 + 1];
          int psB = 0, peB = 0;
          if (cy < cy1) { psB = s_cell[rb + oc + cx0]; peB = s_cell[rb + oc + cx1 + 1]; }
          const int nA = peA - psA, n = nA + (peB - psB);
          for (int k0 = 0; k0 < n; k0 += LC_KM_B) {   // LC_KM_B features' loads issued together
            uint32_t mt[LC_KM_B];
            float2 fuv[LC_KM_B];
            int pp[LC_KM_B];
#pragma unroll
            for (int t = 0; t < LC_KM_B; ++t) {
              const int kk = min(k0 + t, n - 1);
              pp[t] = kk < nA ? psA + kk : psB + (kk - nA);
              if (MODE == 1) mt[t] = s_meta[pp[t]];   // (the octave is implicit in the grid)
              fuv[t] = s_uv[pp[t]];
            }
#pragma unroll
            for (int t = 0; t < LC_KM_B; ++t) {
              if (k0 + t >= n) break;
              if (MODE == 1 && (mt[t] & 0x80000000u)) continue;
              const int w = win_f32(fuv[t], e.fu, e.fv, frp, frm);
              if (w == 0) continue;
              const int sl = min(nc, CPL);   // slot CPL: a sink for the overflow (rescanned)
              s_cand[lane * (CPL + 1) + sl] = (uint16_t)pp[t];
              amb |= (w < 0 ? 1u : 0u) << sl;
              ++nc;
            }
          }
        }
      }
      if (amb && nc <= CPL) {   // rare: one exact projection, drop slots outside the window
        double u, v;
        exact_uv(a, s_T, s_cam, e.q, u, v);
        const double r = (double)prm.th * a.scale[lvl];
        int m = 0;
        for (int i = 0; i < nc; ++i) {
          const int p = s_cand[lane * (CPL + 1) + i];
          const float2 fuv = s_uv[p];
          if ((amb >> i) & 1u) {
            const double du = fabs((double)fuv.x - u), dv = fabs((double)fuv.y - v);
            wedge |= window_edge(du, dv, r);
            if (!(du < r && dv < r)) continue;
          }
          s_cand[lane * (CPL + 1) + m++] = (uint16_t)p;
        }
        nc = m;
      }
    }
    cp_async_wait_all();
    __syncwarp();
    // (2) Hamming of all slotted candidates, warp-wide
    const bool over = act && nc > CPL;
    const int ns = (act && !over) ? nc : 0;
    int incl = ns;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += y;
    }
    const int tot2 = __shfl_sync(0xffffffffu, incl, 31);
    const int ex2 = incl - ns;
    // owner map of the flattened candidates: entry ex2 + i = (lane << 8) | i
#pragma unroll
    for (int i = 0; i < CPL; ++i)
      if (i < ns) s_own[ex2 + i] = (uint16_t)((lane << 8) | i);
    __syncwarp();
    for (int c0 = 0; c0 < tot2; c0 += 32) {
      const int c = c0 + lane;
      if (c < tot2) {
        const uint32_t oi = s_own[c];
        const int own = (int)(oi >> 8), ci = (int)(oi & 0xFFu);
        const int slot = own * CPL + ci;
        const int p = s_cand[own * (CPL + 1) + ci];
        const uint4* dp = a.fc_desc + 2 * (size_t)(fp + p);
        const uint4 b0 = __ldg(dp), b1 = __ldg(dp + 1);
        const uint4* qd = reinterpret_cast<const uint4*>(s_qd + own * 8);
        s_key[slot] = ((uint32_t)popc_desc(qd[0], qd[1], b0, b1) << 16) | (s_meta[p] & 0xFFFFu);
      }
    }
    __syncwarp();
    // (3) per-lane reduction over its own keys (serial rescan when > CPL candidates)
    if (act) {
      uint32_t best = 0xFFFFFFFFu;  // (H << 16) | f
      int second = 256;
      auto take = [&](uint32_t key) {   // branch-free: the larger key of the pair is a "rest" key
        const uint32_t hi = max(key, best);
        best = min(key, best);
        second = min(second, (int)(hi >> 16));
      };
      if (over) {   // > CPL fp32 candidates: serial rescan with the exact window test
        const uint4* qd = reinterpret_cast<const uint4*>(s_qd + lane * 8);
        const uint4 d0 = qd[0], d1 = qd[1];
        double u, v;
        exact_uv(a, s_T, s_cam, e.q, u, v);
        const double r = (double)prm.th * a.scale[lvl];
        nc = 0;
        scan_exact<MODE>(a, s_cam, s_cell, s_uv, s_meta, a.fc_desc + 2 * (size_t)fp, e.fu, e.fv, fr, lvl, u, v, r,
                         d0, d1, take, nc, wedge);
      } else {
#pragma unroll
        for (int i = 0; i < CPL; ++i)
          if (i < ns) take(s_key[lane * CPL + i]);
      }
      cE += nc;
      if (wedge) cW += 1u;
      do {
        if (nc == 0) { cC += 1u; break; }
        const int hb = (int)(best >> 16);
        if (hb > prm.max_hamming) { cC += 1u << 10; break; }
        if (prm.ratio_den > 0 && (long long)prm.ratio_den * hb > (long long)prm.ratio_num * second) {
          cC += 1u << 20; break;
        }
        cP += 1u;
        atomicMin(&win[best & 0xFFFFu], ((unsigned long long)hb << 32) | (unsigned int)e.q);
      } while (0);
      if (dbg_any) {
      const int64_t qi = qbase + (int64_t)(e.jl & 0x07FFFFFFu);   // bits 27-29 level, 30 edge
      if (a.dbg_best) {
        long long val;
        if (nc == 0) val = (256LL << 48) | (256LL << 32) | 0xFFFFFFFFLL;
        else val = ((long long)(best >> 16) << 48) | ((long long)second << 32) | (long long)(best & 0xFFFFu);
        a.dbg_best[qi] = val;
      }
      if (a.dbg_uv) {
        double u, v;
        exact_uv(a, s_T, s_cam, e.q, u, v);
        a.dbg_uv[2 * qi] = u; a.dbg_uv[2 * qi + 1] = v;
      }
      if (a.dbg_ncand) a.dbg_ncand[qi] = nc;
      }
    }
    __syncwarp();
  }
  pdl_trigger();
  uint32_t cnt[6];
  cnt[0] = cE; cnt[1] = cC & 1023u; cnt[2] = (cC >> 10) & 1023u; cnt[3] = (cC >> 20) & 1023u; cnt[4] = cP;
  cnt[5] = cW;
  unsigned long long* cdst = a.counts + (MODE == 1 ? (size_t)unit * LC_NCOUNT : 0);
  block_add<6>(cnt, kMatchSlot2, cdst);
  if (a.sole) {  // all proposals of this unit are in: resolve it here (no extra launch)
    __syncthreads();
    resolve_unit<MODE>(a, unit);
  }
}

// ---------------------------------------------------------------------------
// Per-unit resolve: orientation filter (reading A15) + fuse actions (MODE 0,
// readings O9.1, A20, A21) or output tables (MODE 1). Called by the whole CTA,
// either as the tail of a sole (one-CTA-per-unit) match CTA or by k_resolve.
// ---------------------------------------------------------------------------
enum { R_WINNERS, R_ORIENT, R_ADD, R_VICTIM, R_LOOP, R_BADSLOT, R_N };
__device__ __constant__ int kResolveSlot[R_N] = {LC_COUNT_WINNERS, LC_COUNT_ORIENT_REJ,
                                                 LC_COUNT_ADD, LC_COUNT_VICTIM_PROP,
                                                 LC_COUNT_LOOP_SKIP, LC_COUNT_BAD_SLOT};

__device__ __forceinline__ int rot_bin(float fa, float qa) {
  float rot = fa - qa;
  if (rot < 0.0f) rot += 360.0f;
  long b = lroundf(rot * (30.0f / 360.0f));
  if (b == 30) b = 0;
  return (int)b;
}

template <int MODE>
__device__ void resolve_unit(const MatchArgs& a, int unit) {
  __shared__ int s_hist[30];
  __shared__ int s_keep[3];
  const int k = a.unit_kf[unit];
  const int fb = a.kf_fbeg[k], F = a.kf_fbeg[k + 1] - fb;
  const int64_t woff = a.unit_woff[unit];
  const int64_t toff = (MODE == 1 && a.taken) ? a.unit_toff[unit] : 0;
  const lc_match_params prm = a.params[(MODE == 1 && a.unit_param) ? a.unit_param[unit] : 0];
  unsigned long long* winner = a.winner;
  const uint32_t epoch = MODE == 0 ? *a.epoch : 0u;
  uint32_t cnt[R_N];
#pragma unroll
  for (int i = 0; i < R_N; ++i) cnt[i] = 0;
  if (prm.check_orientation) {
    if (threadIdx.x < 30) s_hist[threadIdx.x] = 0;
    __syncthreads();
    for (int f = threadIdx.x; f < F; f += blockDim.x) {
      unsigned long long w = winner[woff + f];
      if (w == NONE) continue;
      int q = (int)(w & 0xFFFFFFFFull);
      atomicAdd(&s_hist[rot_bin(a.feat_angle[fb + f], a.mp_rec[q].angle)], 1);
    }
    __syncthreads();
    if (threadIdx.x == 0) {  // ComputeThreeMaxima (EXT), reading A15
      int max1 = 0, max2 = 0, max3 = 0, i1 = -1, i2 = -1, i3 = -1;
      for (int i = 0; i < 30; ++i) {
        int s = s_hist[i];
        if (s > max1) { max3 = max2; max2 = max1; max1 = s; i3 = i2; i2 = i1; i1 = i; }
        else if (s > max2) { max3 = max2; max2 = s; i3 = i2; i2 = i; }
        else if (s > max3) { max3 = s; i3 = i; }
      }
      if ((float)max2 < 0.1f * (float)max1) { i2 = -1; i3 = -1; }
      else if ((float)max3 < 0.1f * (float)max1) { i3 = -1; }
      s_keep[0] = i1; s_keep[1] = i2; s_keep[2] = i3;
    }
    __syncthreads();
  }
  // RB features per thread per pass with every load of a phase issued together:
  // (winner, association) -> orientation -> (flags, LoopSet stamp) of held slots
  constexpr int RB = 4;
  const int nt = blockDim.x;
  for (int f0 = threadIdx.x; f0 < F; f0 += RB * nt) {
    unsigned long long w[RB];
    int32_t slot[RB];
#pragma unroll
    for (int i = 0; i < RB; ++i) {
      const int f = f0 + i * nt;
      w[i] = f < F ? winner[woff + f] : NONE;
      slot[i] = (MODE == 0 && f < F) ? a.feat_mp[fb + f] : -1;
    }
    int8_t act[RB];
#pragma unroll
    for (int i = 0; i < RB; ++i) {
      act[i] = 0;
      if (w[i] != NONE) cnt[R_WINNERS]++;
    }
    if (prm.check_orientation) {
#pragma unroll
      for (int i = 0; i < RB; ++i) {
        if (w[i] == NONE) continue;
        const int f = f0 + i * nt;
        const int b = rot_bin(a.feat_angle[fb + f], a.mp_rec[(int)(w[i] & 0xFFFFFFFFull)].angle);
        if (b != s_keep[0] && b != s_keep[1] && b != s_keep[2]) {
          w[i] = NONE;
          winner[woff + f] = NONE;
          cnt[R_ORIENT]++;
          act[i] = 4;
        }
      }
    }
    if (MODE == 0) {
      uint8_t fl[RB];
      uint32_t ep[RB];
#pragma unroll
      for (int i = 0; i < RB; ++i) {
        const bool held = w[i] != NONE && slot[i] >= 0;
        fl[i] = held ? a.mp_flags[slot[i]] : 0;
        ep[i] = held ? a.loop_ep[slot[i]] : 0u;
      }
#pragma unroll
      for (int i = 0; i < RB; ++i) {
        const int f = f0 + i * nt;
        if (w[i] != NONE) {
          if (slot[i] < 0) { act[i] = 1; cnt[R_ADD]++; }
          else if (fl[i] & 1u) { act[i] = 5; cnt[R_BADSLOT]++; }
          else if (ep[i] == epoch) { act[i] = 3; cnt[R_LOOP]++; }
          else { act[i] = 2; cnt[R_VICTIM]++; atomicMin(&a.victim[slot[i]], w[i]); }
        }
        if (a.action && f < F) a.action[woff + f] = act[i];
      }
    } else {
#pragma unroll
      for (int i = 0; i < RB; ++i) {
        const int f = f0 + i * nt;
        if (f >= F) continue;
        const int t = a.taken ? a.taken[toff + f] : -1;
        if (t >= 0) { a.out_mp[woff + f] = t; a.out_dist[woff + f] = -1; }
        else if (w[i] != NONE) { a.out_mp[woff + f] = (int)(w[i] & 0xFFFFFFFFull); a.out_dist[woff + f] = (int)(w[i] >> 32); }
        else { a.out_mp[woff + f] = -1; a.out_dist[woff + f] = -1; }
      }
    }
  }
  unsigned long long* cdst = a.counts + (MODE == 1 ? (size_t)unit * LC_NCOUNT : 0);
  block_add<R_N>(cnt, kResolveSlot, cdst);
}

template <int MODE>
__global__ void __launch_bounds__(LC_NTHREADS) k_resolve(const MatchArgs a) {
  resolve_unit<MODE>(a, a.unit_base + blockIdx.x);
}

// ---------------------------------------------------------------------------
// k_match_sole: the fuse matching of a whole window keyframe in one CTA (sole mode, the
// C5 launch). The keyframe's cell table (octave grids), keypoints and index words are
// staged in shared memory by TMA; each warp then takes 32 survivors at a time in three
// converged phases:
//  A  lane = survivor: cell ranges of the octave grids lvl-1 and lvl (reading A9), the
//     features of those cells counted, a warp prefix sum, and the survivor's items
//     (owner lane, feature position) written to a per-warp queue in shared memory;
//  B  lane = item: 32 (survivor, feature) items per step -- fp32-filtered strict square
//     window (A8), the 32-B descriptor gathered and its Hamming distance taken against
//     the owner's query descriptor (cp.async-staged), the key (H << 16) | f appended to the
//     owner's slots; two steps per iteration so two gathers are in flight per lane;
//  C  lane = survivor: best / second over its slots (an exact fp64 rescan instead when a
//     window decision was fp32-ambiguous or the slots / queue overflowed), threshold,
//     ratio, proposal = 64-bit atomicMin (A17).
// The CTA then resolves its keyframe (orientation, fuse actions, victim proposals).
// ---------------------------------------------------------------------------
#ifndef LC_SOLE_NT
#define LC_SOLE_NT 256
#endif
#ifndef LC_SOLE_MINB
#define LC_SOLE_MINB 3
#endif
constexpr int SOLE_NW = LC_SOLE_NT / 32;
constexpr int SOLE_QCAP = 256;   // queued items per warp (32 survivors); beyond -> serial rescan
constexpr int SOLE_CPL = 4;      // candidate slots per survivor; beyond -> serial rescan
constexpr uint32_t kAmbKey = 1u << 31;

template <int FCAP>
struct SoleSmem {
  static constexpr int QI = 0;                       // per warp: [QCAP] u32 (owner << 16 | p)
  static constexpr int OP = QI + SOLE_QCAP * 4;      // [32] float4 (fu, fv, fr, lvl)
  static constexpr int QD = OP + 32 * 16;            // [32][8] u32 query descriptors
  static constexpr int KEY = QD + 32 * 32;           // [32][CPL] u32
  static constexpr int NC = KEY + 32 * SOLE_CPL * 4; // [32] u32
  static constexpr int WB = NC + 32 * 4;
  static constexpr int UV = SOLE_NW * WB;
  static constexpr int META = UV + FCAP * 8;
  static constexpr int CELL = META + FCAP * 4;       // runtime-size cell table last
};

template <int FCAP>
__global__ void __launch_bounds__(LC_SOLE_NT, LC_SOLE_MINB) k_match_sole(const MatchArgs a) {
  using SM = SoleSmem<FCAP>;
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ __align__(8) uint64_t s_bar;
  __shared__ double s_T[12];
  __shared__ __align__(16) DevCam s_cam;
  __shared__ float s_fsx[LC_MAX_LEVELS], s_fsy[LC_MAX_LEVELS], s_fr[LC_MAX_LEVELS];
  __shared__ int s_oc[LC_MAX_LEVELS], s_or[LC_MAX_LEVELS], s_ob[LC_MAX_LEVELS];
  const int tid = threadIdx.x;
  const int lane = tid & 31, warp = tid >> 5;
  const int blk = a.blk_base + (int)blockIdx.x;
  const int unit = a.blk_unit[blk];
  const int k = a.unit_kf[unit];
  const int fb = a.kf_fbeg[k];
  const int F = a.kf_fbeg[k + 1] - fb;
  const int fp = a.kf_fpad[k];
  float2* s_uv = (float2*)(smem + SM::UV);
  uint32_t* s_meta = (uint32_t*)(smem + SM::META);
  uint16_t* s_cell = (uint16_t*)(smem + SM::CELL);
  unsigned char* wb = smem + warp * SM::WB;
  uint32_t* s_qi = (uint32_t*)(wb + SM::QI);
  float4* s_op = (float4*)(wb + SM::OP);
  uint32_t* s_qd = (uint32_t*)(wb + SM::QD);
  uint32_t* s_key = (uint32_t*)(wb + SM::KEY);
  uint32_t* s_nc = (uint32_t*)(wb + SM::NC);
  const lc_match_params prm = a.params[0];
  if (tid == 0) {
    mbar_init(&s_bar, 1);
    const uint32_t b_cell = (uint32_t)a.Gs * 2u;
    const uint32_t np = (uint32_t)((F + 3) & ~3);   // keyframe blocks are padded to 4 features
    mbar_expect_tx(&s_bar, b_cell + (F > 0 ? np * 12u : 0u));
    tma_load_1d(s_cell, a.kf_cell + (size_t)k * a.Gs, b_cell, &s_bar);
    if (F > 0) {
      tma_load_1d(s_uv, a.fc_uv + fp, np * 8u, &s_bar);
      tma_load_1d(s_meta, a.fc_meta + fp, np * 4u, &s_bar);
    }
  }
  if (tid >= 32 && tid < 44) {   // SE3 part (R, t/s) of the unit's Sim3 (reading A2)
    const double* src = a.unit_S ? a.unit_S + 13 * (size_t)unit : a.kf_S_corr + 13 * (size_t)k;
    const int i = tid - 32;
    s_T[i] = i < 9 ? src[i] : src[i] / src[12];
  }
  if (tid >= 64 && tid < 64 + (int)(sizeof(DevCam) / 16))
    reinterpret_cast<uint4*>(&s_cam)[tid - 64] = reinterpret_cast<const uint4*>(a.cams + a.kf_cam[k])[tid - 64];
  if (tid >= 128 && tid < 128 + LC_MAX_LEVELS) {   // per-octave grid constants, fp32 radii
    const int o = tid - 128;
    const DevCam& c = a.cams[a.kf_cam[k]];
    s_fsx[o] = (float)c.cell_sx[o];
    s_fsy[o] = (float)c.cell_sy[o];
    s_fr[o] = (float)((double)prm.th * a.scale[o]);
    s_oc[o] = a.ocols[o];
    s_or[o] = a.orows[o];
    s_ob[o] = a.obase[o];
  }
  unsigned long long* win = a.winner + a.unit_woff[unit];
  for (int f = tid; f < F; f += LC_SOLE_NT) win[f] = NONE;   // this CTA owns the unit's words
  __syncthreads();

  const bool f32ok = fmax(fabs(s_cam.min_x), fabs(s_cam.max_x)) < 4096.0 &&
                     fmax(fabs(s_cam.min_y), fabs(s_cam.max_y)) < 4096.0;
  const float fminx = (float)s_cam.min_x, fminy = (float)s_cam.min_y;
  const int64_t q0 = a.blk_q0[blk];
  const int64_t qbase = a.unit_qoff[unit] + (q0 - a.unit_lbeg[unit]);
  const bool dbg = a.dbg_best || a.dbg_uv || a.dbg_ncand;
  pdl_wait();   // survivors of k_project from here on
  const Surv* sv = a.surv + a.surv_off[blk];
  const int ns_tot = a.surv_cnt[blk];
  uint32_t cC = 0, cP = 0, cE = 0, cW = 0;   // NOCAND | OVERTH << 10 | RATIO << 20; PROP; CAND; EDGE
  Surv e_nx;
  e_nx.q = 0; e_nx.jl = 0u; e_nx.fu = 0.f; e_nx.fv = 0.f;
  if (warp * 32 + lane < ns_tot) e_nx = sv[warp * 32 + lane];
  mbar_wait(&s_bar, 0);
  for (int i0 = warp * 32; i0 < ns_tot; i0 += SOLE_NW * 32) {
    const bool act = i0 + lane < ns_tot;
    const Surv e = e_nx;
    if (i0 + SOLE_NW * 32 + lane < ns_tot) e_nx = sv[i0 + SOLE_NW * 32 + lane];
    const int lvl = (int)((e.jl >> 27) & 7u);
    const float fr = s_fr[lvl];
    const int olo = max(lvl - 1, 0);
    // ---- A: items of this survivor (two passes over its cell rows: count, then write)
    int n_l = 0;
    if (act) {
      const uint4* rp = reinterpret_cast<const uint4*>(a.mp_rec + e.q);
      cp_async16(s_qd + lane * 8, rp + 2);
      cp_async16(s_qd + lane * 8 + 4, rp + 3);
      for (int o = olo; o <= lvl; ++o) {
        const int oc = s_oc[o], ob = s_ob[o];
        const int cx0 = max(0, (int)floorf((e.fu - fr - 0.01f - fminx) * s_fsx[o]));
        const int cx1 = min(oc - 1, (int)floorf((e.fu + fr + 0.01f - fminx) * s_fsx[o]));
        const int cy0 = max(0, (int)floorf((e.fv - fr - 0.01f - fminy) * s_fsy[o]));
        const int cy1 = min(s_or[o] - 1, (int)floorf((e.fv + fr + 0.01f - fminy) * s_fsy[o]));
        for (int cy = cy0; cy <= cy1; ++cy) n_l += (int)s_cell[ob + cy * oc + cx1 + 1] - (int)s_cell[ob + cy * oc + cx0];
      }
    }
    int incl = n_l;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += y;
    }
    const int ex = incl - n_l;
    // queued items: every survivor whose items fit entirely (the first overflowing one and
    // all after it rescan serially in phase C)
    const int total = __shfl_sync(0xffffffffu, incl, 31);   // (every lane: a full-mask shuffle)
    const int tot = (int)__reduce_min_sync(0xffffffffu, (unsigned)(incl > SOLE_QCAP ? ex : total));
    bool serial = act && incl > SOLE_QCAP;
    if (act && !serial && n_l > 0) {
      int j = ex;
      for (int o = olo; o <= lvl; ++o) {
        const int oc = s_oc[o], ob = s_ob[o];
        const int cx0 = max(0, (int)floorf((e.fu - fr - 0.01f - fminx) * s_fsx[o]));
        const int cx1 = min(oc - 1, (int)floorf((e.fu + fr + 0.01f - fminx) * s_fsx[o]));
        const int cy0 = max(0, (int)floorf((e.fv - fr - 0.01f - fminy) * s_fsy[o]));
        const int cy1 = min(s_or[o] - 1, (int)floorf((e.fv + fr + 0.01f - fminy) * s_fsy[o]));
        for (int cy = cy0; cy <= cy1; ++cy) {
          const int pe = s_cell[ob + cy * oc + cx1 + 1];
          for (int p = s_cell[ob + cy * oc + cx0]; p < pe; ++p) s_qi[j++] = ((uint32_t)lane << 16) | (uint32_t)p;
        }
      }
    }
    s_op[lane] = make_float4(e.fu, e.fv, fr, 0.f);
    s_nc[lane] = 0u;
    cp_async_wait_all();
    __syncwarp();
    // ---- B: items, 2 x 32 per step (two descriptor gathers in flight per lane)
    for (int c0 = 0; c0 < tot; c0 += 64) {
      uint32_t it[2];
      float2 fuv[2];
      int w[2];
      uint4 b0[2], b1[2];
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int c = c0 + 32 * h + lane;
        it[h] = c < tot ? s_qi[c] : 0xFFFFFFFFu;
        w[h] = 0;
        if (it[h] != 0xFFFFFFFFu) {
          const int p = (int)(it[h] & 0xFFFFu);
          const float4 op = s_op[it[h] >> 16];
          fuv[h] = s_uv[p];
          if (!f32ok) {
            w[h] = -1;
          } else {
            const float du = fabsf(fuv[h].x - op.x), dv = fabsf(fuv[h].y - op.y);
            w[h] = (du > op.z + kWinTol || dv > op.z + kWinTol) ? 0
                 : ((du < op.z - kWinTol && dv < op.z - kWinTol) ? 1 : -1);
          }
          if (w[h] != 0) {
            const uint4* dp = a.fc_desc + 2 * (size_t)(fp + p);
            b0[h] = __ldg(dp);
            b1[h] = __ldg(dp + 1);
          }
        }
      }
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        if (w[h] == 0) continue;
        const int own = (int)(it[h] >> 16), p = (int)(it[h] & 0xFFFFu);
        const uint4* qd = reinterpret_cast<const uint4*>(s_qd + own * 8);
        const uint32_t key = ((uint32_t)popc_desc(qd[0], qd[1], b0[h], b1[h]) << 16) | (s_meta[p] & 0xFFFFu) |
                             (w[h] < 0 ? kAmbKey : 0u);
        const uint32_t slot = atomicAdd(&s_nc[own], 1u);
        if (slot < (uint32_t)SOLE_CPL) s_key[own * SOLE_CPL + slot] = key;
      }
    }
    __syncwarp();
    // ---- C: per survivor
    if (act) {
      bool wedge = (e.jl & kSurvEdge) != 0u;
      uint32_t best = 0xFFFFFFFFu;   // (H << 16) | f
      int second = 256, nc = 0;
      auto take = [&](uint32_t key) {   // branch-free: the larger key of the pair is a "rest" key
        const uint32_t hi = max(key, best);
        best = min(key, best);
        second = min(second, (int)(hi >> 16));
      };
      const uint32_t ns = s_nc[lane];
      bool exact = serial || ns > (uint32_t)SOLE_CPL;
      if (!exact) {
        for (uint32_t j = 0; j < ns; ++j) {
          const uint32_t key = s_key[lane * SOLE_CPL + j];
          exact |= (key & kAmbKey) != 0u;
          take(key);
        }
        nc = (int)ns;
      }
      if (exact) {   // rare: exact fp64 rescan of this survivor (global descriptors)
        double u, v;
        exact_uv(a, s_T, s_cam, e.q, u, v);
        const uint4* qd = reinterpret_cast<const uint4*>(s_qd + lane * 8);
        const uint4 d0 = qd[0], d1 = qd[1];
        best = 0xFFFFFFFFu; second = 256; nc = 0;
        scan_exact<0>(a, s_cam, s_cell, s_uv, s_meta, a.fc_desc + 2 * (size_t)fp, e.fu, e.fv, fr, lvl, u, v,
                      (double)prm.th * a.scale[lvl], d0, d1, take, nc, wedge);
      }
      cE += nc;
      if (wedge) cW += 1u;
      do {
        if (nc == 0) { cC += 1u; break; }
        const int hb = (int)(best >> 16);
        if (hb > prm.max_hamming) { cC += 1u << 10; break; }
        if (prm.ratio_den > 0 && (long long)prm.ratio_den * hb > (long long)prm.ratio_num * second) {
          cC += 1u << 20; break;
        }
        cP += 1u;
        atomicMin(&win[best & 0xFFFFu], ((unsigned long long)hb << 32) | (unsigned int)e.q);
      } while (0);
      if (dbg) {
        const int64_t qi = qbase + (int64_t)(e.jl & 0x07FFFFFFu);
        if (a.dbg_best) {
          long long val;
          if (nc == 0) val = (256LL << 48) | (256LL << 32) | 0xFFFFFFFFLL;
          else val = ((long long)(best >> 16) << 48) | ((long long)second << 32) | (long long)(best & 0xFFFFu);
          a.dbg_best[qi] = val;
        }
        if (a.dbg_uv) {
          double u, v;
          exact_uv(a, s_T, s_cam, e.q, u, v);
          a.dbg_uv[2 * qi] = u; a.dbg_uv[2 * qi + 1] = v;
        }
        if (a.dbg_ncand) a.dbg_ncand[qi] = nc;
      }
    }
    __syncwarp();
  }
  pdl_trigger();
  uint32_t cnt[6];
  cnt[0] = cE; cnt[1] = cC & 1023u; cnt[2] = (cC >> 10) & 1023u; cnt[3] = (cC >> 20) & 1023u; cnt[4] = cP;
  cnt[5] = cW;
  block_add<6>(cnt, kMatchSlot2, a.counts);
  __syncthreads();   // all proposals of this unit are in: resolve it here (no extra launch)
  resolve_unit<0>(a, unit);
}

// Per-call setup: LoopSet stamps, winner/victim init, window membership. The call's
// epoch is ep[0] + 1 (device counter, so that a replayed CUDA graph gets a fresh one);
// the last block to finish publishes it in ep[0] for the kernels that follow.
__global__ void k_fuse_prep(int phase, int zero_counts, int64_t skip_lo, int64_t skip_hi, uint32_t* __restrict__ ep, int n_w,
                            const int32_t* __restrict__ window, int64_t n_wfeat,
                            const int32_t* __restrict__ mp_list, int64_t n_list, int n_mp,
                            unsigned long long* __restrict__ winner,
                            unsigned long long* __restrict__ victim, uint32_t* __restrict__ loop_ep,
                            uint32_t* __restrict__ kf_win_ep, int32_t* __restrict__ kf_win_pos,
                            uint32_t* __restrict__ vbits, int n_vbits, int32_t* __restrict__ dirty_n,
                            unsigned long long* __restrict__ counts) {
  pdl_trigger();   // k_project reads none of this kernel's outputs
  if (zero_counts && blockIdx.x == 0 && threadIdx.x < LC_NCOUNT) counts[threadIdx.x] = 0;   // the call's counters
  uint32_t epoch = ep[0] + 1u;
  if (epoch == 0u) epoch = 1u;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const int64_t t0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  for (int64_t i = t0; i < n_w; i += stride) {
    kf_win_ep[window[i]] = epoch;
    kf_win_pos[window[i]] = (int32_t)i;
  }
  for (int64_t i = t0; i < n_vbits; i += stride) vbits[i] = 0u;
  if (t0 == 0) *dirty_n = 0;
  if (phase & LC_FUSE_PLAN) {
    for (int64_t i = t0; i < n_list; i += stride) {
      const int32_t q = mp_list[i];
      if ((unsigned)q < (unsigned)n_mp) loop_ep[q] = epoch;
    }
    // every winner word is NONE after PLAN except those a sole-mode match CTA owns
    // ([skip_lo, skip_hi): the shard's own units, initialised by their CTAs)
    const int64_t lo = min(max(skip_lo, (int64_t)0), n_wfeat), hi = max(min(skip_hi, n_wfeat), lo);
    for (int64_t i = t0; i < lo; i += stride) winner[i] = NONE;   // (no pass over the owned range)
    for (int64_t i = hi + t0; i < n_wfeat; i += stride) winner[i] = NONE;
    const int64_t head = (reinterpret_cast<uintptr_t>(victim) & 15u) ? 1 : 0;   // (a caller's table slice)
    if (head && t0 == 0 && n_mp > 0) victim[0] = NONE;
    for (int64_t i = head + 2 * t0; i < n_mp; i += 2 * stride) {   // 16-B stores from a 16-B boundary
      if (i + 1 < n_mp) *reinterpret_cast<ulonglong2*>(victim + i) = make_ulonglong2(NONE, NONE);
      else victim[i] = NONE;
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    if (atomicAdd(&ep[1], 1u) == gridDim.x - 1) {
      ep[0] = epoch;
      ep[1] = 0u;
      __threadfence();
    }
  }
}

// Forced loop matches of the current keyframe (reading O9.4 / A23), thread per feature f
// of cur_kf: the tables of a separate apply that runs before the search. Map points are
// held once per keyframe, so every victim word gets at most one proposal.
__global__ void k_forced(int n_mp, const uint32_t* ep, int fb, int F,
                         const int32_t* __restrict__ forced, const int32_t* feat_mp,
                         const uint8_t* flags, const uint32_t* loop_ep,
                         unsigned long long* __restrict__ win_cur, unsigned long long* __restrict__ victim,
                         unsigned long long* __restrict__ counts) {
  pdl_wait();   // k_fuse_prep: tables initialised, LoopSet stamped, epoch published
  const uint32_t epoch = *ep;
  uint32_t n = 0;
  for (int f = blockIdx.x * blockDim.x + threadIdx.x; f < F; f += gridDim.x * blockDim.x) {
    const int32_t q = forced[f];
    if (q < 0 || q >= n_mp || (flags[q] & 1u)) continue;
    const int32_t m = feat_mp[fb + f];
    if (m == q) continue;
    if (m < 0) { win_cur[f] = (unsigned long long)(uint32_t)q; ++n; }
    else if ((flags[m] & 1u) || loop_ep[m] == epoch) continue;
    else { atomicMin(&victim[m], (unsigned long long)(uint32_t)q); ++n; }
  }
  pdl_trigger();
  const int slot[1] = {LC_COUNT_FORCED};
  uint32_t loc[1] = {n};
  block_add<1>(loc, slot, counts);
}

// Sparse ADD exchange (lc_fuse_adds): PACK compacts the shard's winner words on empty
// slots; UNPACK scatters gathered (index, word) pairs into a NONE-filled dense table.
__global__ void k_adds_pack(int64_t lo, int64_t hi, const int32_t* __restrict__ wpos_kf,
                            const int64_t* __restrict__ woff, int n_w, const int32_t* __restrict__ kf_fbeg,
                            const int32_t* __restrict__ feat_mp, const unsigned long long* __restrict__ winner,
                            long long* __restrict__ out_idx, long long* __restrict__ out_word,
                            unsigned long long* __restrict__ n_out, long long capacity) {
  for (int64_t j = lo + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < hi; j += (int64_t)gridDim.x * blockDim.x) {
    const unsigned long long w = winner[j];
    bool add = false;
    if (w != NONE) {
      int a = 0, b = n_w - 1;   // window position of j: last i with woff[i] <= j
      while (a < b) {
        const int mid = (a + b + 1) >> 1;
        if (woff[mid] <= j) a = mid; else b = mid - 1;
      }
      add = feat_mp[kf_fbeg[wpos_kf[a]] + (j - woff[a])] == -1;
    }
    if (add) {
      const unsigned long long i = atomicAdd(n_out, 1ull);
      if ((long long)i < capacity) { out_idx[i] = (long long)j; out_word[i] = (long long)w; }
    }
  }
}

__global__ void k_adds_unpack(int64_t n_wfeat, int64_t n, const long long* __restrict__ idx,
                              const long long* __restrict__ word, unsigned long long* __restrict__ winner) {
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < n_wfeat; j += (int64_t)gridDim.x * blockDim.x)
    winner[j] = NONE;
  __threadfence();
}
__global__ void k_adds_scatter(int64_t n_wfeat, int64_t n, const long long* __restrict__ idx,
                               const long long* __restrict__ word, unsigned long long* __restrict__ winner) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    if (idx[i] >= 0 && idx[i] < n_wfeat) winner[idx[i]] = (unsigned long long)word[i];
}

// Victim marking: flags |= bad, replaced_by = survivor (reading O9 (iv)), victim bitmap.
__global__ void k_fuse_victims(int n_mp, const unsigned long long* victim,
                               uint8_t* __restrict__ flags, int32_t* __restrict__ replaced_by,
                               int32_t* __restrict__ nobs,
                               uint32_t* __restrict__ vbits, unsigned long long* __restrict__ counts) {
  pdl_wait();
  uint32_t n = 0;
  const int stride = gridDim.x * blockDim.x;
  for (int q0 = blockIdx.x * blockDim.x; q0 < n_mp; q0 += stride) {
    const int q = q0 + threadIdx.x;
    bool isv = false;
    if (q < n_mp) {
      unsigned long long v = victim[q];
      if (v != NONE) {
        isv = true;
        flags[q] |= 1u;
        replaced_by[q] = (int32_t)(v & 0xFFFFFFFFull);
        // every slot holding a victim is rewired (or cleared) by APPLY, and n_obs counts the
        // slots holding a point (the store's invariant: counted at upload, kept by APPLY), so
        // the victim's count ends at 0 -- set here instead of one atomicSub per slot (a slot
        // rewired to a point that is itself a victim -- a forced-match chain -- still gets
        // its +1 in APPLY, after this)
        nobs[q] = 0;
        ++n;
      }
    }
    const unsigned m = __ballot_sync(0xffffffffu, isv);   // q0 is a multiple of 32
    if ((threadIdx.x & 31) == 0 && m) vbits[(q0 + threadIdx.x) >> 5] = m;
  }
  pdl_trigger();
  const int slot[1] = {LC_COUNT_VICTIMS};
  uint32_t loc[1] = {n};
  block_add<1>(loc, slot, counts);
}

// Apply pass 1: find the keyframes whose slots change (a victim to redirect or a
// winner on an empty window slot) -> compact list. One warp per keyframe, 16-B loads,
// no shared memory (the victim bitmap stays L1-resident).
__global__ void __launch_bounds__(LC_NTHREADS) k_apply_mark(
    int n_kf, const uint32_t* ep, const int32_t* __restrict__ kf_fbeg,
    const uint32_t* kf_win_ep, const int32_t* kf_win_pos,
    const int64_t* woff_of_pos, const unsigned long long* winner,
    const uint32_t* vbits, const int32_t* __restrict__ feat_mp,
    int32_t* __restrict__ dirty_list) {
  pdl_wait();
  pdl_trigger();   // one wave: k_apply_fix may take the remaining slots now
  const uint32_t epoch = *ep;
  const int lane = threadIdx.x & 31;
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  for (int k = gw; k < n_kf; k += nw) {
    const int fb = kf_fbeg[k], fe = kf_fbeg[k + 1];
    const int wpos = (kf_win_ep[k] == epoch) ? kf_win_pos[k] : -1;
    const int64_t wshift = wpos >= 0 ? woff_of_pos[wpos] - fb : 0;   // winner index = f + wshift
    // a window keyframe is listed without the scan: nearly all of them change (their
    // duplicates were fused), and APPLY on an unchanged keyframe writes nothing
    int dirty = wpos >= 0 ? 1 : 0;
    // 4 x 16-B association loads in flight per lane (512 slots per warp round)
    for (int f0 = fb; f0 < fe && !__any_sync(0xffffffffu, dirty); f0 += 512) {
      int32_t m[16];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int f = f0 + 128 * u + 4 * lane;
        if (f + 3 < fe && !(f & 3)) {
          const int4 m4 = __ldg(reinterpret_cast<const int4*>(feat_mp + f));
          m[4 * u] = m4.x; m[4 * u + 1] = m4.y; m[4 * u + 2] = m4.z; m[4 * u + 3] = m4.w;
        } else {
#pragma unroll
          for (int v = 0; v < 4; ++v) m[4 * u + v] = (f + v < fe) ? feat_mp[f + v] : INT32_MIN;
        }
      }
#pragma unroll
      for (int u = 0; u < 16; ++u) {
        const int32_t mm = m[u];
        if (mm >= 0) dirty |= (ld_nc_after_wait(vbits + (mm >> 5)) >> (mm & 31)) & 1u;
        else if (mm != INT32_MIN && wpos >= 0)
          dirty |= winner[f0 + 128 * (u >> 2) + 4 * lane + (u & 3) + wshift] != NONE;
      }
    }
    if (__any_sync(0xffffffffu, dirty) && lane == 0) {
      const int i = atomicAdd(&dirty_list[0], 1);
      dirty_list[1 + i] = k;
    }
  }
}

// Apply pass 2 (dirty keyframes only): redirect victims, add winners to empty window
// slots, per-keyframe duplicate cleanup by least (priority, f) (reading A22), n_obs
// deltas. Only the NEW map points of changed slots are hashed: an unchanged slot can
// only collide with a changed one (the input holds no map point twice in a keyframe).
enum { A_REWIRED, A_DUP, A_ADDED, A_N };
__device__ __constant__ int kApplySlot[A_N] = {LC_COUNT_REWIRED, LC_COUNT_DUP_CLEARED,
                                               LC_COUNT_ADDED};

__global__ void __launch_bounds__(LC_NTHREADS) k_apply_fix(
    const uint32_t* ep, const int32_t* __restrict__ kf_fbeg,
    const uint32_t* kf_win_ep, const int32_t* kf_win_pos,
    const int64_t* woff_of_pos, const unsigned long long* winner,
    const unsigned long long* victim, const uint32_t* vbits,
    const int32_t* dirty_list, int32_t* __restrict__ feat_mp, int32_t* __restrict__ nobs,
    int hash_size, unsigned long long* __restrict__ counts) {
  pdl_wait();
  const uint32_t epoch = *ep;
  extern __shared__ __align__(128) unsigned char smem[];
  uint32_t cnt[A_N] = {0, 0, 0};
  const int nd = dirty_list[0];
  const uint32_t HS = (uint32_t)hash_size;
  int32_t* s_key = (int32_t*)smem;
  uint32_t* s_val = (uint32_t*)(s_key + hash_size);
  uint32_t* s_filt = s_val + hash_size;                          // 2^15-bit pre-filter
  int32_t* s_new = (int32_t*)(s_filt + (1 << (FILT_LOG2 - 5)));   // [F] new association per slot
  auto probe = [&](int32_t key) -> int {   // slot of key in the hash, -1 if absent
    uint32_t h = hslot(key, HS);
    while (true) {
      const int32_t v = s_key[h];
      if (v == key) return (int)h;
      if (v == -1) return -1;
      h = (h + 1 == HS) ? 0 : h + 1;
    }
  };
  auto filt_has = [&](int32_t key) -> bool {
    const uint32_t b = fslot(key);
    return (s_filt[b >> 5] >> (b & 31)) & 1u;
  };
  for (int di = blockIdx.x; di < nd; di += gridDim.x) {
    const int k = dirty_list[1 + di];
    const int fb = kf_fbeg[k], F = kf_fbeg[k + 1] - fb;
    const int wpos = (kf_win_ep[k] == epoch) ? kf_win_pos[k] : -1;
    const int64_t woff = wpos >= 0 ? woff_of_pos[wpos] : 0;
    int32_t* s_old = s_new + F;                // [F] association before the apply
    uint8_t* s_pr = (uint8_t*)(s_old + F);     // [F] priority: 0 unchanged, 1 ADD, 2 rewired
    for (int i = threadIdx.x; i < (int)HS; i += blockDim.x) { s_key[i] = -1; s_val[i] = 0xFFFFFFFFu; }
    for (int i = threadIdx.x; i < (1 << (FILT_LOG2 - 5)); i += blockDim.x) s_filt[i] = 0u;
    __syncthreads();
    // (1) new value per slot (8 slots per thread, their loads in flight together); the
    // new map point of every changed slot is hashed and competes at once with key
    // (priority, f) (reading A22)
    for (int base = 0; base < F; base += 8 * (int)blockDim.x) {
      int32_t m[8];
      unsigned long long w[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int f = base + u * (int)blockDim.x + (int)threadIdx.x;
        m[u] = f < F ? feat_mp[fb + f] : INT32_MIN;
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int f = base + u * (int)blockDim.x + (int)threadIdx.x;
        const bool isv = m[u] >= 0 && ((ld_nc_after_wait(vbits + (m[u] >> 5)) >> (m[u] & 31)) & 1u);
        w[u] = isv ? victim[m[u]] : ((m[u] == -1 && wpos >= 0) ? winner[woff + f] : NONE);
        if (!isv && m[u] >= 0) w[u] = NONE;
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int f = base + u * (int)blockDim.x + (int)threadIdx.x;
        if (f >= F) continue;
        int32_t nv = m[u];
        uint8_t pr = 0;
        if (w[u] != NONE) {
          nv = (int32_t)(w[u] & 0xFFFFFFFFull);
          pr = m[u] >= 0 ? 2 : 1;
          if (pr == 2) cnt[A_REWIRED]++;
        }
        s_new[f] = nv;
        s_old[f] = m[u];
        s_pr[f] = pr;
        if (pr) {
          uint32_t h = hslot(nv, HS);
          while (true) {
            const int32_t prev = atomicCAS(&s_key[h], -1, nv);
            if (prev == -1 || prev == nv) break;
            h = (h + 1 == HS) ? 0 : h + 1;
          }
          atomicMin(&s_val[h], ((uint32_t)pr << 16) | (uint32_t)f);
          const uint32_t b = fslot(nv);
          atomicOr(&s_filt[b >> 5], 1u << (b & 31));
        }
      }
    }
    __syncthreads();
    // (2) unchanged slots holding a hashed map point compete too (priority 0 wins)
    for (int f = threadIdx.x; f < F; f += blockDim.x) {
      const int32_t nv = s_new[f];
      if (nv < 0 || s_pr[f] != 0 || !filt_has(nv)) continue;
      const int h = probe(nv);
      if (h >= 0) atomicMin(&s_val[h], (uint32_t)f);
    }
    __syncthreads();
    // (3) losers of a hashed map point are cleared; write changed slots, n_obs deltas
    for (int f = threadIdx.x; f < F; f += blockDim.x) {
      int32_t nv = s_new[f];
      const uint8_t pr = s_pr[f];
      if (nv < 0 || (pr == 0 && !filt_has(nv))) continue;
      const int h = probe(nv);
      if (h >= 0 && s_val[h] != (((uint32_t)pr << 16) | (uint32_t)f)) { nv = -1; cnt[A_DUP]++; }
      else if (pr == 1) cnt[A_ADDED]++;
      const int32_t m = s_old[f];
      if (nv != m) {
        feat_mp[fb + f] = nv;
        // (m >= 0 here only for a victim, whose count k_fuse_victims already set to 0)
        if (nv >= 0) atomicAdd(&nobs[nv], 1);
      }
    }
    __syncthreads();
  }
  block_add<A_N>(cnt, kApplySlot, counts);
}

// Apply pass 2 for keyframes of <= SPT * LC_NTHREADS slots: the same three steps with each
// thread's SPT slots (f = u * LC_NTHREADS + tid) held in registers across them, so the only
// shared state is the hash of the changed slots' new map points (+ its pre-filter), and only
// the hash entries a keyframe used are reset after it (no per-keyframe table clear).
// Step 2 marks a hashed map point held by an unchanged slot with the key f < 2^16, below
// every changed slot's key (priority 1 or 2 in bits 16-17), exactly as k_apply_fix does.
template <int SPT>
__global__ void __launch_bounds__(LC_NTHREADS) k_apply_fix_r(
    const uint32_t* ep, const int32_t* __restrict__ kf_fbeg,
    const uint32_t* kf_win_ep, const int32_t* kf_win_pos,
    const int64_t* woff_of_pos, const unsigned long long* winner,
    const unsigned long long* victim, const uint32_t* vbits,
    const int32_t* dirty_list, int32_t* __restrict__ feat_mp, int32_t* __restrict__ nobs,
    int hash_size, unsigned long long* __restrict__ counts) {
  extern __shared__ __align__(128) unsigned char smem[];
  const uint32_t HS = (uint32_t)hash_size;
  int32_t* s_key = (int32_t*)smem;
  uint32_t* s_val = (uint32_t*)(s_key + hash_size);
  uint32_t* s_filt = s_val + hash_size;   // 2^15-bit pre-filter
  for (int i = threadIdx.x; i < (int)HS; i += blockDim.x) { s_key[i] = -1; s_val[i] = 0xFFFFFFFFu; }
  for (int i = threadIdx.x; i < (1 << (FILT_LOG2 - 5)); i += blockDim.x) s_filt[i] = 0u;
  pdl_wait();
  const uint32_t epoch = *ep;
  const int nd = dirty_list[0];
  uint32_t cnt[A_N] = {0, 0, 0};
  __syncthreads();
  for (int di = blockIdx.x; di < nd; di += gridDim.x) {
    const int k = dirty_list[1 + di];
    const int fb = kf_fbeg[k], F = kf_fbeg[k + 1] - fb;
    const int wpos = (kf_win_ep[k] == epoch) ? kf_win_pos[k] : -1;
    const int64_t woff = wpos >= 0 ? woff_of_pos[wpos] : 0;
    int32_t m[SPT], nv[SPT], h[SPT];
    uint32_t prb = 0;   // 2 bits per slot: 0 unchanged, 1 ADD, 2 rewired
    // (1) new value per slot, every load of a phase issued together
#pragma unroll
    for (int u = 0; u < SPT; ++u) {
      const int f = u * LC_NTHREADS + (int)threadIdx.x;
      m[u] = f < F ? feat_mp[fb + f] : INT32_MIN;
    }
    bool isv[SPT];
#pragma unroll
    for (int u = 0; u < SPT; ++u) isv[u] = m[u] >= 0 && ((ld_nc_after_wait(vbits + (m[u] >> 5)) >> (m[u] & 31)) & 1u);
    unsigned long long w[SPT];
#pragma unroll
    for (int u = 0; u < SPT; ++u) {
      const int f = u * LC_NTHREADS + (int)threadIdx.x;
      w[u] = isv[u] ? victim[m[u]] : ((m[u] == -1 && wpos >= 0) ? winner[woff + f] : NONE);
    }
#pragma unroll
    for (int u = 0; u < SPT; ++u) {
      const int f = u * LC_NTHREADS + (int)threadIdx.x;
      nv[u] = m[u];
      h[u] = -1;
      if (w[u] != NONE) {
        const uint32_t pr = isv[u] ? 2u : 1u;
        nv[u] = (int32_t)(w[u] & 0xFFFFFFFFull);
        prb |= pr << (2 * u);
        if (pr == 2) cnt[A_REWIRED]++;
        uint32_t hh = hslot(nv[u], HS);
        while (true) {
          const int32_t prev = atomicCAS(&s_key[hh], -1, nv[u]);
          if (prev == -1 || prev == nv[u]) break;
          hh = (hh + 1 == HS) ? 0 : hh + 1;
        }
        h[u] = (int)hh;
        atomicMin(&s_val[hh], (pr << 16) | (uint32_t)f);
        const uint32_t b = fslot(nv[u]);
        atomicOr(&s_filt[b >> 5], 1u << (b & 31));
      }
    }
    __syncthreads();
    // (2) an unchanged slot holding a hashed map point keeps it (priority 0 wins)
#pragma unroll
    for (int u = 0; u < SPT; ++u) {
      if (((prb >> (2 * u)) & 3u) || nv[u] < 0) continue;
      const uint32_t b = fslot(nv[u]);
      if (!((s_filt[b >> 5] >> (b & 31)) & 1u)) continue;
      uint32_t hh = hslot(nv[u], HS);
      while (true) {
        const int32_t v = s_key[hh];
        if (v == nv[u]) { atomicMin(&s_val[hh], (uint32_t)(u * LC_NTHREADS + (int)threadIdx.x)); break; }
        if (v == -1) break;
        hh = (hh + 1 == HS) ? 0 : hh + 1;
      }
    }
    __syncthreads();
    // (3) losers of a hashed map point are cleared; changed slots written, n_obs deltas
#pragma unroll
    for (int u = 0; u < SPT; ++u) {
      const uint32_t pr = (prb >> (2 * u)) & 3u;
      if (!pr) continue;
      const int f = u * LC_NTHREADS + (int)threadIdx.x;
      int32_t v = nv[u];
      if (s_val[h[u]] != ((pr << 16) | (uint32_t)f)) { v = -1; cnt[A_DUP]++; }
      else if (pr == 1) cnt[A_ADDED]++;
      if (v != m[u]) {
        feat_mp[fb + f] = v;
        // (m >= 0 here only for a victim, whose count k_fuse_victims already set to 0)
        if (v >= 0) atomicAdd(&nobs[v], 1);
      }
    }
    __syncthreads();
    // reset the entries this keyframe used (every set filter word belongs to a changed slot)
#pragma unroll
    for (int u = 0; u < SPT; ++u) {
      if (h[u] < 0) continue;
      s_key[h[u]] = -1;
      s_val[h[u]] = 0xFFFFFFFFu;
      s_filt[fslot(nv[u]) >> 5] = 0u;
    }
    __syncthreads();
  }
  block_add<A_N>(cnt, kApplySlot, counts);
}

// lc_fuse with device-resident list offsets: unit i = block i = list i, its queries
// [begin[i], begin[i+1]); t = [lbeg | qoff | blk_q0 | blk_q1 | surv_off] (n each)
__global__ void k_csr_units(int n, const int32_t* __restrict__ begin, int64_t* __restrict__ t) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int64_t b = begin[i], e = begin[i + 1];
  t[i] = b;
  t[n + i] = b;
  t[2 * (size_t)n + i] = b;
  t[3 * (size_t)n + i] = e;
  t[4 * (size_t)n + i] = b;
}

int grid_for(int64_t n) {
  int64_t b = (n + LC_NTHREADS - 1) / LC_NTHREADS;
  if (b < 1) b = 1;
  if (b > 148 * 16) b = 148 * 16;
  return (int)b;
}


}  // namespace

template <int MODE, int FCAP>
cudaError_t launch_match_t(const MatchArgs& a, int n_blocks, int part, bool pdl, cudaStream_t s) {
  using SM = MatchSmem<FCAP>;
  auto go = [&](auto kernel, size_t smem) -> cudaError_t {
    if (pdl) return launch_pdl(kernel, dim3(n_blocks), dim3(LC_NTHREADS), smem, s, a);
    kernel<<<n_blocks, LC_NTHREADS, smem, s>>>(a);
    return cudaGetLastError();
  };
  if (part == 0) {
    const int hb = HashSize<FCAP>::HS * (int)sizeof(int32_t) + 3 * LC_NTHREADS * 32;   // hash + record ring
    cudaError_t e = set_smem_attr((const void*)k_project<MODE, FCAP>, hb);
    if (e != cudaSuccess) return e;
    return go(k_project<MODE, FCAP>, (size_t)hb);
  }
  if (MODE == 0 && a.sole == 2 && FCAP <= 4096) {
    using SS = SoleSmem<FCAP>;
    const size_t smem = (size_t)SS::CELL + (((size_t)a.Gs * 2 + 15) & ~(size_t)15);
    cudaError_t e = set_smem_attr((const void*)k_match_sole<FCAP>, (int)smem, true);
    if (e != cudaSuccess) return e;
    if (pdl) return launch_pdl(k_match_sole<FCAP>, dim3(n_blocks), dim3(LC_SOLE_NT), smem, s, a);
    k_match_sole<FCAP><<<n_blocks, LC_SOLE_NT, smem, s>>>(a);
    return cudaGetLastError();
  }
  const size_t smem = (size_t)SM::CELL + (((size_t)a.Gs * 2 + 15) & ~(size_t)15);
  cudaError_t e = set_smem_attr((const void*)k_match<MODE, FCAP>, (int)smem, true);
  if (e != cudaSuccess) return e;
  return go(k_match<MODE, FCAP>, smem);
}

template <int MODE>
cudaError_t launch_match_m(const MatchArgs& a, int n_blocks, int F_max, int part, bool pdl, cudaStream_t s) {
  if (F_max <= 512) return launch_match_t<MODE, 512>(a, n_blocks, part, pdl, s);
  if (F_max <= 1024) return launch_match_t<MODE, 1024>(a, n_blocks, part, pdl, s);
  if (F_max <= 2048) return launch_match_t<MODE, 2048>(a, n_blocks, part, pdl, s);
  if (F_max <= 4096) return launch_match_t<MODE, 4096>(a, n_blocks, part, pdl, s);
  return launch_match_t<MODE, 8192>(a, n_blocks, part, pdl, s);
}

cudaError_t launch_match(lc_ctx* c, int mode, const MatchArgs& a, int n_blocks, int F_max, int part,
                         cudaStream_t s, bool pdl) {
  if (n_blocks <= 0) return cudaSuccess;
  cudaError_t e = mode == 0 ? launch_match_m<0>(a, n_blocks, F_max, part, pdl, s)
                            : launch_match_m<1>(a, n_blocks, F_max, part, pdl, s);
  c->launches += 1;
  return e;
}

cudaError_t launch_resolve(lc_ctx* c, int mode, const MatchArgs& a, int n_units, cudaStream_t s) {
  if (n_units <= 0) return cudaSuccess;
  if (mode == 0) k_resolve<0><<<n_units, LC_NTHREADS, 0, s>>>(a);
  else k_resolve<1><<<n_units, LC_NTHREADS, 0, s>>>(a);
  c->launches++;
  return cudaGetLastError();
}

cudaError_t launch_csr_units(lc_ctx* c, int n, const int32_t* d_begin, int64_t* d_t, cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  k_csr_units<<<(n + LC_NTHREADS - 1) / LC_NTHREADS, LC_NTHREADS, 0, s>>>(n, d_begin, d_t);
  c->launches++;
  return cudaGetLastError();
}

cudaError_t launch_fuse_prep(lc_ctx* c, int phase, int zero_counts, int64_t skip_lo, int64_t skip_hi, int n_w,
                             const int32_t* d_window, int64_t n_wfeat, const int32_t* mp_list,
                             int64_t n_list_total,
                             unsigned long long* winner, unsigned long long* victim,
                             unsigned long long* counts, cudaStream_t s) {
  Store& st = c->st;
  const int n_vbits = (st.n_mp + 31) / 32;
  int64_t n = std::max<int64_t>(n_w, n_vbits);
  if (phase & LC_FUSE_PLAN) {
    n = std::max<int64_t>(n, n_list_total);
    if (skip_hi - skip_lo < n_wfeat) n = std::max<int64_t>(n, n_wfeat);
    n = std::max<int64_t>(n, st.n_mp);
  }
  // (a grid of at most 2 CTAs per SM: every CTA ends with an atomic on the one epoch word,
  // and 2,368 of them serialised on it cost more than the fills)
  k_fuse_prep<<<std::min(grid_for(n), 148 * 2), LC_NTHREADS, 0, s>>>(phase, zero_counts, skip_lo, skip_hi, st.ep, n_w,
                                                                   d_window, n_wfeat,
                                                 mp_list, n_list_total, st.n_mp, winner, victim,
                                                 st.mp_loop_ep, st.kf_win_ep, st.kf_win_pos,
                                                 st.mp_vbits, n_vbits, st.kf_dirty, counts);
  c->launches++;
  return cudaGetLastError();
}

cudaError_t launch_forced(lc_ctx* c, int cur_kf, const int32_t* d_forced, unsigned long long* win_cur,
                          unsigned long long* victim, unsigned long long* counts, cudaStream_t s) {
  Store& st = c->st;
  const int fb = st.h_fbeg[cur_kf], F = st.h_fbeg[cur_kf + 1] - fb;
  cudaError_t e = launch_pdl(k_forced, dim3(std::max(1, (F + LC_NTHREADS - 1) / LC_NTHREADS)), dim3(LC_NTHREADS), 0, s,
                             st.n_mp, (const uint32_t*)st.ep, fb, F, d_forced, (const int32_t*)st.feat_mp,
                             (const uint8_t*)st.mp_flags, (const uint32_t*)st.mp_loop_ep, win_cur, victim, counts);
  c->launches++;
  return e;
}

cudaError_t launch_fuse_apply(lc_ctx* c, const int64_t* d_woff, const unsigned long long* winner,
                              const unsigned long long* victim, unsigned long long* counts,
                              cudaStream_t s) {
  Store& st = c->st;
  if (st.n_mp > 0) {
    cudaError_t e = launch_pdl(k_fuse_victims, dim3(grid_for(st.n_mp)), dim3(LC_NTHREADS), 0, s, st.n_mp,
                               victim, st.mp_flags, st.mp_replaced_by, st.mp_nobs, st.mp_vbits, counts);
    if (e != cudaSuccess) return e;
    c->launches++;
  }
  if (st.n_kf > 0) {
    cudaError_t e = launch_pdl(k_apply_mark, dim3(std::min((st.n_kf + NWARP - 1) / NWARP, 148 * 8)),
                               dim3(LC_NTHREADS), 0, s, st.n_kf, (const uint32_t*)st.ep,
                               (const int32_t*)st.kf_fbeg, (const uint32_t*)st.kf_win_ep,
                               (const int32_t*)st.kf_win_pos, d_woff, winner, (const uint32_t*)st.mp_vbits,
                               (const int32_t*)st.feat_mp, st.kf_dirty);
    if (e != cudaSuccess) return e;
    const int Fm = st.max_F > 0 ? st.max_F : 1;
    const int H = ((Fm + Fm / 2 + 1) + 31) & ~31;
    if (Fm <= 8 * LC_NTHREADS && !getenv("LC_APPLY_SMEM")) {   // slots in registers (k_apply_fix_r)
      const size_t sm = (size_t)H * 8 + (size_t)(1 << (FILT_LOG2 - 3));
      auto go = [&](auto kern) -> cudaError_t {
        cudaError_t e2 = set_smem_attr((const void*)kern, (int)sm);
        if (e2 != cudaSuccess) return e2;
        return launch_pdl(kern, dim3(std::min(st.n_kf, 148 * 4)), dim3(LC_NTHREADS), sm, s,
                          (const uint32_t*)st.ep, (const int32_t*)st.kf_fbeg, (const uint32_t*)st.kf_win_ep,
                          (const int32_t*)st.kf_win_pos, d_woff, winner, victim, (const uint32_t*)st.mp_vbits,
                          (const int32_t*)st.kf_dirty, st.feat_mp, st.mp_nobs, H, counts);
      };
      e = Fm <= 2 * LC_NTHREADS ? go(k_apply_fix_r<2>) : Fm <= 4 * LC_NTHREADS ? go(k_apply_fix_r<4>)
                                                                                 : go(k_apply_fix_r<8>);
      if (e != cudaSuccess) return e;
      c->launches += 2;
      return cudaGetLastError();
    }
    size_t smem = (size_t)H * 8 + (size_t)(1 << (FILT_LOG2 - 3)) + (size_t)Fm * 9 + 16;
    smem = (smem + 15) & ~(size_t)15;
    e = set_smem_attr((const void*)k_apply_fix, (int)smem);
    if (e != cudaSuccess) return e;
    e = launch_pdl(k_apply_fix, dim3(std::min(st.n_kf, 148 * 4)), dim3(LC_NTHREADS), smem, s,
                   (const uint32_t*)st.ep, (const int32_t*)st.kf_fbeg, (const uint32_t*)st.kf_win_ep,
                   (const int32_t*)st.kf_win_pos, d_woff, winner, victim, (const uint32_t*)st.mp_vbits,
                   (const int32_t*)st.kf_dirty, st.feat_mp, st.mp_nobs, H, counts);
    if (e != cudaSuccess) return e;
    c->launches += 2;
  }
  return cudaGetLastError();
}

cudaError_t launch_adds(lc_ctx* c, int op, int n_w, const int32_t* d_window, const int64_t* d_woff, int64_t n_wfeat,
                        int64_t lo, int64_t hi, unsigned long long* winner, long long* idx, long long* word,
                        unsigned long long* d_n, int64_t n_in, int64_t capacity, cudaStream_t s) {
  Store& st = c->st;
  if (op == LC_ADDS_PACK) {
    cudaError_t e = cudaMemsetAsync(d_n, 0, sizeof(unsigned long long), s);
    if (e != cudaSuccess) return e;
    if (hi > lo)
      k_adds_pack<<<grid_for(hi - lo), LC_NTHREADS, 0, s>>>(lo, hi, d_window, d_woff, n_w, st.kf_fbeg, st.feat_mp,
                                                           winner, idx, word, d_n, (long long)capacity);
    c->launches++;
  } else {
    k_adds_unpack<<<grid_for(n_wfeat), LC_NTHREADS, 0, s>>>(n_wfeat, n_in, idx, word, winner);
    if (n_in > 0) k_adds_scatter<<<grid_for(n_in), LC_NTHREADS, 0, s>>>(n_wfeat, n_in, idx, word, winner);
    c->launches += n_in > 0 ? 2 : 1;
  }
  return cudaGetLastError();
}
