// k_refresh.cu -- map-point refresh after a merge (PAPER.md:95
// "identify and merge duplicate map points"; the refresh itself is inherited
// ORB-SLAM3 behaviour, readings A33-A37, include/lc.h lc_refresh_mappoints).
//
// Two steps, all on the device store:
//   (1) observation lists: exclusive scan of n_obs (the association count the apply
//       keeps exact) -> per-point offsets; one thread per feature scatters its index
//       (unordered inside a point; step 2 orders them);
//   (2) warp per refreshed point: rank-sort its observations by feature index (A34),
//       stage their descriptors in shared memory, all-pairs Hamming rows with the
//       row median by counting (distances are <= 256), warp argmin of
//       (median, observation rank) (A35); lane 0 then sums the unit viewing vectors
//       in observation order in fp64 (A36) and the depth bound from the reference
//       keyframe's first observation (A37). Points with more observations than fit a
//       warp's shared staging take a global-memory path with the same arithmetic.
#include <cuda_runtime.h>

#include <algorithm>

#include "lc_internal.cuh"

namespace {

constexpr int SCAN_PER = 8;                       // elements per thread in the scan
constexpr int SCAN_SEG = LC_NTHREADS * SCAN_PER;  // elements per block
constexpr int OBS_CAP = 64;                       // observations staged per warp
constexpr int RWARPS = LC_NTHREADS / 32;

// block-local exclusive scan of in[0, n) (n_obs), block totals to bsum
__global__ void k_scan_a(const int32_t* __restrict__ in, int n, int32_t* __restrict__ out,
                         int32_t* __restrict__ bsum) {
  __shared__ int32_t s_w[RWARPS];
  const int base = blockIdx.x * SCAN_SEG + threadIdx.x * SCAN_PER;
  int32_t v[SCAN_PER], t = 0;
#pragma unroll
  for (int i = 0; i < SCAN_PER; ++i) {
    v[i] = base + i < n ? in[base + i] : 0;
    t += v[i];
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int32_t incl = t;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int32_t y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += y;
  }
  if (lane == 31) s_w[warp] = incl;
  __syncthreads();
  int32_t woff = 0;
  for (int w = 0; w < warp; ++w) woff += s_w[w];
  int32_t acc = woff + incl - t;
#pragma unroll
  for (int i = 0; i < SCAN_PER; ++i) {
    if (base + i < n) out[base + i] = acc;
    acc += v[i];
  }
  if (threadIdx.x == LC_NTHREADS - 1) bsum[blockIdx.x] = woff + incl;
}

// exclusive scan of the block totals (one block, sequential chunks with a carry);
// out[n] = total
__global__ void k_scan_b(int32_t* __restrict__ bsum, int nb, int32_t* __restrict__ total) {
  __shared__ int32_t s_carry;
  if (threadIdx.x == 0) s_carry = 0;
  __syncthreads();
  for (int c0 = 0; c0 < nb; c0 += LC_NTHREADS) {
    const int i = c0 + threadIdx.x;
    const int32_t v = i < nb ? bsum[i] : 0;
    __shared__ int32_t s_v[LC_NTHREADS];
    s_v[threadIdx.x] = v;
    __syncthreads();
    if (threadIdx.x == 0) {
      int32_t acc = s_carry;
      for (int j = 0; j < LC_NTHREADS; ++j) { const int32_t x = s_v[j]; s_v[j] = acc; acc += x; }
      s_carry = acc;
    }
    __syncthreads();
    if (i < nb) bsum[i] = s_v[threadIdx.x];
    __syncthreads();
  }
  if (threadIdx.x == 0) *total = s_carry;
}

__global__ void k_scan_c(int32_t* __restrict__ out, int n, const int32_t* __restrict__ bsum,
                         int32_t* __restrict__ cursor) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) {
    const int32_t x = out[i] + bsum[i / SCAN_SEG];
    out[i] = x;
    cursor[i] = x;
  }
}

// (1) scatter (feature, keyframe) into their point's observation segment: a CTA per
// keyframe, so the keyframe of each observation is known without a search
__global__ void k_obs_fill(int n_kf, int n_mp, const int32_t* __restrict__ kf_fbeg,
                           const int32_t* __restrict__ feat_mp, const int32_t* __restrict__ obeg,
                           int32_t* __restrict__ cursor, int32_t* __restrict__ obs,
                           int32_t* __restrict__ obs_kf) {
  for (int k = blockIdx.x; k < n_kf; k += gridDim.x) {
    const int fe = kf_fbeg[k + 1];
    for (int f = kf_fbeg[k] + threadIdx.x; f < fe; f += blockDim.x) {
      const int32_t q = feat_mp[f];
      if ((unsigned)q >= (unsigned)n_mp) continue;
      const int32_t p = atomicAdd(&cursor[q], 1);
      if (p < obeg[q + 1]) { obs[p] = f; obs_kf[p] = k; }
    }
  }
}

__device__ __forceinline__ int kf_of_feature(const int32_t* __restrict__ kf_fbeg, int n_kf, int f) {
  int lo = 0, hi = n_kf - 1;   // largest k with kf_fbeg[k] <= f
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (kf_fbeg[mid] <= f) lo = mid; else hi = mid - 1;
  }
  return lo;
}

// camera centre Ow = -R^T (t/s) of a keyframe pose (reading A2), in the oracle's order
__device__ __forceinline__ void kf_centre(const double* __restrict__ kf_pose, int k, double* O) {
  double S[13], T[13];
  for (int i = 0; i < 13; ++i) S[i] = kf_pose[13 * (size_t)k + i];
  lc_sim3_se3(S, T);
  for (int i = 0; i < 3; ++i) O[i] = -lc_col3(T, i, T + 9);
}

__device__ __forceinline__ int hamming32(const uint4& a0, const uint4& a1, const uint4& b0, const uint4& b1) {
  return __popc(a0.x ^ b0.x) + __popc(a0.y ^ b0.y) + __popc(a0.z ^ b0.z) + __popc(a0.w ^ b0.w) +
         __popc(a1.x ^ b1.x) + __popc(a1.y ^ b1.y) + __popc(a1.z ^ b1.z) + __popc(a1.w ^ b1.w);
}

struct RefreshArgs {
  int n_sel, n_mp, n_kf, n_levels, what;
  const int32_t* idx;
  const int32_t* obeg;
  const int32_t* obs;
  const int32_t* obs_kf;   // keyframe of each observation (same layout as obs)
  const int32_t* feat_cpos;
  const uint32_t* fc_meta;
  const uint4* fc_desc;
  const int32_t* kf_fbeg;
  const double* kf_pose;
  const uint8_t* flags;
  const int32_t* ref_kf;
  MpRec* rec;
  unsigned long long* counts;
  double scale[LC_MAX_LEVELS];
};

// lane 0: normal (A36) and depth bound (A37) of point q from its ordered observations
__device__ void refresh_geometry(const RefreshArgs& a, int q, int N, const int32_t* ord,
                                 const int32_t* gobs) {
  MpRec& r = a.rec[q];
  const double p[3] = {(double)r.pos[0], (double)r.pos[1], (double)r.pos[2]};
  auto obs_at = [&](int i) -> int32_t {   // the i-th smallest feature index (A34)
    if (ord) return ord[i];
    int32_t last = INT32_MIN, cur = INT32_MAX;   // global path: O(N) per step (rare)
    for (int r0 = 0; r0 <= i; ++r0) {
      cur = INT32_MAX;
      for (int j = 0; j < N; ++j)
        if (gobs[j] > last && gobs[j] < cur) cur = gobs[j];
      last = cur;
    }
    return cur;
  };
  double acc[3] = {0.0, 0.0, 0.0};
  int nn = 0;
  for (int i = 0; i < N; ++i) {
    const int32_t f = obs_at(i);
    double O[3], v[3];
    kf_centre(a.kf_pose, kf_of_feature(a.kf_fbeg, a.n_kf, f), O);
    for (int j = 0; j < 3; ++j) v[j] = p[j] - O[j];
    const double len = sqrt((v[0] * v[0] + v[1] * v[1]) + v[2] * v[2]);
    if (len == 0.0) continue;
    for (int j = 0; j < 3; ++j) acc[j] = acc[j] + v[j] / len;
    ++nn;
  }
  if (nn > 0)
    for (int j = 0; j < 3; ++j) r.normal[j] = (float)(acc[j] / (double)nn);
  const int ref = a.ref_kf[q];
  for (int i = 0; i < N; ++i) {
    const int32_t f = obs_at(i);
    if (kf_of_feature(a.kf_fbeg, a.n_kf, f) != ref) continue;
    double O[3], v[3];
    kf_centre(a.kf_pose, ref, O);
    for (int j = 0; j < 3; ++j) v[j] = p[j] - O[j];
    const double dist = sqrt((v[0] * v[0] + v[1] * v[1]) + v[2] * v[2]);
    int lvl = (int)((a.fc_meta[a.feat_cpos[f]] >> 16) & 0xFFu);
    if (lvl >= a.n_levels) lvl = a.n_levels - 1;
    r.dmax = (float)(dist * a.scale[lvl]);
    break;
  }
}

// median (element floor((N-1)/2) of the sorted row) of distances <= 256, by counting
template <typename DistAt>
__device__ __forceinline__ int row_median(int N, DistAt dist_at) {
  const int k = (N - 1) / 2;
  int lo = 0, hi = 256;   // smallest v with #{d <= v} >= k + 1
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    int c = 0;
    for (int j = 0; j < N; ++j) c += dist_at(j) <= mid;
    if (c >= k + 1) hi = mid; else lo = mid + 1;
  }
  return lo;
}

// One point with <= 16 observations on a 16-lane group (lane gl, group mask): the full-warp
// path's expressions and orders (A34-A37), so the results are the same bits.
__device__ __forceinline__ void point_small(const RefreshArgs& a, const int q, const int b, const int N,
                                            const int gl, const unsigned mask, int32_t* tmp, int32_t* ord,
                                            int32_t* kfa, uint4 (*d)[2], double (*u)[3], double* len) {
  const int32_t* gobs = a.obs + b;
  if (gl < N) tmp[gl] = gobs[gl];
  __syncwarp(mask);
  if (gl < N) {   // A34: rank by feature index (distinct)
    const int32_t f = tmp[gl];
    int r = 0;
    for (int j = 0; j < N; ++j) r += tmp[j] < f;
    ord[r] = f;
    kfa[r] = a.obs_kf[b + gl];
  }
  __syncwarp(mask);
  if (gl < N) {
    const int cp = a.feat_cpos[ord[gl]];
    d[gl][0] = a.fc_desc[2 * (size_t)cp];
    d[gl][1] = a.fc_desc[2 * (size_t)cp + 1];
  }
  __syncwarp(mask);
  if (a.what & LC_REFRESH_DESC) {   // A35
    uint32_t best = 0xFFFFFFFFu;
    if (gl < N) {
      const uint4 x0 = d[gl][0], x1 = d[gl][1];
      int row[16];
#pragma unroll
      for (int j = 0; j < 16; ++j) row[j] = j < N ? hamming32(x0, x1, d[j][0], d[j][1]) : 1 << 20;
      const int k = (N - 1) / 2;
      int lo = 0, hi = 256;
      while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        int c = 0;
#pragma unroll
        for (int j = 0; j < 16; ++j) c += row[j] <= mid;
        if (c >= k + 1) hi = mid; else lo = mid + 1;
      }
      best = ((uint32_t)lo << 16) | (uint32_t)gl;
    }
#pragma unroll
    for (int o = 8; o > 0; o >>= 1) best = min(best, __shfl_xor_sync(mask, best, o));
    if (gl == 0) {
      const int i = (int)(best & 0xFFFFu);
      uint4* dst = reinterpret_cast<uint4*>(&a.rec[q].desc[0]);
      dst[0] = d[i][0];
      dst[1] = d[i][1];
    }
  }
  if (a.what & LC_REFRESH_NORMAL) {   // A36 / A37
    MpRec& r = a.rec[q];
    const double p[3] = {(double)r.pos[0], (double)r.pos[1], (double)r.pos[2]};
    if (gl < N) {
      const int k = kfa[gl];
      double O[3], v[3];
      kf_centre(a.kf_pose, k, O);
      for (int j = 0; j < 3; ++j) v[j] = p[j] - O[j];
      const double l = sqrt((v[0] * v[0] + v[1] * v[1]) + v[2] * v[2]);
      for (int j = 0; j < 3; ++j) u[gl][j] = l == 0.0 ? 0.0 : v[j] / l;
      len[gl] = l;
    }
    __syncwarp(mask);
    if (gl == 0) {
      double acc[3] = {0.0, 0.0, 0.0};
      int nn = 0;
      for (int i = 0; i < N; ++i) {
        if (len[i] == 0.0) continue;
        for (int j = 0; j < 3; ++j) acc[j] = acc[j] + u[i][j];
        ++nn;
      }
      if (nn > 0)
        for (int j = 0; j < 3; ++j) r.normal[j] = (float)(acc[j] / (double)nn);
      const int ref = a.ref_kf[q];
      for (int i = 0; i < N; ++i) {
        if (kfa[i] != ref) continue;
        int lvl = (int)((a.fc_meta[a.feat_cpos[ord[i]]] >> 16) & 0xFFu);
        if (lvl >= a.n_levels) lvl = a.n_levels - 1;
        r.dmax = (float)(len[i] * a.scale[lvl]);
        break;
      }
    }
  }
  __syncwarp(mask);
}

#ifndef LC_RF_MINB
#define LC_RF_MINB 5   // k_refresh CTAs per SM the register budget is cut for (shared memory allows 5)
#endif
__global__ void __launch_bounds__(LC_NTHREADS, LC_RF_MINB) k_refresh(const RefreshArgs a) {
  __shared__ int32_t s_tmp[RWARPS][OBS_CAP];
  __shared__ int32_t s_ord[RWARPS][OBS_CAP];
  __shared__ uint4 s_d[RWARPS][OBS_CAP][2];
  __shared__ double s_u[RWARPS][OBS_CAP][3];
  __shared__ double s_len[RWARPS][OBS_CAP];
  __shared__ int32_t s_kf[RWARPS][OBS_CAP];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint32_t c_mp = 0, c_obs = 0;
  // A33: the point of selection entry t, or -1 (out of range, bad, unobserved)
  auto point_of = [&](int t, int& q, int& b, int& N) {
    q = a.idx ? a.idx[t] : t;
    N = 0;
    if ((unsigned)q >= (unsigned)a.n_mp || (a.flags[q] & 1u)) return;
    b = a.obeg[q];
    N = a.obeg[q + 1] - b;
  };
  // one point with the whole warp (any N)
  auto full_point = [&](const int q, const int b, const int N) {
    if (lane == 0) { ++c_mp; c_obs += (uint32_t)N; }
    const int32_t* gobs = a.obs + b;
    if (N <= OBS_CAP) {
      // A34: rank sort by feature index (distinct), then stage the descriptors
      for (int i = lane; i < N; i += 32) s_tmp[warp][i] = gobs[i];
      __syncwarp();
      for (int i = lane; i < N; i += 32) {
        const int32_t f = s_tmp[warp][i];
        int r = 0;
        for (int j = 0; j < N; ++j) r += s_tmp[warp][j] < f;
        s_ord[warp][r] = f;
        s_kf[warp][r] = a.obs_kf[b + i];
      }
      __syncwarp();
      for (int i = lane; i < N; i += 32) {
        const int cp = a.feat_cpos[s_ord[warp][i]];
        s_d[warp][i][0] = a.fc_desc[2 * (size_t)cp];
        s_d[warp][i][1] = a.fc_desc[2 * (size_t)cp + 1];
      }
      __syncwarp();
      if (a.what & LC_REFRESH_DESC) {   // A35
        uint32_t best = 0xFFFFFFFFu;   // (median << 16) | rank
        if (N <= 16) {   // the common case: the row in registers (fully unrolled, no local memory)
          for (int i = lane; i < N; i += 32) {
            const uint4 x0 = s_d[warp][i][0], x1 = s_d[warp][i][1];
            int row[16];
#pragma unroll
            for (int j = 0; j < 16; ++j)
              row[j] = j < N ? hamming32(x0, x1, s_d[warp][j][0], s_d[warp][j][1]) : 1 << 20;
            const int k = (N - 1) / 2;
            int lo = 0, hi = 256;   // smallest v with #{d <= v} >= k + 1 (as row_median)
            while (lo < hi) {
              const int mid = (lo + hi) >> 1;
              int c = 0;
#pragma unroll
              for (int j = 0; j < 16; ++j) c += row[j] <= mid;
              if (c >= k + 1) hi = mid; else lo = mid + 1;
            }
            best = min(best, ((uint32_t)lo << 16) | (uint32_t)i);
          }
        } else {
          for (int i = lane; i < N; i += 32) {
            const uint4 x0 = s_d[warp][i][0], x1 = s_d[warp][i][1];
            uint16_t row[OBS_CAP];   // the row once; the median search then only compares
            for (int j = 0; j < N; ++j) row[j] = (uint16_t)hamming32(x0, x1, s_d[warp][j][0], s_d[warp][j][1]);
            const int med = row_median(N, [&](int j) { return (int)row[j]; });
            best = min(best, ((uint32_t)med << 16) | (uint32_t)i);
          }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) best = min(best, __shfl_xor_sync(0xffffffffu, best, o));
        if (lane == 0) {
          const int i = (int)(best & 0xFFFFu);
          uint4* d = reinterpret_cast<uint4*>(&a.rec[q].desc[0]);
          d[0] = s_d[warp][i][0];
          d[1] = s_d[warp][i][1];
        }
      }
      if (a.what & LC_REFRESH_NORMAL) {
        // per observation (one lane each): keyframe, unit viewing vector, length; then
        // lane 0 sums in observation order (A36) -- the oracle's expressions and order
        MpRec& r = a.rec[q];
        const double p[3] = {(double)r.pos[0], (double)r.pos[1], (double)r.pos[2]};
        for (int i = lane; i < N; i += 32) {
          const int k = s_kf[warp][i];
          double O[3], v[3];
          kf_centre(a.kf_pose, k, O);
          for (int j = 0; j < 3; ++j) v[j] = p[j] - O[j];
          const double len = sqrt((v[0] * v[0] + v[1] * v[1]) + v[2] * v[2]);
          for (int j = 0; j < 3; ++j) s_u[warp][i][j] = len == 0.0 ? 0.0 : v[j] / len;
          s_len[warp][i] = len;
        }
        __syncwarp();
        if (lane == 0) {
          double acc[3] = {0.0, 0.0, 0.0};
          int nn = 0;
          for (int i = 0; i < N; ++i) {
            if (s_len[warp][i] == 0.0) continue;
            for (int j = 0; j < 3; ++j) acc[j] = acc[j] + s_u[warp][i][j];
            ++nn;
          }
          if (nn > 0)
            for (int j = 0; j < 3; ++j) r.normal[j] = (float)(acc[j] / (double)nn);
          const int ref = a.ref_kf[q];
          for (int i = 0; i < N; ++i) {
            if (s_kf[warp][i] != ref) continue;
            int lvl = (int)((a.fc_meta[a.feat_cpos[s_ord[warp][i]]] >> 16) & 0xFFu);
            if (lvl >= a.n_levels) lvl = a.n_levels - 1;
            r.dmax = (float)(s_len[warp][i] * a.scale[lvl]);   // A37: |p - O_ref| of that observation
            break;
          }
        }
      }
    } else {
      // many observations: same arithmetic from global memory
      if (a.what & LC_REFRESH_DESC) {
        uint32_t best = 0xFFFFFFFFu;
        for (int i = lane; i < N; i += 32) {
          const int32_t fi = gobs[i];
          int rank = 0;
          for (int j = 0; j < N; ++j) rank += gobs[j] < fi;
          const int ci = a.feat_cpos[fi];
          const uint4 x0 = a.fc_desc[2 * (size_t)ci], x1 = a.fc_desc[2 * (size_t)ci + 1];
          const int med = row_median(N, [&](int j) {
            const int cj = a.feat_cpos[gobs[j]];
            return hamming32(x0, x1, a.fc_desc[2 * (size_t)cj], a.fc_desc[2 * (size_t)cj + 1]);
          });
          best = min(best, ((uint32_t)med << 16) | (uint32_t)rank);
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) best = min(best, __shfl_xor_sync(0xffffffffu, best, o));
        // the observation of that rank
        const uint32_t want = best & 0xFFFFu;
        for (int i = lane; i < N; i += 32) {
          const int32_t fi = gobs[i];
          uint32_t rank = 0;
          for (int j = 0; j < N; ++j) rank += gobs[j] < fi;
          if (rank == want) {
            const int ci = a.feat_cpos[fi];
            uint4* d = reinterpret_cast<uint4*>(&a.rec[q].desc[0]);
            d[0] = a.fc_desc[2 * (size_t)ci];
            d[1] = a.fc_desc[2 * (size_t)ci + 1];
          }
        }
      }
      if ((a.what & LC_REFRESH_NORMAL) && lane == 0) refresh_geometry(a, q, N, nullptr, gobs);
    }
  };
  // points are taken two at a time: when both have <= 16 observations (the common case)
  // each half-warp refreshes one (point_small, the same expressions and orders), else the
  // whole warp does them one after the other
  for (int t0 = 2 * (blockIdx.x * RWARPS + warp); t0 < a.n_sel; t0 += 2 * gridDim.x * RWARPS) {
    int qq[2] = {0, 0}, bb[2] = {0, 0}, NN[2] = {0, 0};
    point_of(t0, qq[0], bb[0], NN[0]);
    if (t0 + 1 < a.n_sel) point_of(t0 + 1, qq[1], bb[1], NN[1]);
    if (NN[0] <= 16 && NN[1] <= 16) {
      const int h = lane >> 4, gl = lane & 15;
      if (NN[h] > 0) {
        if (gl == 0) { ++c_mp; c_obs += (uint32_t)NN[h]; }
        point_small(a, qq[h], bb[h], NN[h], gl, 0xFFFFu << (16 * h), &s_tmp[warp][32 * h], &s_ord[warp][32 * h],
                    &s_kf[warp][32 * h], &s_d[warp][32 * h], &s_u[warp][32 * h], &s_len[warp][32 * h]);
      }
    } else {
      for (int h = 0; h < 2; ++h)
        if (NN[h] > 0) {
          full_point(qq[h], bb[h], NN[h]);
          __syncwarp();
        }
    }
    __syncwarp();
  }
  // counters
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    c_mp += __shfl_down_sync(0xffffffffu, c_mp, o);
    c_obs += __shfl_down_sync(0xffffffffu, c_obs, o);
  }
  if (lane == 0 && c_mp) {
    atomicAdd(&a.counts[LC_COUNT_REFRESH_MP], (unsigned long long)c_mp);
    atomicAdd(&a.counts[LC_COUNT_REFRESH_OBS], (unsigned long long)c_obs);
  }
}

__global__ void k_rec_gather(int n_mp, const MpRec* __restrict__ rec, float* __restrict__ normal,
                             float* __restrict__ dmax, uint8_t* __restrict__ desc) {
  for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < n_mp; q += gridDim.x * blockDim.x) {
    const MpRec& r = rec[q];
    if (normal) { normal[3 * q] = r.normal[0]; normal[3 * q + 1] = r.normal[1]; normal[3 * q + 2] = r.normal[2]; }
    if (dmax) dmax[q] = r.dmax;
    if (desc)
      for (int i = 0; i < 32; ++i) desc[32 * (size_t)q + i] = reinterpret_cast<const uint8_t*>(r.desc)[i];
  }
}

int grid_of(int64_t n, int per_block) {
  int64_t b = (n + per_block - 1) / per_block;
  return (int)std::max<int64_t>(1, std::min<int64_t>(b, 148 * 32));
}

}  // namespace

cudaError_t launch_obs_lists(lc_ctx* c, int32_t* d_obeg, int32_t* d_cursor, int32_t* d_bsum,
                             int32_t* d_obs, int32_t* d_obs_kf, cudaStream_t s) {
  Store& st = c->st;
  if (st.n_mp <= 0) return cudaSuccess;
  const int nb = (st.n_mp + SCAN_SEG - 1) / SCAN_SEG;
  k_scan_a<<<nb, LC_NTHREADS, 0, s>>>(st.mp_nobs, st.n_mp, d_obeg, d_bsum);
  k_scan_b<<<1, LC_NTHREADS, 0, s>>>(d_bsum, nb, d_obeg + st.n_mp);
  k_scan_c<<<(st.n_mp + LC_NTHREADS - 1) / LC_NTHREADS, LC_NTHREADS, 0, s>>>(d_obeg, st.n_mp, d_bsum, d_cursor);
  k_obs_fill<<<std::max(1, std::min(st.n_kf, 148 * 16)), LC_NTHREADS, 0, s>>>(
      st.n_kf, st.n_mp, st.kf_fbeg, st.feat_mp, d_obeg, d_cursor, d_obs, d_obs_kf);
  c->launches += 4;
  return cudaGetLastError();
}

int obs_scan_blocks(int n_mp) { return (n_mp + SCAN_SEG - 1) / SCAN_SEG; }

cudaError_t launch_refresh(lc_ctx* c, int n_sel, const int32_t* d_idx, int what, int32_t* d_obeg,
                           int32_t* d_cursor, int32_t* d_bsum, int32_t* d_obs, int32_t* d_obs_kf,
                           unsigned long long* counts, cudaStream_t s) {
  Store& st = c->st;
  if (st.n_mp <= 0) return cudaSuccess;
  cudaError_t e = launch_obs_lists(c, d_obeg, d_cursor, d_bsum, d_obs, d_obs_kf, s);
  if (e != cudaSuccess) return e;
  if (n_sel > 0) {
    RefreshArgs a;
    a.n_sel = n_sel; a.n_mp = st.n_mp; a.n_kf = st.n_kf; a.n_levels = st.n_levels; a.what = what;
    a.idx = d_idx; a.obeg = d_obeg; a.obs = d_obs; a.obs_kf = d_obs_kf; a.feat_cpos = st.feat_cpos; a.fc_meta = st.fc_meta;
    a.fc_desc = st.fc_desc; a.kf_fbeg = st.kf_fbeg; a.kf_pose = st.kf_pose; a.flags = st.mp_flags;
    a.ref_kf = st.mp_ref_kf; a.rec = st.mp_rec; a.counts = counts;
    for (int i = 0; i < LC_MAX_LEVELS; ++i) a.scale[i] = st.scale[i];
    k_refresh<<<grid_of(n_sel, RWARPS), LC_NTHREADS, 0, s>>>(a);
    c->launches++;
  }
  return cudaGetLastError();
}

cudaError_t launch_download_rec(lc_ctx* c, float* normal, float* dmax, uint8_t* desc, cudaStream_t s) {
  if (c->st.n_mp <= 0 || (!normal && !dmax && !desc)) return cudaSuccess;
  k_rec_gather<<<grid_of(c->st.n_mp, LC_NTHREADS), LC_NTHREADS, 0, s>>>(c->st.n_mp, c->st.mp_rec, normal,
                                                                        dmax, desc);
  c->launches++;
  return cudaGetLastError();
}
