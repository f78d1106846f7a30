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

#include "lc_internal.cuh"

namespace {

constexpr unsigned long long NONE = 0x7FFFFFFFFFFFFFFFull;

// local per-thread counters of the matching kernel (subset of LC_COUNT_*)
enum { M_QUERIES, M_BAD, M_FOUND, M_DEPTH, M_BOUNDS, M_DIST, M_ANGLE, M_CAND, M_NOCAND,
       M_OVERTH, M_RATIO, M_PROP, M_N };
__device__ __constant__ int kMatchSlot[M_N] = {
    LC_COUNT_QUERIES, LC_COUNT_SKIP_BAD, LC_COUNT_SKIP_FOUND, LC_COUNT_CULL_DEPTH,
    LC_COUNT_CULL_BOUNDS, LC_COUNT_CULL_DIST, LC_COUNT_CULL_ANGLE, LC_COUNT_CANDIDATES,
    LC_COUNT_NO_CAND, LC_COUNT_OVER_TH, LC_COUNT_RATIO_REJ, LC_COUNT_PROPOSALS};

__device__ __forceinline__ uint32_t hash_slot(int32_t key, int shift) {
  return ((uint32_t)key * 2654435769u) >> shift;
}

__device__ __forceinline__ void hash_insert(int32_t* tab, int mask, int shift, int32_t key) {
  uint32_t h = hash_slot(key, shift);
  while (true) {
    int32_t prev = atomicCAS(&tab[h], -1, key);
    if (prev == -1 || prev == key) return;
    h = (h + 1) & mask;
  }
}

__device__ __forceinline__ bool hash_contains(const int32_t* tab, int mask, int shift, int32_t key) {
  uint32_t h = hash_slot(key, shift);
  while (true) {
    int32_t v = tab[h];
    if (v == key) return true;
    if (v == -1) return false;
    h = (h + 1) & mask;
  }
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
// MODE 0: fuse (already found = associated in the keyframe)
// MODE 1: projection search (already found = pair_taken; taken features excluded)
// ---------------------------------------------------------------------------
template <int MODE>
__global__ void __launch_bounds__(LC_NTHREADS) k_project_match(const MatchArgs a) {
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ double s_T[12];  // R row-major, tt = t / s
  __shared__ double s_Ow[3];
  __shared__ DevCam s_cam;
  const int unit = a.blk_unit[blockIdx.x];
  const int k = a.unit_kf[unit];
  const int fb = a.kf_fbeg[k];
  const int F = a.kf_fbeg[k + 1] - fb;
  const int H = a.hash_size;
  const int hmask = H - 1;
  const int hshift = 32 - __ffs(H) + 1;
  float2* s_uv = (float2*)smem;
  uint32_t* s_meta = (uint32_t*)(s_uv + F);
  int32_t* s_hash = (int32_t*)(s_meta + F);
  uint16_t* s_cell = (uint16_t*)(s_hash + H);
  const int G1 = a.G + 1;
  const int64_t toff = (MODE == 1 && a.taken) ? a.unit_toff[unit] : 0;

  // ---- stage the keyframe ------------------------------------------------------
  for (int i = threadIdx.x; i < H; i += blockDim.x) s_hash[i] = -1;
  const uint16_t* gcell = a.kf_cell + (size_t)k * G1;
  for (int i = threadIdx.x; i < G1; i += blockDim.x) s_cell[i] = gcell[i];
  for (int p = threadIdx.x; p < F; p += blockDim.x) {
    s_uv[p] = a.fc_uv[fb + p];
    uint32_t m = a.fc_meta[fb + p];
    if (MODE == 1 && a.taken && a.taken[toff + (m & 0xFFFFu)] >= 0) m |= 0x80000000u;
    s_meta[p] = m;
  }
  if (threadIdx.x == 0) {
    double S[13], T[13];
    const double* src = a.unit_S ? a.unit_S + 13 * (size_t)unit : a.kf_S_corr + 13 * (size_t)k;
    for (int i = 0; i < 13; ++i) S[i] = src[i];
    lc_sim3_se3(S, T);  // reading A2: project with (R, t/s)
    for (int i = 0; i < 12; ++i) s_T[i] = T[i];
    for (int i = 0; i < 3; ++i) s_Ow[i] = -lc_col3(T, i, T + 9);
    s_cam = a.cams[a.kf_cam[k]];
  }
  __syncthreads();
  for (int f = threadIdx.x; f < F; f += blockDim.x) {
    int32_t m = (MODE == 0) ? a.feat_mp[fb + f] : (a.taken ? a.taken[toff + f] : -1);
    if (m >= 0) hash_insert(s_hash, hmask, hshift, m);
  }
  __syncthreads();

  const lc_match_params prm = a.params[(MODE == 1 && a.unit_param) ? a.unit_param[unit] : 0];
  const double R0 = s_T[0], R1 = s_T[1], R2 = s_T[2], R3 = s_T[3], R4 = s_T[4], R5 = s_T[5];
  const double R6 = s_T[6], R7 = s_T[7], R8 = s_T[8], t0 = s_T[9], t1 = s_T[10], t2 = s_T[11];
  const double Ow0 = s_Ow[0], Ow1 = s_Ow[1], Ow2 = s_Ow[2];
  const int L = a.n_levels;
  const double sLm1 = a.scale[L - 1];
  const int cols = a.cols, rows = a.rows;
  unsigned long long* win = a.winner + a.unit_woff[unit];
  const int64_t lbeg = a.unit_lbeg[unit];
  const int64_t qoff = a.unit_qoff[unit];
  uint32_t cnt[M_N];
#pragma unroll
  for (int i = 0; i < M_N; ++i) cnt[i] = 0;

  const int64_t q1 = a.blk_q1[blockIdx.x];
  for (int64_t j = a.blk_q0[blockIdx.x] + threadIdx.x; j < q1; j += blockDim.x) {
    const int32_t q = a.mp_list[j];
    const int64_t qi = qoff + (j - lbeg);
    cnt[M_QUERIES]++;
    int status = 0;
    double u = 0.0, v = 0.0;
    int ncand = 0;
    uint32_t best = 0xFFFFFFFFu;  // (H << 16) | f
    int second = 256;
    do {
      if ((unsigned)q >= (unsigned)a.n_mp || (a.mp_flags[q] & 1u)) {  // out of range: as bad
        status = LC_Q_BAD; cnt[M_BAD]++; break;
      }
      if (hash_contains(s_hash, hmask, hshift, q)) { status = LC_Q_FOUND; cnt[M_FOUND]++; break; }
      const uint4* rp = reinterpret_cast<const uint4*>(a.mp_rec + q);
      const uint4 w0 = __ldg(rp + 0), w1 = __ldg(rp + 1);
      const double p0 = __uint_as_float(w0.x), p1 = __uint_as_float(w0.y), p2 = __uint_as_float(w0.z);
      const double dmax = __uint_as_float(w0.w);
      const double n0 = __uint_as_float(w1.x), n1 = __uint_as_float(w1.y), n2 = __uint_as_float(w1.z);
      const double x = (R0 * p0 + R1 * p1) + R2 * p2 + t0;
      const double y = (R3 * p0 + R4 * p1) + R5 * p2 + t1;
      const double z = (R6 * p0 + R7 * p1) + R8 * p2 + t2;
      if (z <= 0.0) { status = LC_Q_DEPTH; cnt[M_DEPTH]++; break; }
      lc_project(s_cam, x, y, z, u, v);
      if (!(u >= s_cam.min_x && u < s_cam.max_x && v >= s_cam.min_y && v < s_cam.max_y)) {
        status = LC_Q_BOUNDS; cnt[M_BOUNDS]++; break;
      }
      const double PO0 = p0 - Ow0, PO1 = p1 - Ow1, PO2 = p2 - Ow2;
      const double d = sqrt((PO0 * PO0 + PO1 * PO1) + PO2 * PO2);
      const double dmin_i = 0.8 * (dmax / sLm1);
      const double dmax_i = 1.2 * dmax;
      if (d < dmin_i || d > dmax_i) { status = LC_Q_DIST; cnt[M_DIST]++; break; }
      if ((PO0 * n0 + PO1 * n1) + PO2 * n2 < 0.5 * d) { status = LC_Q_ANGLE; cnt[M_ANGLE]++; break; }
      int lvl = L - 1;
      for (int n = 0; n < L; ++n)
        if (d * a.scale[n] >= dmax) { lvl = n; break; }
      const double r = (double)prm.th * a.scale[lvl];
      // candidate cells: conservative (1e-6 cell) superset of the exact square window
      int cx0 = (int)fmax(0.0, floor(((u - r) - s_cam.min_x) * s_cam.cell_sx - 1e-6));
      int cx1 = (int)fmin((double)(cols - 1), floor(((u + r) - s_cam.min_x) * s_cam.cell_sx + 1e-6));
      int cy0 = (int)fmax(0.0, floor(((v - r) - s_cam.min_y) * s_cam.cell_sy - 1e-6));
      int cy1 = (int)fmin((double)(rows - 1), floor(((v + r) - s_cam.min_y) * s_cam.cell_sy + 1e-6));
      const uint4 d0 = __ldg(rp + 2), d1 = __ldg(rp + 3);
      const int lo = lvl - 1;
      for (int cy = cy0; cy <= cy1; ++cy) {
        const int pb = s_cell[cy * cols + cx0], pe = s_cell[cy * cols + cx1 + 1];
        for (int p = pb; p < pe; ++p) {
          const uint32_t meta = s_meta[p];
          const int oct = (int)((meta >> 16) & 0xFFu);
          if (oct < lo || oct > lvl) continue;
          if (MODE == 1 && (meta & 0x80000000u)) continue;
          const float2 fuv = s_uv[p];
          const double du = fabs((double)fuv.x - u), dv = fabs((double)fuv.y - v);
          if (!(du < r && dv < r)) continue;
          ++ncand;
          const uint4* dp = a.fc_desc + 2 * (size_t)(fb + p);
          const int h = popc_desc(d0, d1, __ldg(dp), __ldg(dp + 1));
          const uint32_t key = ((uint32_t)h << 16) | (meta & 0xFFFFu);
          if (key < best) {
            if (best != 0xFFFFFFFFu) second = min(second, (int)(best >> 16));
            best = key;
          } else {
            second = min(second, h);
          }
        }
      }
      cnt[M_CAND] += ncand;
      if (ncand == 0) { cnt[M_NOCAND]++; break; }
      const int hb = (int)(best >> 16);
      if (hb > prm.max_hamming) { cnt[M_OVERTH]++; break; }
      if (prm.ratio_den > 0 &&
          (long long)prm.ratio_den * hb > (long long)prm.ratio_num * second) {
        cnt[M_RATIO]++; break;
      }
      cnt[M_PROP]++;
      atomicMin(&win[best & 0xFFFFu], ((unsigned long long)hb << 32) | (unsigned int)q);
    } while (0);
    if (a.dbg_best) {
      long long val;
      if (status < 0) val = status;
      else if (ncand == 0) val = (256LL << 48) | (256LL << 32) | 0xFFFFFFFFLL;
      else val = ((long long)(best >> 16) << 48) | ((long long)second << 32) | (long long)(best & 0xFFFFu);
      a.dbg_best[qi] = val;
    }
    if (a.dbg_uv) { a.dbg_uv[2 * qi] = u; a.dbg_uv[2 * qi + 1] = v; }
    if (a.dbg_ncand) a.dbg_ncand[qi] = ncand;
  }
  unsigned long long* cdst = a.counts + (MODE == 1 ? (size_t)unit * LC_NCOUNT : 0);
  block_add<M_N>(cnt, kMatchSlot, cdst);
}

// Orientation filter + fuse actions (MODE 0) / output tables (MODE 1); one CTA per unit.
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
__global__ void __launch_bounds__(LC_NTHREADS) k_resolve(
    const int32_t* __restrict__ unit_kf, const int64_t* __restrict__ unit_woff,
    const int64_t* __restrict__ unit_toff, const int32_t* __restrict__ unit_param,
    const lc_match_params* __restrict__ params, const int32_t* __restrict__ kf_fbeg,
    const int32_t* __restrict__ feat_mp, const float* __restrict__ feat_angle,
    const MpRec* __restrict__ mp_rec, const uint8_t* __restrict__ mp_flags,
    const uint32_t* __restrict__ loop_ep, uint32_t epoch, const int32_t* __restrict__ taken,
    unsigned long long* __restrict__ winner, unsigned long long* __restrict__ victim,
    int8_t* __restrict__ action, int32_t* __restrict__ out_mp, int32_t* __restrict__ out_dist,
    unsigned long long* __restrict__ counts) {
  __shared__ int s_hist[30];
  __shared__ int s_keep[3];
  const int unit = blockIdx.x;
  const int k = unit_kf[unit];
  const int fb = kf_fbeg[k], F = kf_fbeg[k + 1] - fb;
  const int64_t woff = unit_woff[unit];
  const int64_t toff = (MODE == 1 && taken) ? unit_toff[unit] : 0;
  const lc_match_params prm = params[(MODE == 1 && unit_param) ? unit_param[unit] : 0];
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
      atomicAdd(&s_hist[rot_bin(feat_angle[fb + f], mp_rec[q].angle)], 1);
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
  for (int f = threadIdx.x; f < F; f += blockDim.x) {
    unsigned long long w = winner[woff + f];
    int8_t act = 0;
    if (w != NONE) {
      cnt[R_WINNERS]++;
      int q = (int)(w & 0xFFFFFFFFull);
      if (prm.check_orientation) {
        int b = rot_bin(feat_angle[fb + f], mp_rec[q].angle);
        if (b != s_keep[0] && b != s_keep[1] && b != s_keep[2]) {
          w = NONE;
          winner[woff + f] = NONE;
          cnt[R_ORIENT]++;
          act = 4;
        }
      }
      if (MODE == 0 && w != NONE) {
        int slot = feat_mp[fb + f];
        if (slot < 0) { act = 1; cnt[R_ADD]++; }
        else if (mp_flags[slot] & 1u) { act = 5; cnt[R_BADSLOT]++; }
        else if (loop_ep[slot] == epoch) { act = 3; cnt[R_LOOP]++; }
        else { act = 2; cnt[R_VICTIM]++; atomicMin(&victim[slot], w); }
      }
    }
    if (MODE == 0) {
      if (action) action[woff + f] = act;
    } else {
      int t = taken ? taken[toff + f] : -1;
      if (t >= 0) { out_mp[woff + f] = t; out_dist[woff + f] = -1; }
      else if (w != NONE) { out_mp[woff + f] = (int)(w & 0xFFFFFFFFull); out_dist[woff + f] = (int)(w >> 32); }
      else { out_mp[woff + f] = -1; out_dist[woff + f] = -1; }
    }
  }
  unsigned long long* cdst = counts + (MODE == 1 ? (size_t)unit * LC_NCOUNT : 0);
  block_add<R_N>(cnt, kResolveSlot, cdst);
}

// Per-call setup: LoopSet stamps, winner/victim init, window membership.
__global__ void k_fuse_prep(int phase, uint32_t epoch, int n_w, const int32_t* __restrict__ window,
                            int64_t n_wfeat, const int32_t* __restrict__ mp_list, int64_t n_list,
                            int n_mp, unsigned long long* __restrict__ winner,
                            unsigned long long* __restrict__ victim, uint32_t* __restrict__ loop_ep,
                            uint32_t* __restrict__ kf_win_ep, int32_t* __restrict__ kf_win_pos) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const int64_t t0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  for (int64_t i = t0; i < n_w; i += stride) {
    kf_win_ep[window[i]] = epoch;
    kf_win_pos[window[i]] = (int32_t)i;
  }
  if (!(phase & LC_FUSE_PLAN)) return;
  for (int64_t i = t0; i < n_list; i += stride) {
    const int32_t q = mp_list[i];
    if ((unsigned)q < (unsigned)n_mp) loop_ep[q] = epoch;
  }
  for (int64_t i = t0; i < n_wfeat; i += stride) winner[i] = NONE;
  for (int64_t i = t0; i < n_mp; i += stride) victim[i] = NONE;
}

// Victim marking: flags |= bad, replaced_by = survivor (reading O9 (iv)).
__global__ void k_fuse_victims(int n_mp, const unsigned long long* __restrict__ victim,
                               uint8_t* __restrict__ flags, int32_t* __restrict__ replaced_by,
                               unsigned long long* __restrict__ counts) {
  uint32_t n = 0;
  for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < n_mp; q += gridDim.x * blockDim.x) {
    unsigned long long v = victim[q];
    if (v == NONE) continue;
    flags[q] |= 1u;
    replaced_by[q] = (int32_t)(v & 0xFFFFFFFFull);
    ++n;
  }
  const int slot[1] = {LC_COUNT_VICTIMS};
  uint32_t loc[1] = {n};
  block_add<1>(loc, slot, counts);
}

// Apply: redirect victims map-wide, add winners to empty window slots, per-keyframe
// duplicate cleanup by least (priority, f), n_obs deltas. One CTA per keyframe.
enum { A_REWIRED, A_DUP, A_ADDED, A_N };
__device__ __constant__ int kApplySlot[A_N] = {LC_COUNT_REWIRED, LC_COUNT_DUP_CLEARED,
                                               LC_COUNT_ADDED};

__global__ void __launch_bounds__(LC_NTHREADS) k_fuse_apply(
    uint32_t epoch, const int32_t* __restrict__ kf_fbeg, const uint32_t* __restrict__ kf_win_ep,
    const int32_t* __restrict__ kf_win_pos, const int64_t* __restrict__ woff_of_pos,
    const unsigned long long* __restrict__ winner, const unsigned long long* __restrict__ victim,
    int32_t* __restrict__ feat_mp, int32_t* __restrict__ nobs, int hash_size,
    unsigned long long* __restrict__ counts) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int k = blockIdx.x;
  const int fb = kf_fbeg[k], F = kf_fbeg[k + 1] - fb;
  const int wpos = (kf_win_ep[k] == epoch) ? kf_win_pos[k] : -1;
  const int64_t woff = wpos >= 0 ? woff_of_pos[wpos] : 0;
  int32_t* s_new = (int32_t*)smem;
  int32_t* s_old = s_new + F;
  int32_t* s_key = s_old + F;
  uint32_t* s_val = (uint32_t*)(s_key + hash_size);
  uint8_t* s_pr = (uint8_t*)(s_val + hash_size);
  uint32_t cnt[A_N] = {0, 0, 0};
  int any = 0;
  for (int f = threadIdx.x; f < F; f += blockDim.x) {
    int32_t m = feat_mp[fb + f];
    int32_t nv = m;
    uint8_t pr = 0;
    if (m >= 0) {
      unsigned long long vw = victim[m];
      if (vw != NONE) { nv = (int32_t)(vw & 0xFFFFFFFFull); pr = 2; cnt[A_REWIRED]++; }
    } else if (wpos >= 0) {
      unsigned long long w = winner[woff + f];
      if (w != NONE) { nv = (int32_t)(w & 0xFFFFFFFFull); pr = 1; }
    }
    s_old[f] = m;
    s_new[f] = nv;
    s_pr[f] = pr;
    any |= (pr != 0);
  }
  any = __syncthreads_or(any);
  if (any) {
    const int hmask = hash_size - 1;
    const int hshift = 32 - __ffs(hash_size) + 1;
    for (int i = threadIdx.x; i < hash_size; i += blockDim.x) { s_key[i] = -1; s_val[i] = 0xFFFFFFFFu; }
    __syncthreads();
    for (int f = threadIdx.x; f < F; f += blockDim.x) {
      int32_t nv = s_new[f];
      if (nv < 0) continue;
      uint32_t h = hash_slot(nv, hshift);
      while (true) {
        int32_t prev = atomicCAS(&s_key[h], -1, nv);
        if (prev == -1 || prev == nv) break;
        h = (h + 1) & hmask;
      }
      atomicMin(&s_val[h], ((uint32_t)s_pr[f] << 16) | (uint32_t)f);
    }
    __syncthreads();
    for (int f = threadIdx.x; f < F; f += blockDim.x) {
      int32_t nv = s_new[f];
      const int32_t m = s_old[f];
      if (nv >= 0) {
        uint32_t h = hash_slot(nv, hshift);
        while (s_key[h] != nv) h = (h + 1) & hmask;
        if (s_val[h] != (((uint32_t)s_pr[f] << 16) | (uint32_t)f)) { nv = -1; cnt[A_DUP]++; }
        else if (s_pr[f] == 1) cnt[A_ADDED]++;
      }
      if (nv != m) {
        feat_mp[fb + f] = nv;
        if (m >= 0) atomicSub(&nobs[m], 1);
        if (nv >= 0) atomicAdd(&nobs[nv], 1);
      }
    }
  }
  block_add<A_N>(cnt, kApplySlot, counts);
}

int grid_for(int64_t n) {
  int64_t b = (n + LC_NTHREADS - 1) / LC_NTHREADS;
  if (b < 1) b = 1;
  if (b > 148 * 16) b = 148 * 16;
  return (int)b;
}

int pow2_at_least(int x) {
  int h = 64;
  while (h < x) h <<= 1;
  return h;
}

}  // namespace

cudaError_t launch_match(lc_ctx* c, int mode, const MatchArgs& a_in, int n_blocks, int F_max,
                         cudaStream_t s) {
  if (n_blocks <= 0) return cudaSuccess;
  MatchArgs a = a_in;
  a.hash_size = pow2_at_least(2 * (F_max > 0 ? F_max : 1));
  size_t smem = (size_t)F_max * 12 + (size_t)a.hash_size * 4 + (size_t)(a.G + 1) * 2;
  smem = (smem + 15) & ~(size_t)15;
  cudaError_t e;
  if (mode == 0) {
    e = cudaFuncSetAttribute(k_project_match<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    k_project_match<0><<<n_blocks, LC_NTHREADS, smem, s>>>(a);
  } else {
    e = cudaFuncSetAttribute(k_project_match<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    k_project_match<1><<<n_blocks, LC_NTHREADS, smem, s>>>(a);
  }
  c->launches++;
  return cudaGetLastError();
}

cudaError_t launch_fuse_prep(lc_ctx* c, int phase, int n_w, const int32_t* d_window,
                             const int64_t* d_woff, int64_t n_wfeat, const int32_t* mp_list,
                             int64_t n_list_total, unsigned long long* winner,
                             unsigned long long* victim, cudaStream_t s) {
  (void)d_woff;
  int64_t n = n_w;
  if (phase & LC_FUSE_PLAN) {
    n = n > n_list_total ? n : n_list_total;
    n = n > n_wfeat ? n : n_wfeat;
    n = n > c->st.n_mp ? n : c->st.n_mp;
  }
  k_fuse_prep<<<grid_for(n), LC_NTHREADS, 0, s>>>(phase, c->epoch, n_w, d_window, n_wfeat, mp_list,
                                                 n_list_total, c->st.n_mp, winner, victim,
                                                 c->st.mp_loop_ep, c->st.kf_win_ep, c->st.kf_win_pos);
  c->launches++;
  return cudaGetLastError();
}

cudaError_t launch_fuse_resolve(lc_ctx* c, int mode, int n_units, const int32_t* unit_kf,
                                const int64_t* unit_woff, const int64_t* unit_toff,
                                const int32_t* unit_param, const lc_match_params* params,
                                const int32_t* taken, unsigned long long* winner,
                                unsigned long long* victim, int8_t* action, int32_t* out_mp,
                                int32_t* out_dist, unsigned long long* counts, int F_max,
                                cudaStream_t s) {
  (void)F_max;
  if (n_units <= 0) return cudaSuccess;
  Store& st = c->st;
  if (mode == 0)
    k_resolve<0><<<n_units, LC_NTHREADS, 0, s>>>(unit_kf, unit_woff, unit_toff, unit_param, params,
                                                 st.kf_fbeg, st.feat_mp, st.feat_angle, st.mp_rec,
                                                 st.mp_flags, st.mp_loop_ep, c->epoch, taken,
                                                 winner, victim, action, out_mp, out_dist, counts);
  else
    k_resolve<1><<<n_units, LC_NTHREADS, 0, s>>>(unit_kf, unit_woff, unit_toff, unit_param, params,
                                                 st.kf_fbeg, st.feat_mp, st.feat_angle, st.mp_rec,
                                                 st.mp_flags, st.mp_loop_ep, c->epoch, taken,
                                                 winner, victim, action, out_mp, out_dist, counts);
  c->launches++;
  return cudaGetLastError();
}

cudaError_t launch_fuse_apply(lc_ctx* c, const int64_t* d_woff, const unsigned long long* winner,
                              const unsigned long long* victim, unsigned long long* counts,
                              cudaStream_t s) {
  Store& st = c->st;
  if (st.n_mp > 0) {
    k_fuse_victims<<<grid_for(st.n_mp), LC_NTHREADS, 0, s>>>(st.n_mp, victim, st.mp_flags,
                                                             st.mp_replaced_by, counts);
    c->launches++;
  }
  if (st.n_kf > 0) {
    int H = pow2_at_least(2 * (st.max_F > 0 ? st.max_F : 1));
    size_t smem = (size_t)st.max_F * 9 + (size_t)H * 8;
    smem = (smem + 15) & ~(size_t)15;
    cudaError_t e = cudaFuncSetAttribute(k_fuse_apply, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    k_fuse_apply<<<st.n_kf, LC_NTHREADS, smem, s>>>(c->epoch, st.kf_fbeg, st.kf_win_ep, st.kf_win_pos,
                                                   d_woff, winner, victim, st.feat_mp, st.mp_nobs,
                                                   H, counts);
    c->launches++;
  }
  return cudaGetLastError();
}
