// k_correct.cu -- Sim3 correction of keyframes and map points.
//
// WINDOW (§III.B "correcting their poses using the estimated Sim3
// transformation"; reading O3) and ALL ("propagates the loop
// correction to the rest of the map"; reading O10). Both are
// streaming passes over the map-point records (HBM-bound); the per-keyframe
// transforms are computed once into a small scratch table first, so every point
// applies two precomputed Sim3s in fp64 (loaded as 16-B vectors, L1-resident when
// consecutive map points share their keyframe, as in creation order).
//
// WINDOW = 3 kernels (+2 memsets): S^corr per window position, owner election, then
// [point re-anchoring || pose write-back]; ALL = 2 kernels.
#include <cuda_runtime.h>

#include <algorithm>

#include "lc_internal.cuh"

namespace {

// WINDOW scratch per window position i (16-B aligned rows of WSTR doubles):
//   [0, 13) T_iw^old | [14, 27) inverse(S_i^corr) | [28, 41) S_i^corr | [42, 55) SE3(S_i^corr)
constexpr int WSTR = 56;
// ALL scratch per keyframe: [0, 13) S^pre | [14, 27) inverse(S^opt)
constexpr int ASTR = 28;
constexpr int32_t OWNER_NONE = 0x7F7F7F7F;  // memset byte pattern 0x7F
#ifndef LC_PT_MINB
#ifndef LC_PT_MINB
#define LC_PT_MINB 2   // point kernels: CTAs per SM the register budget is cut for
#endif
#endif
#ifndef LC_OWN_PRECHECK
#define LC_OWN_PRECHECK 0
#endif

// owner election step: a plain (possibly stale) read can only over-estimate the
// current owner, so skipping the reduction when it is already <= i is exact
__device__ __forceinline__ void own_min(int32_t* owner, int m, int i) {
#if LC_OWN_PRECHECK
  if (owner[m] <= i) return;
#endif
  atomicMin(&owner[m], i);
}

// (a predecessor's output read after the PDL wait: plain coherent loads through a pointer
// without __restrict__ -- an ld.global.nc / const __restrict__ load may be scheduled above
// griddepcontrol.wait)
__device__ __forceinline__ void load13(const double* src, double* d) {
  const double2* s2 = reinterpret_cast<const double2*>(src);
#pragma unroll
  for (int i = 0; i < 6; ++i) {
    const double2 x = s2[i];
    d[2 * i] = x.x;
    d[2 * i + 1] = x.y;
  }
  d[12] = src[12];
}

__device__ __forceinline__ void warp_count(uint32_t n, unsigned long long* dst) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) n += __shfl_down_sync(0xffffffffu, n, o);
  if ((threadIdx.x & 31) == 0 && n) atomicAdd(dst, (unsigned long long)n);
}

// Thread i = window position i: S_i^corr = (T_iw * inverse(T_cw)) * S_cw^corr from the
// OLD poses (S_c^corr = S_cw^corr) into scratch, with T_iw^old and inverse(S_i^corr).
__global__ void k_win_sim3(int n_w, int cur_pos, const int32_t* __restrict__ window,
                           const double* __restrict__ kf_pose, const double* __restrict__ Scw,
                           double* __restrict__ scr,
                           double* __restrict__ kf_S_corr, int32_t* __restrict__ kf_in_win,
                           double* __restrict__ out_S, unsigned long long* __restrict__ counts) {
  pdl_trigger();   // k_win_mark reads none of this kernel's outputs
  if (blockIdx.x == 0 && threadIdx.x < LC_NCOUNT) counts[threadIdx.x] = 0;   // the call's counters
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n_w) return;
  const int k = window[i];
  double T[13], S[13], Si[13];
  for (int j = 0; j < 13; ++j) T[j] = kf_pose[13 * (size_t)k + j];
  if (i == cur_pos) {
    for (int j = 0; j < 13; ++j) S[j] = Scw[j];
  } else {
    double Tc[13], Tci[13], Sic[13];
    const int c = window[cur_pos];
    for (int j = 0; j < 13; ++j) Tc[j] = kf_pose[13 * (size_t)c + j];
    lc_sim3_inverse(Tc, Tci);
    lc_sim3_compose(T, Tci, Sic);   // S_ic = T_iw * inverse(T_cw)
    lc_sim3_compose(Sic, Scw, S);   // S_iw^corr = S_ic * S_cw^corr
  }
  lc_sim3_inverse(S, Si);
  double* o = scr + (size_t)WSTR * i;
  for (int j = 0; j < 13; ++j) { o[j] = T[j]; o[14 + j] = Si[j]; o[28 + j] = S[j]; }
  lc_sim3_se3(S, T);
  for (int j = 0; j < 13; ++j) o[42 + j] = T[j];
  o[13] = o[27] = o[41] = o[55] = 0.0;
  for (int j = 0; j < 13; ++j) kf_S_corr[13 * (size_t)k + j] = S[j];
  if (out_S)
    for (int j = 0; j < 13; ++j) out_S[13 * (size_t)i + j] = S[j];
  kf_in_win[k] = 1;
}

// Warp per window position: owner(m) = min window position observing map point m
// (fire-and-forget atomicMin reductions), 16-B association loads. Bad map points get an
// owner too; k_win_b ignores them (it reads the flags coalesced, per point).
__global__ void __launch_bounds__(LC_NTHREADS) k_win_mark(
    int n_w, const int32_t* __restrict__ window, const int32_t* __restrict__ kf_fbeg,
    const int32_t* __restrict__ feat_mp, int32_t* owner) {
  const int lane = threadIdx.x & 31;
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  for (int i = gw; i < n_w; i += nw) {
    const int k = window[i];
    const int fb = kf_fbeg[k], fe = kf_fbeg[k + 1];
    const int vb = min(fe, (fb + 3) & ~3), ve = max(vb, fe & ~3);
    for (int f = fb + lane; f < vb; f += 32) {
      const int m = feat_mp[f];
      if (m >= 0) own_min(owner, m, i);
    }
    for (int f = vb + 4 * lane; f < ve; f += 128) {
      const int4 m4 = __ldg(reinterpret_cast<const int4*>(feat_mp + f));
      if (m4.x >= 0) own_min(owner, m4.x, i);
      if (m4.y >= 0) own_min(owner, m4.y, i);
      if (m4.z >= 0) own_min(owner, m4.z, i);
      if (m4.w >= 0) own_min(owner, m4.w, i);
    }
    for (int f = ve + lane; f < fe; f += 32) {
      const int m = feat_mp[f];
      if (m >= 0) own_min(owner, m, i);
    }
  }
  pdl_wait();   // (PDL) independent of k_win_sim3; completes after it
}

// Blocks [0, nb_mp): p <- fl32( inverse(S_o^corr)( T_o,w^old(p) ) ), corr_ref <- window[o]
// (or -1); blocks [nb_mp, ...): window pose write-back T_iw <- SE3(S_i^corr).
__global__ void __launch_bounds__(LC_NTHREADS, LC_PT_MINB) k_win_b(
    int n_mp, int nb_mp, int n_w, int mp_lo, int mp_hi, const int32_t* owner, const uint8_t* __restrict__ flags,
    const int32_t* __restrict__ window, const double* scr, MpRec* __restrict__ rec,
    int32_t* __restrict__ corr_ref, double* __restrict__ kf_pose,
    unsigned long long* __restrict__ counts) {
  uint32_t n = 0;
  if ((int)blockIdx.x < nb_mp) {   // two adjacent points per thread (2 nb_mp blockDim.x >= n_mp)
    const int q0 = 2 * (blockIdx.x * blockDim.x + threadIdx.x);
    uint8_t fl[2] = {1, 1};
    float4 pf[2];
#pragma unroll
    for (int u = 0; u < 2; ++u) {   // independent of the predecessors: before the PDL wait
      pf[u] = make_float4(0.f, 0.f, 0.f, 0.f);
      if (q0 + u < n_mp) fl[u] = flags[q0 + u];
    }
    pdl_wait();
    int o[2] = {OWNER_NONE, OWNER_NONE};
#pragma unroll
    for (int u = 0; u < 2; ++u)
      if (q0 + u < n_mp) o[u] = owner[q0 + u];
    // the records only of the points this pass re-anchors (owned, not bad, this rank's
    // slice): the map points no window keyframe observes -- half of them at C5 -- are not read
#pragma unroll
    for (int u = 0; u < 2; ++u)
      if (q0 + u < n_mp && o[u] != OWNER_NONE && !(fl[u] & 1u) && q0 + u >= mp_lo && q0 + u < mp_hi)
        pf[u] = *reinterpret_cast<const float4*>(rec + q0 + u);
    bool go[2];
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const int q = q0 + u;
      go[u] = false;
      if (q >= n_mp) continue;
      if (o[u] == OWNER_NONE || (fl[u] & 1u)) {   // unobserved by the window, or bad
        corr_ref[q] = -1;
        continue;
      }
      corr_ref[q] = window[o[u]];   // (every point: the owner bookkeeping stays replicated)
      go[u] = q >= mp_lo && q < mp_hi;   // (else another rank's point slice, lc_set_point_range)
    }
    double T[13], Si[13];
    if (go[0] || go[1]) {
      const double* S = scr + (size_t)WSTR * (go[0] ? o[0] : o[1]);
      load13(S, T);
      load13(S + 14, Si);
    }
    double pw[2][3];
    if (go[0] && go[1] && o[0] == o[1]) {   // one owner (the common case): two chains interleaved
      double p0[3] = {pf[0].x, pf[0].y, pf[0].z}, p1[3] = {pf[1].x, pf[1].y, pf[1].z}, c0[3], c1[3];
      lc_sim3_apply(T, p0, c0);
      lc_sim3_apply(T, p1, c1);
      lc_sim3_apply(Si, c0, pw[0]);
      lc_sim3_apply(Si, c1, pw[1]);
    } else {
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        if (!go[u]) continue;
        if (u == 1 && go[0] && o[1] != o[0]) {
          const double* S = scr + (size_t)WSTR * o[1];
          load13(S, T);
          load13(S + 14, Si);
        }
        double p[3] = {pf[u].x, pf[u].y, pf[u].z}, pc[3];
        lc_sim3_apply(T, p, pc);
        lc_sim3_apply(Si, pc, pw[u]);
      }
    }
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      if (!go[u]) continue;
      rec[q0 + u].pos[0] = __double2float_rn(pw[u][0]);
      rec[q0 + u].pos[1] = __double2float_rn(pw[u][1]);
      rec[q0 + u].pos[2] = __double2float_rn(pw[u][2]);
      ++n;
    }
    warp_count(n, &counts[LC_COUNT_CORR_MP]);
  } else {
    pdl_wait();
    const int i = (blockIdx.x - nb_mp) * blockDim.x + threadIdx.x;
    if (i < n_w) {
      const double* T = scr + (size_t)WSTR * i + 42;
      for (int j = 0; j < 13; ++j) kf_pose[13 * (size_t)window[i] + j] = T[j];
      n = 1;
    }
    warp_count(n, &counts[LC_COUNT_CORR_KF]);
  }
}

// ALL: per keyframe S^pre and inverse(S^opt) into scratch, pose <- SE3(S^opt)
__global__ void k_all_kf(int n_kf, const double* __restrict__ Sopt, double* __restrict__ kf_pose,
                         const double* __restrict__ kf_S_corr, int32_t* __restrict__ kf_in_win,
                         double* __restrict__ scr, unsigned long long* __restrict__ counts) {
  pdl_trigger();   // k_all_points' prologue reads none of this kernel's outputs
  if (blockIdx.x == 0 && threadIdx.x < LC_NCOUNT)   // the call's counters (k_all_points adds later)
    counts[threadIdx.x] = threadIdx.x == LC_COUNT_CORR_KF ? (unsigned long long)n_kf : 0ull;
  int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k < n_kf) {
    double pre[13], opt[13], inv[13], T[13];
    const double* src = kf_in_win[k] ? kf_S_corr + 13 * (size_t)k : kf_pose + 13 * (size_t)k;
    for (int j = 0; j < 13; ++j) pre[j] = src[j];
    for (int j = 0; j < 13; ++j) opt[j] = Sopt[13 * (size_t)k + j];
    lc_sim3_inverse(opt, inv);
    lc_sim3_se3(opt, T);
    double* o = scr + (size_t)ASTR * k;
    for (int j = 0; j < 13; ++j) { o[j] = pre[j]; o[14 + j] = inv[j]; }
    o[13] = o[27] = 0.0;
    for (int j = 0; j < 13; ++j) kf_pose[13 * (size_t)k + j] = T[j];
    kf_in_win[k] = 0;
  }
}

// Two adjacent points per thread (they share their reference keyframe in creation
// order, so the two 13-double transforms are loaded once): every per-point load is
// issued before the PDL wait, the transform gather after it.
__global__ void __launch_bounds__(LC_NTHREADS, LC_PT_MINB) k_all_points(
    int n_mp, int mp_lo, int mp_hi, const double* scr, const int32_t* __restrict__ ref_kf,
    const uint8_t* flags, MpRec* __restrict__ rec, int32_t* __restrict__ corr_ref,
    unsigned long long* __restrict__ counts) {
  uint32_t n = 0;
  const int q0 = 2 * (blockIdx.x * blockDim.x + threadIdx.x);
  int cr[2] = {-1, -1}, rk[2] = {0, 0};
  uint8_t fl[2] = {1, 1};
  float4 pf[2];
#pragma unroll
  for (int u = 0; u < 2; ++u) {
    pf[u] = make_float4(0.f, 0.f, 0.f, 0.f);
    if (q0 + u < n_mp) {
      cr[u] = corr_ref[q0 + u];
      rk[u] = ref_kf[q0 + u];
      fl[u] = flags[q0 + u];
    }
  }
  // the records of the points this pass moves only (not bad -- the fused duplicates are --
  // and this rank's slice); the flags are final (the fuse that set them has completed)
#pragma unroll
  for (int u = 0; u < 2; ++u)
    if (q0 + u < n_mp && !(fl[u] & 1u) && q0 + u >= mp_lo && q0 + u < mp_hi)
      pf[u] = *reinterpret_cast<const float4*>(rec + q0 + u);
  pdl_wait();
  bool go[2];
  int r[2];
#pragma unroll
  for (int u = 0; u < 2; ++u) {
    const int q = q0 + u;
    go[u] = q < n_mp && !(fl[u] & 1u) && q >= mp_lo && q < mp_hi;   // not bad, this rank's slice
    r[u] = cr[u] >= 0 ? cr[u] : rk[u];
    if (q < n_mp && cr[u] >= 0) corr_ref[q] = -1;
  }
  double pre[13], inv[13];
  if (go[0] || go[1]) {
    const double* S = scr + (size_t)ASTR * (go[0] ? r[0] : r[1]);
    load13(S, pre);
    load13(S + 14, inv);
  }
  double pw[2][3];
  if (go[0] && go[1] && r[0] == r[1]) {   // the common case (creation order): both points with
    double p0[3] = {pf[0].x, pf[0].y, pf[0].z}, p1[3] = {pf[1].x, pf[1].y, pf[1].z}, c0[3], c1[3];
    lc_sim3_apply(pre, p0, c0);             // one transform pair, the two fp64 chains interleaved
    lc_sim3_apply(pre, p1, c1);
    lc_sim3_apply(inv, c0, pw[0]);
    lc_sim3_apply(inv, c1, pw[1]);
  } else {
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      if (!go[u]) continue;
      if (u == 1 && go[0] && r[1] != r[0]) {
        const double* S = scr + (size_t)ASTR * r[1];
        load13(S, pre);
        load13(S + 14, inv);
      }
      double p[3] = {pf[u].x, pf[u].y, pf[u].z}, pc[3];
      lc_sim3_apply(pre, p, pc);
      lc_sim3_apply(inv, pc, pw[u]);
    }
  }
#pragma unroll
  for (int u = 0; u < 2; ++u) {
    if (!go[u]) continue;
    rec[q0 + u].pos[0] = __double2float_rn(pw[u][0]);
    rec[q0 + u].pos[1] = __double2float_rn(pw[u][1]);
    rec[q0 + u].pos[2] = __double2float_rn(pw[u][2]);
    ++n;
  }
  warp_count(n, &counts[LC_COUNT_CORR_MP]);
}

// ---------------------------------------------------------------------------
// WINDOW | DRY_RUN over a batch of hypotheses (oracle O3'): the
// same S^corr / owner / re-anchoring arithmetic as the WINDOW kernels above, per batch
// b (its window = slots [wbeg[b], wbeg[b+1]) of the concatenated window list), with
// nothing written back: S^corr rows and the corrected positions of the owned points
// (ascending map-point index, CSR by batch) go to the caller's buffers.
// ---------------------------------------------------------------------------
__device__ __forceinline__ int batch_of(const int32_t* __restrict__ wbeg, int n_batch, int j) {
  int lo = 0, hi = n_batch - 1;   // last b with wbeg[b] <= j
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (wbeg[mid] <= j) lo = mid; else hi = mid - 1;
  }
  return lo;
}

// thread per window slot j: S_j^corr = (T_jw * inverse(T_cw)) * S_cw^corr[b] (cur first)
__global__ void k_dry_sim3(int n_slots, int n_batch, const int32_t* __restrict__ wbeg,
                           const int32_t* __restrict__ window, const double* __restrict__ kf_pose,
                           const double* __restrict__ Scw, double* __restrict__ scr, double* __restrict__ out_S,
                           unsigned long long* __restrict__ counts) {
  if (blockIdx.x == 0 && threadIdx.x < LC_NCOUNT)   // the call's counters
    counts[threadIdx.x] = threadIdx.x == LC_COUNT_CORR_KF ? (unsigned long long)n_slots : 0ull;
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= n_slots) return;
  const int b = batch_of(wbeg, n_batch, j);
  const int k = window[j];
  double T[13], S[13], Si[13];
  for (int i = 0; i < 13; ++i) T[i] = kf_pose[13 * (size_t)k + i];
  if (j == wbeg[b]) {
    for (int i = 0; i < 13; ++i) S[i] = Scw[13 * (size_t)b + i];
  } else {
    double Tc[13], Tci[13], Sic[13];
    const int c = window[wbeg[b]];
    for (int i = 0; i < 13; ++i) Tc[i] = kf_pose[13 * (size_t)c + i];
    lc_sim3_inverse(Tc, Tci);
    lc_sim3_compose(T, Tci, Sic);
    lc_sim3_compose(Sic, Scw + 13 * (size_t)b, S);
  }
  lc_sim3_inverse(S, Si);
  double* o = scr + (size_t)WSTR * j;
  for (int i = 0; i < 13; ++i) { o[i] = T[i]; o[14 + i] = Si[i]; o[28 + i] = S[i]; }
  o[13] = o[27] = o[41] = 0.0;
  if (out_S)
    for (int i = 0; i < 13; ++i) out_S[13 * (size_t)j + i] = S[i];
}

// warp per window slot j: owner[b][m] = min local position observing m
__global__ void __launch_bounds__(LC_NTHREADS) k_dry_mark(
    int n_slots, int n_batch, int n_mp, const int32_t* __restrict__ wbeg, const int32_t* __restrict__ window,
    const int32_t* __restrict__ kf_fbeg, const int32_t* __restrict__ feat_mp, int32_t* owner) {
  const int lane = threadIdx.x & 31;
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  for (int j = gw; j < n_slots; j += nw) {
    const int b = batch_of(wbeg, n_batch, j);
    const int i = j - wbeg[b];
    int32_t* ob = owner + (size_t)b * n_mp;
    const int k = window[j];
    for (int f = kf_fbeg[k] + lane; f < kf_fbeg[k + 1]; f += 32) {
      const int m = feat_mp[f];
      if (m >= 0) atomicMin(&ob[m], i);
    }
  }
}

// (b, q) grid, one point per thread: per-block count of owned non-bad points
__global__ void __launch_bounds__(LC_NTHREADS) k_dry_count(int n_mp, int nblk, const int32_t* __restrict__ owner,
                                                           const uint8_t* __restrict__ flags, int32_t* __restrict__ bcnt) {
  const int b = blockIdx.y;
  const int q = blockIdx.x * blockDim.x + threadIdx.x;
  const bool own = q < n_mp && owner[(size_t)b * n_mp + q] != OWNER_NONE && !(flags[q] & 1u);
  const int n = __syncthreads_count(own);
  if (threadIdx.x == 0) bcnt[(size_t)b * nblk + blockIdx.x] = n;
}

// one CTA: exclusive scan of the block counts (batch-major) -> block offsets, CSR begin
__global__ void __launch_bounds__(1024) k_dry_scan(int n_batch, int nblk, int32_t* __restrict__ bcnt,
                                                   int32_t* __restrict__ mp_begin) {
  __shared__ int32_t s_w[32];
  __shared__ int32_t s_carry;
  const int n = n_batch * nblk;
  if (threadIdx.x == 0) s_carry = 0;
  __syncthreads();
  for (int base = 0; base < n; base += blockDim.x) {
    const int i = base + threadIdx.x;
    const int v = i < n ? bcnt[i] : 0;
    int x = v;
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, x, o);
      if ((threadIdx.x & 31) >= o) x += y;
    }
    if ((threadIdx.x & 31) == 31) s_w[threadIdx.x >> 5] = x;
    __syncthreads();
    if (threadIdx.x < 32) {
      int w = threadIdx.x < (int)(blockDim.x >> 5) ? s_w[threadIdx.x] : 0;
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, w, o);
        if (threadIdx.x >= o) w += y;
      }
      s_w[threadIdx.x] = w;
    }
    __syncthreads();
    const int excl = s_carry + (threadIdx.x >= 32 ? s_w[(threadIdx.x >> 5) - 1] : 0) + x - v;
    if (i < n) {
      bcnt[i] = excl;
      if (i % nblk == 0) mp_begin[i / nblk] = excl;
    }
    __syncthreads();
    if (threadIdx.x == blockDim.x - 1) s_carry = excl + v;
    __syncthreads();
  }
  if (threadIdx.x == 0) mp_begin[n_batch] = s_carry;
}

// (b, q) grid: owned point -> (idx, fl32(inverse(S_o^corr)(T_ow^old(p)))) at its CSR slot
__global__ void __launch_bounds__(LC_NTHREADS) k_dry_points(
    int n_mp, int nblk, long long capacity, const int32_t* __restrict__ wbeg, const int32_t* __restrict__ owner,
    const uint8_t* __restrict__ flags, const int32_t* __restrict__ boff, const double* __restrict__ scr,
    const MpRec* __restrict__ rec, int32_t* __restrict__ out_idx, float* __restrict__ out_pos,
    unsigned long long* __restrict__ counts) {
  __shared__ int32_t s_w[LC_NTHREADS / 32];
  const int b = blockIdx.y;
  const int q = blockIdx.x * blockDim.x + threadIdx.x;
  const int o = q < n_mp ? owner[(size_t)b * n_mp + q] : OWNER_NONE;
  const bool own = o != OWNER_NONE && !(flags[q] & 1u);
  const unsigned m = __ballot_sync(0xffffffffu, own);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (lane == 0) s_w[warp] = __popc(m);
  __syncthreads();
  int before = 0;
  for (int w = 0; w < warp; ++w) before += s_w[w];
  if (own) {
    const long long slot = (long long)boff[(size_t)b * nblk + blockIdx.x] + before + __popc(m & ((1u << lane) - 1u));
    if (slot < capacity) {
      const double* S = scr + (size_t)WSTR * (wbeg[b] + o);
      double T[13], Si[13];
      load13(S, T);
      load13(S + 14, Si);
      double p[3] = {rec[q].pos[0], rec[q].pos[1], rec[q].pos[2]}, pc[3], pw[3];
      lc_sim3_apply(T, p, pc);
      lc_sim3_apply(Si, pc, pw);
      out_idx[slot] = q;
      out_pos[3 * slot + 0] = __double2float_rn(pw[0]);
      out_pos[3 * slot + 1] = __double2float_rn(pw[1]);
      out_pos[3 * slot + 2] = __double2float_rn(pw[2]);
    }
  }
  warp_count(own ? 1u : 0u, &counts[LC_COUNT_CORR_MP]);
}

}  // namespace

int correct_window_scratch_stride() { return WSTR; }
int correct_all_scratch_stride() { return ASTR; }

cudaError_t launch_correct_window(lc_ctx* c, int cur_pos, int n_w, const int32_t* d_window,
                                  const double* d_Scw, double* d_scr, double* d_outS,
                                  unsigned long long* counts, cudaStream_t s) {
  Store& st = c->st;
  cudaError_t e;
  if (st.n_mp > 0 && (e = cudaMemsetAsync(st.mp_owner, 0x7F, sizeof(int32_t) * st.n_mp, s)) != cudaSuccess)
    return e;
  if ((e = cudaMemsetAsync(st.kf_in_win, 0, sizeof(int32_t) * st.n_kf, s)) != cudaSuccess) return e;
  k_win_sim3<<<(n_w + 63) / 64, 64, 0, s>>>(n_w, cur_pos, d_window, st.kf_pose, d_Scw, d_scr,
                                            st.kf_S_corr, st.kf_in_win, d_outS, counts);
  if ((e = launch_pdl(k_win_mark, dim3(std::min((n_w + 7) / 8, 148 * 8)), dim3(LC_NTHREADS), 0, s, n_w,
                      d_window, st.kf_fbeg, st.feat_mp, st.mp_owner)) != cudaSuccess)
    return e;
  const int nb_mp = st.n_mp > 0 ? (st.n_mp + 2 * LC_NTHREADS - 1) / (2 * LC_NTHREADS) : 0;
  const int nb_w = (n_w + LC_NTHREADS - 1) / LC_NTHREADS;
  if ((e = launch_pdl(k_win_b, dim3(nb_mp + nb_w), dim3(LC_NTHREADS), 0, s, st.n_mp, nb_mp, n_w,
                      c->mp_lo, c->mp_hi < 0 ? st.n_mp : c->mp_hi, st.mp_owner, st.mp_flags, d_window, d_scr, st.mp_rec, st.mp_corr_ref, st.kf_pose,
                      counts)) != cudaSuccess)
    return e;
  c->launches += 3;
  return cudaGetLastError();
}

cudaError_t launch_correct_all(lc_ctx* c, const double* d_Sopt, double* d_scr,
                               unsigned long long* counts, cudaStream_t s) {
  Store& st = c->st;
  k_all_kf<<<std::max(1, (st.n_kf + 127) / 128), 128, 0, s>>>(st.n_kf, d_Sopt, st.kf_pose, st.kf_S_corr,
                                                st.kf_in_win, d_scr, counts);
  c->launches++;
  if (st.n_mp > 0) {
    cudaError_t e = launch_pdl(k_all_points, dim3((st.n_mp + 2 * LC_NTHREADS - 1) / (2 * LC_NTHREADS)),
                               dim3(LC_NTHREADS), 0, s, st.n_mp, c->mp_lo,
                               c->mp_hi < 0 ? st.n_mp : c->mp_hi, (const double*)d_scr,
                               (const int32_t*)st.mp_ref_kf, (const uint8_t*)st.mp_flags, st.mp_rec,
                               st.mp_corr_ref, counts);
    if (e != cudaSuccess) return e;
    c->launches++;
  }
  return cudaGetLastError();
}

namespace {
// lc_mp_positions: fp32 positions of map points [lo, hi) out of / into the records
__global__ void k_pos_get(int lo, int hi, const MpRec* __restrict__ rec, float* __restrict__ xyz) {
  for (int q = lo + blockIdx.x * blockDim.x + threadIdx.x; q < hi; q += gridDim.x * blockDim.x) {
    const float4 p = *reinterpret_cast<const float4*>(rec + q);
    float* o = xyz + 3 * (size_t)(q - lo);
    o[0] = p.x; o[1] = p.y; o[2] = p.z;
  }
}
__global__ void k_pos_set(int lo, int hi, const float* __restrict__ xyz, MpRec* __restrict__ rec) {
  for (int q = lo + blockIdx.x * blockDim.x + threadIdx.x; q < hi; q += gridDim.x * blockDim.x) {
    const float* i = xyz + 3 * (size_t)(q - lo);
    rec[q].pos[0] = i[0]; rec[q].pos[1] = i[1]; rec[q].pos[2] = i[2];
  }
}

}  // namespace

cudaError_t launch_mp_positions(lc_ctx* c, int op, int lo, int hi, float* xyz, cudaStream_t s) {
  if (hi <= lo) return cudaSuccess;
  const int g = std::min((hi - lo + LC_NTHREADS - 1) / LC_NTHREADS, 148 * 8);
  if (op == LC_POS_GET) k_pos_get<<<g, LC_NTHREADS, 0, s>>>(lo, hi, c->st.mp_rec, xyz);
  else k_pos_set<<<g, LC_NTHREADS, 0, s>>>(lo, hi, xyz, c->st.mp_rec);
  c->launches++;
  return cudaGetLastError();
}

size_t correct_dry_scratch_bytes(int n_batch, int n_slots, int n_mp) {
  const int nblk = std::max(1, (n_mp + LC_NTHREADS - 1) / LC_NTHREADS);
  return sizeof(double) * WSTR * (size_t)std::max(n_slots, 1) + sizeof(int32_t) * (size_t)n_batch * std::max(n_mp, 1) +
         sizeof(int32_t) * ((size_t)n_batch * nblk + 64);
}

cudaError_t launch_correct_dry(lc_ctx* c, int n_batch, int n_slots, const int32_t* d_wbeg, const int32_t* d_window,
                               const double* d_Scw, void* scratch, double* d_outS, int32_t* d_mp_begin,
                               int64_t capacity, int32_t* d_idx, float* d_pos, unsigned long long* counts,
                               cudaStream_t s) {
  Store& st = c->st;
  const int n_mp = st.n_mp;
  const int nblk = std::max(1, (n_mp + LC_NTHREADS - 1) / LC_NTHREADS);
  double* scr = (double*)scratch;
  int32_t* owner = (int32_t*)(scr + (size_t)WSTR * std::max(n_slots, 1));
  int32_t* bcnt = owner + (size_t)n_batch * std::max(n_mp, 1);
  cudaError_t e;
  if (n_mp > 0 && (e = cudaMemsetAsync(owner, 0x7F, sizeof(int32_t) * (size_t)n_batch * n_mp, s)) != cudaSuccess)
    return e;
  k_dry_sim3<<<(n_slots + 63) / 64, 64, 0, s>>>(n_slots, n_batch, d_wbeg, d_window, st.kf_pose, d_Scw, scr, d_outS,
                                              counts);
  k_dry_mark<<<std::min((n_slots + 7) / 8, 148 * 8), LC_NTHREADS, 0, s>>>(n_slots, n_batch, n_mp, d_wbeg, d_window,
                                                                       st.kf_fbeg, st.feat_mp, owner);
  const dim3 g2(nblk, n_batch);
  k_dry_count<<<g2, LC_NTHREADS, 0, s>>>(n_mp, nblk, owner, st.mp_flags, bcnt);
  k_dry_scan<<<1, 1024, 0, s>>>(n_batch, nblk, bcnt, d_mp_begin);
  k_dry_points<<<g2, LC_NTHREADS, 0, s>>>(n_mp, nblk, (long long)capacity, d_wbeg, owner, st.mp_flags, bcnt, scr,
                                         st.mp_rec, d_idx, d_pos, counts);
  c->launches += 5;
  return cudaGetLastError();
}
