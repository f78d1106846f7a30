// k_lists.cu -- loop map-point lists built on the device from the resident map (oracle
// orc_loop_lists; "Loop list = MPs of the matched pass-A KF and its
// top-10 covisibles, ascending unique", C5: "each has its own list: MPs of its 10 nearest
// pass-A KFs"; EXT LoopClosing mvpLoopMapPoints). The paper builds them on the CPU; here
// they never leave the GPU, so a loop event uploads keyframe ids instead of map-point
// lists (C5: 110 KB instead of 35 MB).
//
// Main path: two kernels around one host synchronisation (the caller needs the offsets):
//   k_lists_bitmap CTA per list: the [min, max] range of its source keyframes' map points
//                  (one pass), then one bit per map point id of that range in shared
//                  memory (a second pass, atomicOr) -- written to a per-list global bitmap
//                  with the distinct count; map point ids of neighbouring keyframes span a
//                  few thousand ids, so no hashing and no sort is needed;
//   k_lists_emit   CTA per list: the bitmap read back, a block scan of per-word popcounts,
//                  and the set bits written in order: the ascending unique list.
// Lists whose id range exceeds the bitmap capacity take the general path:
//   k_lists_dedup  CTA per list: the associations of its source keyframes go into a
//                  shared-memory hash set (open addressing, LIST_HCAP slots); the distinct
//                  map points are compacted (block scan, deterministic positions) into a
//                  per-list region of a scratch buffer, their count into counts[l];
//   k_lists_sort   CTA per list: the region is loaded into shared memory, bitonic-sorted
//                  and written ascending at out_begin[l].
#include <cuda_runtime.h>

#include <algorithm>

#include "lc_internal.cuh"

namespace {

constexpr int LIST_NT = 256;

__device__ __forceinline__ uint32_t lhash(int32_t key) { return (uint32_t)key * 2654435769u; }

// the hash set holds up to 3/4 of its slots; HCAP 8192 first, the lists that overflow it
// again with HCAP 32768 (their count then is exact up to LIST_MAX_UNIQUE)
template <int HCAP>
__global__ void __launch_bounds__(LIST_NT) k_lists_dedup(int n, const int32_t* __restrict__ sel,
                                                         const int32_t* __restrict__ sbeg,
                                                         const int32_t* __restrict__ skf,
                                                         const int32_t* __restrict__ kf_fbeg,
                                                         const int32_t* __restrict__ feat_mp,
                                                         const int64_t* __restrict__ reg_off,
                                                         int32_t* __restrict__ reg, int32_t* __restrict__ counts) {
  constexpr int LIST_HCAP = HCAP, LIST_UMAX = HCAP / 4 * 3;
  extern __shared__ int32_t s_h[];   // [HCAP]
  __shared__ int32_t s_n;
  __shared__ int32_t s_part[LIST_NT];
  for (int li = blockIdx.x; li < n; li += gridDim.x) {
    const int l = sel ? sel[li] : li;
    for (int i = threadIdx.x; i < LIST_HCAP; i += LIST_NT) s_h[i] = -1;
    if (threadIdx.x == 0) s_n = 0;
    __syncthreads();
    for (int j = sbeg[l]; j < sbeg[l + 1]; ++j) {
      const int k = skf[j];
      for (int f = kf_fbeg[k] + threadIdx.x; f < kf_fbeg[k + 1]; f += LIST_NT) {
        const int32_t m = feat_mp[f];
        if (m < 0) continue;
        uint32_t h = lhash(m) >> (32 - __ffs(LIST_HCAP) + 1);
        for (int probe = 0; probe < LIST_HCAP; ++probe) {
          const int32_t prev = atomicCAS(&s_h[h], -1, m);
          if (prev == -1) { atomicAdd(&s_n, 1); break; }
          if (prev == m) break;
          h = (h + 1) & (LIST_HCAP - 1);
        }
      }
    }
    __syncthreads();
    const int u = s_n;
    if (threadIdx.x == 0) counts[l] = u > LIST_UMAX ? -1 : u;   // -1: overflow, retry larger
    if (u <= LIST_UMAX) {   // compact: thread t owns slots [t * S, (t + 1) * S), block scan
      constexpr int S = LIST_HCAP / LIST_NT;
      int c = 0;
      for (int i = 0; i < S; ++i) c += s_h[threadIdx.x * S + i] >= 0;
      s_part[threadIdx.x] = c;
      __syncthreads();
      if (threadIdx.x == 0) {
        int acc = 0;
        for (int t = 0; t < LIST_NT; ++t) { const int x = s_part[t]; s_part[t] = acc; acc += x; }
      }
      __syncthreads();
      int32_t* out = reg + reg_off[l];
      int o = s_part[threadIdx.x];
      for (int i = 0; i < S; ++i) {
        const int32_t m = s_h[threadIdx.x * S + i];
        if (m >= 0) out[o++] = m;
      }
    }
    __syncthreads();
  }
}

__global__ void __launch_bounds__(LIST_NT) k_lists_sort(int n, const int64_t* __restrict__ reg_off,
                                                        const int32_t* __restrict__ reg,
                                                        const int32_t* __restrict__ out_begin,
                                                        int32_t* __restrict__ out) {
  extern __shared__ int32_t s[];   // [next power of two of the longest list]
  for (int l = blockIdx.x; l < n; l += gridDim.x) {
    const int u = out_begin[l + 1] - out_begin[l];
    int p2 = 1;
    while (p2 < u) p2 <<= 1;
    for (int i = threadIdx.x; i < p2; i += LIST_NT) s[i] = i < u ? reg[reg_off[l] + i] : 0x7FFFFFFF;
    __syncthreads();
    for (int size = 2; size <= p2; size <<= 1)
      for (int stride = size >> 1; stride > 0; stride >>= 1) {
        for (int i = threadIdx.x; i < p2 / 2; i += LIST_NT) {   // compare-exchange pairs
          const int lo = 2 * i - (i & (stride - 1));
          const int hi = lo + stride;
          const bool up = ((lo & size) == 0);
          const int32_t a = s[lo], b = s[hi];
          if ((a > b) == up) { s[lo] = b; s[hi] = a; }
        }
        __syncthreads();
      }
    for (int i = threadIdx.x; i < u; i += LIST_NT) out[out_begin[l] + i] = s[i];
    __syncthreads();
  }
}

// per-thread batches of 8 association loads in flight (the loop is load-latency bound)
template <typename F>
__device__ __forceinline__ void for_assoc(int l, const int32_t* __restrict__ sbeg, const int32_t* __restrict__ skf,
                                          const int32_t* __restrict__ kf_fbeg, const int32_t* __restrict__ feat_mp,
                                          F&& fn) {
  for (int j = sbeg[l]; j < sbeg[l + 1]; ++j) {
    const int k = skf[j];
    const int fb = kf_fbeg[k], fe = kf_fbeg[k + 1];
    for (int f0 = fb + threadIdx.x; f0 < fe; f0 += 8 * LIST_NT) {
      int32_t m[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) m[u] = f0 + u * LIST_NT < fe ? __ldg(feat_mp + f0 + u * LIST_NT) : -1;
#pragma unroll
      for (int u = 0; u < 8; ++u)
        if (m[u] >= 0) fn(m[u]);
    }
  }
}

// per source keyframe: [min, max] of its associated map point ids (-1/-1 if none) -- the
// lists' id ranges without a pass over their associations
__global__ void __launch_bounds__(LIST_NT) k_kf_idrange(int n_src, const int32_t* __restrict__ skf,
                                                        const int32_t* __restrict__ kf_fbeg,
                                                        const int32_t* __restrict__ feat_mp,
                                                        int2* __restrict__ rng) {
  const int lane = threadIdx.x & 31;
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = (gridDim.x * blockDim.x) >> 5;
  for (int j = gw; j < n_src; j += nw) {
    const int k = skf[j];
    int lo = 0x7FFFFFFF, hi = -1;
    for (int f0 = kf_fbeg[k] + lane; f0 < kf_fbeg[k + 1]; f0 += 8 * 32) {
      int32_t m[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) m[u] = f0 + 32 * u < kf_fbeg[k + 1] ? __ldg(feat_mp + f0 + 32 * u) : -1;
#pragma unroll
      for (int u = 0; u < 8; ++u)
        if (m[u] >= 0) { lo = min(lo, m[u]); hi = max(hi, m[u]); }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      lo = min(lo, __shfl_xor_sync(0xffffffffu, lo, o));
      hi = max(hi, __shfl_xor_sync(0xffffffffu, hi, o));
    }
    if (lane == 0) rng[j] = make_int2(lo, hi);
  }
}

// lists sel[i] (or i) -> bitmap region i * maxw of bm; lo_out[l] / lo_out[n_lists + l] =
// the list's first id / its bitmap words, counts[l] = distinct ids (-1: range too wide)
// only_wide: lists whose count is still -1 (too wide for the first pass) only, counted in
// shared memory without a global bitmap (lo_out words stored negated: "rebuild at emit")
__global__ void __launch_bounds__(LIST_NT) k_lists_bitmap(int n, int n_lists, const int32_t* __restrict__ sel, int maxw,
                                                          int only_wide,
                                                          const int2* __restrict__ src_rng,
                                                          const int32_t* __restrict__ sbeg,
                                                          const int32_t* __restrict__ skf,
                                                          const int32_t* __restrict__ kf_fbeg,
                                                          const int32_t* __restrict__ feat_mp,
                                                          uint32_t* __restrict__ bm, int32_t* __restrict__ lo_out,
                                                          int32_t* __restrict__ counts) {
  extern __shared__ uint32_t s_bm[];   // [maxw]
  __shared__ int s_lo, s_hi, s_cnt;
  for (int li = blockIdx.x; li < n; li += gridDim.x) {
    const int l = sel ? sel[li] : li;
    if (only_wide && counts[l] >= 0) continue;   // (uniform over the CTA; written below after syncs)
    if (threadIdx.x == 0) {   // the list's id range from its sources' ranges
      int lo0 = 0x7FFFFFFF, hi0 = -1;
      for (int j = sbeg[l]; j < sbeg[l + 1]; ++j) {
        const int2 r = src_rng[j];
        if (r.y >= 0) { lo0 = min(lo0, r.x); hi0 = max(hi0, r.y); }
      }
      s_lo = lo0; s_hi = hi0; s_cnt = 0;
    }
    __syncthreads();
    const int lo = s_lo, hi = s_hi;
    const int words = hi >= lo ? ((hi - lo) >> 5) + 1 : 0;
    if (words > maxw) {   // id range too wide for this bitmap: a larger one (or the general path)
      if (threadIdx.x == 0) { counts[l] = -1; lo_out[n_lists + l] = -1; }
      __syncthreads();
      continue;
    }
    for (int i = threadIdx.x; i < words; i += LIST_NT) s_bm[i] = 0u;
    __syncthreads();
    for_assoc(l, sbeg, skf, kf_fbeg, feat_mp, [&](int32_t m) {
      const int b = m - lo;
      atomicOr(&s_bm[b >> 5], 1u << (b & 31));
    });
    __syncthreads();
    uint32_t* g = only_wide ? nullptr : bm + (size_t)li * maxw;
    int c = 0;
    for (int i = threadIdx.x; i < words; i += LIST_NT) {
      const uint32_t x = s_bm[i];
      if (g) g[i] = x;
      c += __popc(x);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
    if ((threadIdx.x & 31) == 0 && c) atomicAdd(&s_cnt, c);
    __syncthreads();
    if (threadIdx.x == 0) {
      counts[l] = s_cnt;
      lo_out[l] = words ? lo : 0;
      lo_out[n_lists + l] = only_wide ? -words : words;
    }
    __syncthreads();
  }
}

constexpr int EMIT_STAGE = 8192;   // ids staged in shared memory for coalesced stores
__global__ void __launch_bounds__(LIST_NT) k_lists_emit(int n, const uint32_t* __restrict__ bm,
                                                        const int64_t* __restrict__ bm_off,
                                                        const int32_t* __restrict__ lo_in,
                                                        const int32_t* __restrict__ counts,
                                                        const int32_t* __restrict__ out_begin,
                                                        int32_t* __restrict__ out) {
  __shared__ int32_t s_ids[EMIT_STAGE];
  __shared__ int s_w[LIST_NT / 32 + 1];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int l = blockIdx.x; l < n; l += gridDim.x) {
    if (counts[l] < 0 || lo_in[n + l] < 0) continue;   // (uniform; hashed / rebuilt at emit)
    const int words = lo_in[n + l], lo = lo_in[l];
    const int cnt = counts[l];
    const uint32_t* g = bm + bm_off[l];
    int32_t* dst = out + out_begin[l];
    int base = 0;   // ids emitted before this chunk of LIST_NT words
    for (int w0 = 0; w0 < words; w0 += LIST_NT) {
      const int i = w0 + threadIdx.x;
      uint32_t x = i < words ? g[i] : 0u;
      const int c = __popc(x);
      int incl = c;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
      }
      if (lane == 31) s_w[warp] = incl;
      __syncthreads();
      if (threadIdx.x == 0) {
        int acc = 0;
        for (int t = 0; t < LIST_NT / 32; ++t) { const int v = s_w[t]; s_w[t] = acc; acc += v; }
        s_w[LIST_NT / 32] = acc;
      }
      __syncthreads();
      int r = base + s_w[warp] + incl - c;
      const bool stage = cnt <= EMIT_STAGE;
      const int idb = lo + 32 * i;
      while (x) {
        const int b = __ffs(x) - 1;
        if (stage) s_ids[r] = idb + b;
        else dst[r] = idb + b;
        ++r;
        x &= x - 1;
      }
      base += s_w[LIST_NT / 32];
      __syncthreads();
    }
    if (cnt <= EMIT_STAGE) {
      for (int j = threadIdx.x; j < cnt; j += LIST_NT) dst[j] = s_ids[j];
      __syncthreads();
    }
  }
}

// device-resident offsets (lc_loop_lists with a device out_begin): out_begin[0] = 0,
// out_begin[l + 1] = out_begin[l] + counts[l], one CTA
__global__ void __launch_bounds__(1024) k_lists_scan(int n, const int32_t* __restrict__ counts,
                                                     int32_t* __restrict__ out_begin) {
  __shared__ int s_w[33];
  __shared__ int s_carry;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) { s_carry = 0; out_begin[0] = 0; }
  __syncthreads();
  for (int b = 0; b < n; b += 1024) {
    const int i = b + threadIdx.x;
    const int c = i < n ? counts[i] : 0;
    int incl = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += y;
    }
    if (lane == 31) s_w[warp] = incl;
    __syncthreads();
    if (threadIdx.x == 0) {
      int acc = 0;
      for (int t = 0; t < 32; ++t) { const int v = s_w[t]; s_w[t] = acc; acc += v; }
      s_w[32] = acc;
    }
    __syncthreads();
    if (i < n) out_begin[i + 1] = s_carry + s_w[warp] + incl;
    __syncthreads();
    if (threadIdx.x == 0) s_carry += s_w[32];
    __syncthreads();
  }
}

// the lists counted by the only_wide pass (words stored negated): bitmap rebuilt in shared
// memory from their sources' associations and the ids written in order at out_begin[l]
__global__ void __launch_bounds__(LIST_NT) k_lists_emit_wide(int n, const int32_t* __restrict__ sbeg,
                                                             const int32_t* __restrict__ skf,
                                                             const int32_t* __restrict__ kf_fbeg,
                                                             const int32_t* __restrict__ feat_mp,
                                                             const int32_t* __restrict__ lo_in,
                                                             const int32_t* __restrict__ out_begin,
                                                             int32_t* __restrict__ out) {
  extern __shared__ uint32_t s_bm[];
  __shared__ int s_w[LIST_NT / 32 + 1];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int l = blockIdx.x; l < n; l += gridDim.x) {
    if (lo_in[n + l] >= 0) continue;   // (uniform) not rebuilt here
    const int words = -lo_in[n + l], lo = lo_in[l];
    for (int i = threadIdx.x; i < words; i += LIST_NT) s_bm[i] = 0u;
    __syncthreads();
    for_assoc(l, sbeg, skf, kf_fbeg, feat_mp, [&](int32_t m) {
      const int b = m - lo;
      atomicOr(&s_bm[b >> 5], 1u << (b & 31));
    });
    __syncthreads();
    int32_t* dst = out + out_begin[l];
    int base = 0;
    for (int w0 = 0; w0 < words; w0 += LIST_NT) {
      const int i = w0 + threadIdx.x;
      uint32_t x = i < words ? s_bm[i] : 0u;
      const int c = __popc(x);
      int incl = c;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
      }
      if (lane == 31) s_w[warp] = incl;
      __syncthreads();
      if (threadIdx.x == 0) {
        int acc = 0;
        for (int t = 0; t < LIST_NT / 32; ++t) { const int v = s_w[t]; s_w[t] = acc; acc += v; }
        s_w[LIST_NT / 32] = acc;
      }
      __syncthreads();
      int r = base + s_w[warp] + incl - c;
      while (x) {
        dst[r++] = lo + 32 * i + (__ffs(x) - 1);
        x &= x - 1;
      }
      base += s_w[LIST_NT / 32];
      __syncthreads();
    }
  }
}

}  // namespace

int lists_max_unique() { return 32768 / 4 * 3; }
int lists_small_unique() { return 8192 / 4 * 3; }

cudaError_t launch_lists_dedup(lc_ctx* c, bool large, int n, const int32_t* d_sel, const int32_t* d_sbeg,
                               const int32_t* d_skf, const int64_t* d_reg_off, int32_t* d_reg, int32_t* d_counts,
                               cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  cudaError_t e;
  if (!large) {
    if ((e = set_smem_attr((const void*)k_lists_dedup<8192>, 8192 * 4)) != cudaSuccess) return e;
    k_lists_dedup<8192><<<std::min(n, 148 * 5), LIST_NT, 8192 * 4, s>>>(n, d_sel, d_sbeg, d_skf, c->st.kf_fbeg,
                                                                        c->st.feat_mp, d_reg_off, d_reg, d_counts);
  } else {
    if ((e = set_smem_attr((const void*)k_lists_dedup<32768>, 32768 * 4)) != cudaSuccess) return e;
    k_lists_dedup<32768><<<std::min(n, 148), LIST_NT, 32768 * 4, s>>>(n, d_sel, d_sbeg, d_skf, c->st.kf_fbeg,
                                                                      c->st.feat_mp, d_reg_off, d_reg, d_counts);
  }
  c->launches++;
  return cudaGetLastError();
}

cudaError_t launch_lists_sort(lc_ctx* c, int n, int max_u, const int64_t* d_reg_off, const int32_t* d_reg,
                              const int32_t* d_out_begin, int32_t* d_out, cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  int p2 = 1;
  while (p2 < max_u) p2 <<= 1;
  const int smem = std::max(p2, 1) * 4;
  cudaError_t e = set_smem_attr((const void*)k_lists_sort, 32768 * 4);
  if (e != cudaSuccess) return e;
  k_lists_sort<<<std::min(n, 148 * 4), LIST_NT, smem, s>>>(n, d_reg_off, d_reg, d_out_begin, d_out);
  c->launches++;
  return cudaGetLastError();
}

int lists_bitmap_words() { return 8192; }             // first pass: id ranges up to 262,144
int lists_bitmap_words_max() { return 56 * 1024; }    // second pass: up to 1,835,008 (224 KB)

cudaError_t launch_kf_idrange(lc_ctx* c, int n_src, const int32_t* d_skf, int2* d_rng, cudaStream_t s) {
  if (n_src <= 0) return cudaSuccess;
  k_kf_idrange<<<std::min((n_src + 7) / 8, 148 * 16), LIST_NT, 0, s>>>(n_src, d_skf, c->st.kf_fbeg, c->st.feat_mp, d_rng);
  c->launches++;
  return cudaGetLastError();
}

cudaError_t launch_lists_bitmap(lc_ctx* c, int n, int n_lists, const int32_t* d_sel, int maxw, const int2* d_rng,
                                uint32_t* d_bm, int32_t* d_lo, int32_t* d_counts, const int32_t* d_sbeg,
                                const int32_t* d_skf, cudaStream_t s, bool only_wide) {
  if (n <= 0) return cudaSuccess;
  cudaError_t e = set_smem_attr((const void*)k_lists_bitmap, maxw * 4);
  if (e != cudaSuccess) return e;
  const int per_sm = std::max(1, 200 * 1024 / (maxw * 4 + 1024));
  k_lists_bitmap<<<std::min(n, 148 * per_sm), LIST_NT, maxw * 4, s>>>(n, n_lists, d_sel, maxw, only_wide ? 1 : 0,
                                                                     d_rng, d_sbeg, d_skf,
                                                                     c->st.kf_fbeg, c->st.feat_mp, d_bm,
                                                                     d_lo, d_counts);
  c->launches++;
  return cudaGetLastError();
}

cudaError_t launch_lists_emit(lc_ctx* c, int n, const uint32_t* d_bm, const int64_t* d_bm_off, const int32_t* d_lo,
                              const int32_t* d_counts, const int32_t* d_out_begin, int32_t* d_out, cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  k_lists_emit<<<std::min(n, 148 * 6), LIST_NT, 0, s>>>(n, d_bm, d_bm_off, d_lo, d_counts, d_out_begin, d_out);
  c->launches++;
  return cudaGetLastError();
}

cudaError_t launch_lists_scan(lc_ctx* c, int n, const int32_t* d_counts, int32_t* d_out_begin, cudaStream_t s) {
  k_lists_scan<<<1, 1024, 0, s>>>(n, d_counts, d_out_begin);
  c->launches++;
  return cudaGetLastError();
}

cudaError_t launch_lists_emit_wide(lc_ctx* c, int n, int maxw, const int32_t* d_sbeg, const int32_t* d_skf,
                                   const int32_t* d_lo, const int32_t* d_out_begin, int32_t* d_out, cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  cudaError_t e = set_smem_attr((const void*)k_lists_emit_wide, maxw * 4);
  if (e != cudaSuccess) return e;
  k_lists_emit_wide<<<std::min(n, 148), LIST_NT, maxw * 4, s>>>(n, d_sbeg, d_skf, c->st.kf_fbeg, c->st.feat_mp, d_lo,
                                                               d_out_begin, d_out);
  c->launches++;
  return cudaGetLastError();
}
