// k_covis.cu -- covisibility recount after the merge (PAPER.md:95
// "creates new connections in the covisibility and essential graphs", PAPER.md:228;
// SPEC.md update_connections; readings A38-A40; include/lc.h
// lc_update_connections). The paper keeps this step on the CPU ("irregular memory
// access patterns and strong data dependencies"); here it is one CTA
// per keyframe over the device observation lists (k_refresh.cu launch_obs_lists):
//   weight(k, k2) = number of distinct non-bad map points held by both (A38), counted
//   in a shared-memory array indexed by keyframe; edges >= th, or the single strongest
//   (A39), rank-sorted by (weight desc, id asc) (A40).
#include <cuda_runtime.h>

#include <algorithm>

#include "lc_internal.cuh"

namespace {

constexpr int EDGE_CAP = 2048;   // edges ranked per keyframe in shared memory

// feat_first[f] = 1 iff feature f is the smallest slot of its keyframe holding its map
// point (A38: a keyframe counts a point once). Thread per observation position.
__global__ void k_feat_first(int n_mp, const int32_t* __restrict__ feat_mp,
                             const int32_t* __restrict__ obeg, const int32_t* __restrict__ obs,
                             const int32_t* __restrict__ obs_kf, uint8_t* __restrict__ feat_first) {
  const int n_obs_total = obeg[n_mp];   // the lists' length (associations)
  for (int p = blockIdx.x * blockDim.x + threadIdx.x; p < n_obs_total; p += gridDim.x * blockDim.x) {
    const int f = obs[p], k = obs_kf[p];
    const int q = feat_mp[f];
    if ((unsigned)q >= (unsigned)n_mp) continue;
    const int b = obeg[q], e = obeg[q + 1];
    bool first = true;
    for (int i = b; i < e; ++i)
      if (obs_kf[i] == k && obs[i] < f) { first = false; break; }
    feat_first[f] = first ? 1 : 0;
  }
}

struct ConnArgs {
  int n_sel, n_kf, n_mp, th, max_edges;
  const int32_t* idx;
  const int32_t* kf_fbeg;
  const int32_t* feat_mp;
  const uint8_t* flags;
  const int32_t* obeg;
  const int32_t* obs;
  const int32_t* obs_kf;
  const uint8_t* feat_first;
  int32_t* out_n;
  int32_t* out_kf;
  int32_t* out_w;
  unsigned long long* counts;
};

__global__ void __launch_bounds__(LC_NTHREADS) k_connections(const ConnArgs a) {
  extern __shared__ __align__(16) int32_t s_w[];   // [n_kf] weights
  __shared__ unsigned long long s_e[EDGE_CAP];     // (~weight << 32) | k2 of the edges
  __shared__ int s_ne, s_best;
  uint32_t c_kf = 0, c_edges = 0;
  for (int t = blockIdx.x; t < a.n_sel; t += gridDim.x) {
    const int k = a.idx ? a.idx[t] : t;
    if ((unsigned)k >= (unsigned)a.n_kf) {
      if (threadIdx.x == 0 && a.out_n) a.out_n[t] = 0;
      continue;
    }
    for (int i = threadIdx.x; i < a.n_kf; i += blockDim.x) s_w[i] = 0;
    if (threadIdx.x == 0) { s_ne = 0; s_best = -1; }
    __syncthreads();
    const int fb = a.kf_fbeg[k], fe = a.kf_fbeg[k + 1];
    for (int f = fb + threadIdx.x; f < fe; f += blockDim.x) {
      const int q = a.feat_mp[f];
      if ((unsigned)q >= (unsigned)a.n_mp || (a.flags[q] & 1u)) continue;   // A38: not bad
      if (!a.feat_first[f]) continue;                   // distinct in k
      const int32_t* ob = a.obs + a.obeg[q];
      const int32_t* okf = a.obs_kf + a.obeg[q];
      const int no = a.obeg[q + 1] - a.obeg[q];
      for (int j = 0; j < no; ++j) {
        const int k2 = okf[j];
        if (k2 == k || !a.feat_first[ob[j]]) continue;   // once per k2
        atomicAdd(&s_w[k2], 1);
      }
    }
    __syncthreads();
    // A39: edges >= th (rank-sorted below); the strongest as the fallback
    for (int k2 = threadIdx.x; k2 < a.n_kf; k2 += blockDim.x) {
      const int w = s_w[k2];
      if (w <= 0) continue;
      if (w >= a.th) {
        const int e = atomicAdd(&s_ne, 1);
        if (e < EDGE_CAP) s_e[e] = ((unsigned long long)(0x7FFFFFFF - w) << 32) | (unsigned)k2;
      }
    }
    __syncthreads();
    int ne = s_ne;
    if (ne == 0) {   // strongest edge: max weight, lowest id (serial over n_kf in thread 0)
      if (threadIdx.x == 0) {
        int best = -1;
        for (int k2 = 0; k2 < a.n_kf; ++k2)
          if (s_w[k2] > 0 && (best < 0 || s_w[k2] > s_w[best])) best = k2;
        s_best = best;
        if (best >= 0) s_e[0] = ((unsigned long long)(0x7FFFFFFF - s_w[best]) << 32) | (unsigned)best;
      }
      __syncthreads();
      ne = s_best >= 0 ? 1 : 0;
    }
    // A40: rank of each edge key (distinct keys) -> output slot
    if (ne > EDGE_CAP) {   // rare: more edges than the shared list holds -> rank every edge
      for (int k2 = threadIdx.x; k2 < a.n_kf; k2 += blockDim.x) {   // against the weight array itself
        const int w = s_w[k2];
        if (w < a.th) continue;
        int r = 0;
        for (int j = 0; j < a.n_kf && r < a.max_edges; ++j) {
          const int wj = s_w[j];
          r += (wj >= a.th) && (wj > w || (wj == w && j < k2));
        }
        if (r < a.max_edges && a.out_kf) {
          a.out_kf[(size_t)t * a.max_edges + r] = k2;
          a.out_w[(size_t)t * a.max_edges + r] = w;
        }
      }
    }
    const int nr = ne > EDGE_CAP ? 0 : ne;
    for (int e = threadIdx.x; e < nr; e += blockDim.x) {
      const unsigned long long key = s_e[e];
      int r = 0;
      for (int j = 0; j < nr; ++j) r += s_e[j] < key;
      if (r < a.max_edges && a.out_kf) {
        a.out_kf[(size_t)t * a.max_edges + r] = (int32_t)(key & 0xFFFFFFFFull);
        a.out_w[(size_t)t * a.max_edges + r] = 0x7FFFFFFF - (int32_t)(key >> 32);
      }
    }
    if (threadIdx.x == 0) {
      if (a.out_n) a.out_n[t] = ne;
      ++c_kf;
      c_edges += (uint32_t)ne;
    }
    __syncthreads();
  }
  if (threadIdx.x == 0 && c_kf) {
    atomicAdd(&a.counts[LC_COUNT_CONN_KF], (unsigned long long)c_kf);
    atomicAdd(&a.counts[LC_COUNT_CONN_EDGES], (unsigned long long)c_edges);
  }
}

}  // namespace

int connections_max_kf() { return 40000; }

cudaError_t launch_connections(lc_ctx* c, int n_sel, const int32_t* d_idx, int th, int max_edges,
                               const int32_t* d_obeg, const int32_t* d_obs, const int32_t* d_obs_kf,
                               uint8_t* d_first, int32_t* out_n,
                               int32_t* out_kf, int32_t* out_w, unsigned long long* counts,
                               cudaStream_t s) {
  Store& st = c->st;
  if (n_sel <= 0) return cudaSuccess;
  ConnArgs a;
  a.n_sel = n_sel; a.n_kf = st.n_kf; a.n_mp = st.n_mp; a.th = th; a.max_edges = max_edges;
  a.idx = d_idx; a.kf_fbeg = st.kf_fbeg; a.feat_mp = st.feat_mp; a.flags = st.mp_flags;
  a.obeg = d_obeg; a.obs = d_obs; a.obs_kf = d_obs_kf; a.feat_first = d_first; a.out_n = out_n; a.out_kf = out_kf; a.out_w = out_w; a.counts = counts;
  if (st.n_feat > 0) {   // first-slot flags over every observation
    k_feat_first<<<std::min<int64_t>(((int64_t)st.n_feat + LC_NTHREADS - 1) / LC_NTHREADS, 148 * 32),
                   LC_NTHREADS, 0, s>>>(st.n_mp, st.feat_mp, d_obeg, d_obs, d_obs_kf, d_first);
    c->launches++;
  }
  const size_t smem = sizeof(int32_t) * (size_t)std::max(st.n_kf, 1);
  cudaError_t e = set_smem_attr((const void*)k_connections, (int)smem);
  if (e != cudaSuccess) return e;
  k_connections<<<std::min(n_sel, 148 * 4), LC_NTHREADS, smem, s>>>(a);
  c->launches++;
  return cudaGetLastError();
}
