// k_store.cu -- device map store: SoA -> packed store, per-keyframe grid build,
// association recount, state save/restore (keyframes
// kept GPU-resident in a "lightweight wrapper structure", allocated once).
#include <cuda_runtime.h>

#include <cstring>

#include "lc_internal.cuh"

namespace {

enum { ERR_OCTAVE = 0, ERR_FEAT_MP, ERR_REF_KF, ERR_CAM, ERR_N };

// Map-point rows: pos, dmax, normal, angle, descriptor -> one 64-B record.
__global__ void k_pack_mp(int n_mp, int n_kf, const float* __restrict__ pos,
                          const float* __restrict__ nrm, const float* __restrict__ dmax,
                          const uint8_t* __restrict__ desc, const float* __restrict__ ang,
                          const int32_t* __restrict__ ref_kf, MpRec* __restrict__ out,
                          int32_t* __restrict__ replaced_by, int32_t* __restrict__ corr_ref,
                          uint32_t* __restrict__ loop_ep, int32_t* __restrict__ nobs,
                          uint32_t* __restrict__ errs) {
  for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < n_mp; q += gridDim.x * blockDim.x) {
    MpRec r;
    r.pos[0] = pos[3 * q + 0]; r.pos[1] = pos[3 * q + 1]; r.pos[2] = pos[3 * q + 2];
    r.dmax = dmax[q];
    r.normal[0] = nrm[3 * q + 0]; r.normal[1] = nrm[3 * q + 1]; r.normal[2] = nrm[3 * q + 2];
    r.angle = ang[q];
    uint32_t w[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const uint8_t* d = desc + 32 * (size_t)q + 4 * i;
      w[i] = (uint32_t)d[0] | ((uint32_t)d[1] << 8) | ((uint32_t)d[2] << 16) | ((uint32_t)d[3] << 24);
    }
    r.desc[0] = make_uint4(w[0], w[1], w[2], w[3]);
    r.desc[1] = make_uint4(w[4], w[5], w[6], w[7]);
    out[q] = r;
    replaced_by[q] = -1;
    corr_ref[q] = -1;
    loop_ep[q] = 0u;
    nobs[q] = 0;
    int rk = ref_kf[q];
    if (rk < 0 || rk >= n_kf) atomicAdd(&errs[ERR_REF_KF], 1u);
  }
}

__global__ void k_count_nobs(int n_feat, int n_mp, const int32_t* __restrict__ feat_mp,
                             int32_t* __restrict__ nobs, uint32_t* __restrict__ errs) {
  for (int f = blockIdx.x * blockDim.x + threadIdx.x; f < n_feat; f += gridDim.x * blockDim.x) {
    int m = feat_mp[f];
    if (m >= n_mp || m < -1) { atomicAdd(&errs[ERR_FEAT_MP], 1u); continue; }
    if (m >= 0) atomicAdd(&nobs[m], 1);
  }
}

// Per-keyframe counting sort of features into the per-octave grid cells (one CTA per
// keyframe). A feature of octave o goes to cell (o, floor((v-min_y)*rows_o/(max_y-min_y)),
// floor((u-min_x)*cols_o/(max_x-min_x))), clamped; the cell table and the feature arrays
// are (octave, row, col)-major, and within a cell features keep ascending original index.
__global__ void __launch_bounds__(LC_NTHREADS) k_grid_build(
    int kf0, int f0, int n_levels, int n_cams, int Gs, int G, MatchArgs g, const int32_t* __restrict__ fbeg,
    const int32_t* __restrict__ fpad, const int32_t* __restrict__ kf_cam,
    const DevCam* __restrict__ cams, const float* __restrict__ fuv, const uint8_t* __restrict__ foct,
    const uint8_t* __restrict__ fdesc, uint16_t* __restrict__ kf_cell, float2* __restrict__ fc_uv,
    uint32_t* __restrict__ fc_meta, uint4* __restrict__ fc_desc, int32_t* __restrict__ feat_cpos,
    uint32_t* __restrict__ errs) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int k = kf0 + blockIdx.x;     // keyframes [kf0, kf0 + gridDim.x) of the store
  const int fb = fbeg[k];
  const int F = fbeg[k + 1] - fb;
  const int fp = fpad[k];
  const int ci = kf_cam[k];
  const int fi = fb - f0;             // the inputs hold the features from store index f0 on
  if (ci < 0 || ci >= n_cams) {
    if (threadIdx.x == 0) atomicAdd(&errs[ERR_CAM], 1u);
    return;
  }
  const DevCam& cam = cams[ci];
  int* s_cnt = (int*)smem;                              // [G+1]
  uint16_t* s_cellof = (uint16_t*)(s_cnt + G + 1);      // [F]
  uint16_t* s_perm = s_cellof + F;                      // [F]
  __shared__ int s_part[LC_NTHREADS];
  for (int i = threadIdx.x; i <= G; i += blockDim.x) s_cnt[i] = 0;
  __syncthreads();
  for (int f = threadIdx.x; f < F; f += blockDim.x) {
    const int o = foct[fi + f];
    if (o >= n_levels) { atomicAdd(&errs[ERR_OCTAVE], 1u); s_cellof[f] = 0; continue; }
    const int cols = g.ocols[o], rows = g.orows[o];
    double u = (double)fuv[2 * (fi + f)], v = (double)fuv[2 * (fi + f) + 1];
    double x = floor((u - cam.min_x) * cam.cell_sx[o]);
    double y = floor((v - cam.min_y) * cam.cell_sy[o]);
    int cx = x >= 0.0 ? (x < (double)cols ? (int)x : cols - 1) : 0;
    int cy = y >= 0.0 ? (y < (double)rows ? (int)y : rows - 1) : 0;
    int cell = g.obase[o] + cy * cols + cx;
    s_cellof[f] = (uint16_t)cell;
    atomicAdd(&s_cnt[cell], 1);
  }
  __syncthreads();
  // exclusive scan over G cells: each thread owns a contiguous chunk
  const int per = (G + blockDim.x - 1) / blockDim.x;
  const int c0 = threadIdx.x * per, c1 = min(G, c0 + per);
  int sum = 0;
  for (int i = c0; i < c1; ++i) sum += s_cnt[i];
  s_part[threadIdx.x] = sum;
  __syncthreads();
  if (threadIdx.x == 0) {
    int acc = 0;
    for (int t = 0; t < (int)blockDim.x; ++t) { int x = s_part[t]; s_part[t] = acc; acc += x; }
  }
  __syncthreads();
  int acc = s_part[threadIdx.x];
  for (int i = c0; i < c1; ++i) { int x = s_cnt[i]; s_cnt[i] = acc; acc += x; }
  __syncthreads();
  uint16_t* cell_out = kf_cell + (size_t)k * Gs;
  for (int i = threadIdx.x; i < G; i += blockDim.x) cell_out[i] = (uint16_t)s_cnt[i];
  if (threadIdx.x == 0) { cell_out[G] = (uint16_t)F; s_cnt[G] = F; }
  __syncthreads();
  // scatter with per-cell cursors (order fixed below); s_cnt becomes cell end
  for (int f = threadIdx.x; f < F; f += blockDim.x) {
    int p = atomicAdd(&s_cnt[s_cellof[f]], 1);
    s_perm[p] = (uint16_t)f;
  }
  __syncthreads();
  // sort each cell's slots by original index (cells hold ~1 feature)
  for (int cell = threadIdx.x; cell < G; cell += blockDim.x) {
    int b = cell_out[cell], e = (cell + 1 < G) ? (int)cell_out[cell + 1] : F;
    for (int i = b + 1; i < e; ++i) {
      uint16_t x = s_perm[i];
      int j = i - 1;
      while (j >= b && s_perm[j] > x) { s_perm[j + 1] = s_perm[j]; --j; }
      s_perm[j + 1] = x;
    }
  }
  __syncthreads();
  for (int p = threadIdx.x; p < F; p += blockDim.x) {
    int f = s_perm[p];
    fc_uv[fp + p] = make_float2(fuv[2 * (fi + f)], fuv[2 * (fi + f) + 1]);
    fc_meta[fp + p] = (uint32_t)f | ((uint32_t)foct[fi + f] << 16);
    feat_cpos[fb + f] = fp + p;   // original order -> cell-major position
    const uint8_t* d = fdesc + 32 * (size_t)(fi + f);
    uint32_t w[8];
#pragma unroll
    for (int i = 0; i < 8; ++i)
      w[i] = (uint32_t)d[4 * i] | ((uint32_t)d[4 * i + 1] << 8) | ((uint32_t)d[4 * i + 2] << 16) |
             ((uint32_t)d[4 * i + 3] << 24);
    fc_desc[2 * (size_t)(fp + p)] = make_uint4(w[0], w[1], w[2], w[3]);
    fc_desc[2 * (size_t)(fp + p) + 1] = make_uint4(w[4], w[5], w[6], w[7]);
  }
}

__global__ void k_pos_gather(int n_mp, const MpRec* __restrict__ rec, float* __restrict__ out) {
  for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < n_mp; q += gridDim.x * blockDim.x) {
    out[3 * q + 0] = rec[q].pos[0];
    out[3 * q + 1] = rec[q].pos[1];
    out[3 * q + 2] = rec[q].pos[2];
  }
}

__global__ void k_fill_u64(unsigned long long* p, int64_t n, unsigned long long v) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    p[i] = v;
}

int grid_for(int64_t n) {
  int64_t b = (n + LC_NTHREADS - 1) / LC_NTHREADS;
  if (b < 1) b = 1;
  if (b > 148 * 16) b = 148 * 16;
  return (int)b;
}

}  // namespace

cudaError_t launch_fill_u64(lc_ctx* c, unsigned long long* p, int64_t n, unsigned long long v,
                            cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  k_fill_u64<<<grid_for(n), LC_NTHREADS, 0, s>>>(p, n, v);
  c->launches++;
  return cudaGetLastError();
}

// Packs the store entries [kf0, n_kf), [f0, n_feat), [mp0, n_mp) from the caller's SoA
// inputs (which hold exactly those entries): a whole map (REPLACE: all offsets 0) or the
// keyframes / map points appended by LC_UPLOAD_APPEND.
cudaError_t launch_upload_pack(lc_ctx* c, int kf0, int f0, int mp0, const float* pos, const float* nrm,
                               const float* dmax, const uint8_t* desc, const float* ang, const float* fuv,
                               const uint8_t* foct, const uint8_t* fdesc, uint32_t* d_errs, cudaStream_t s) {
  Store& st = c->st;
  const int n_mp = st.n_mp - mp0, n_feat = st.n_feat - f0, n_kf = st.n_kf - kf0;
  if (n_mp > 0) {
    k_pack_mp<<<grid_for(n_mp), LC_NTHREADS, 0, s>>>(
        n_mp, st.n_kf, pos, nrm, dmax, desc, ang, st.mp_ref_kf + mp0, st.mp_rec + mp0, st.mp_replaced_by + mp0,
        st.mp_corr_ref + mp0, st.mp_loop_ep + mp0, st.mp_nobs + mp0, d_errs);
    c->launches++;
  }
  if (n_feat > 0) {   // n_obs of the referenced points (old or new) += new observations
    k_count_nobs<<<grid_for(n_feat), LC_NTHREADS, 0, s>>>(n_feat, st.n_mp, st.feat_mp + f0, st.mp_nobs, d_errs);
    c->launches++;
  }
  if (n_kf > 0) {
    size_t smem = sizeof(int) * (size_t)(st.G + 1) + 2 * sizeof(uint16_t) * (size_t)st.max_F;
    smem = (smem + 15) & ~(size_t)15;
    cudaError_t e = set_smem_attr((const void*)k_grid_build, (int)smem);
    if (e != cudaSuccess) return e;
    MatchArgs g;   // only the per-octave grid dims are read
    memset(&g, 0, sizeof(g));
    for (int i = 0; i < LC_MAX_LEVELS; ++i) { g.ocols[i] = st.ocols[i]; g.orows[i] = st.orows[i]; }
    for (int i = 0; i <= LC_MAX_LEVELS; ++i) g.obase[i] = st.obase[i];
    k_grid_build<<<n_kf, LC_NTHREADS, smem, s>>>(kf0, f0, st.n_levels, st.n_cams, st.Gs, st.G, g, st.kf_fbeg,
                                                 st.kf_fpad, st.kf_cam, st.cams, fuv, foct, fdesc, st.kf_cell,
                                                 st.fc_uv, st.fc_meta, st.fc_desc, st.feat_cpos, d_errs);
    c->launches++;
  }
  return cudaGetLastError();
}

// Saved-state layout (bytes): kf_pose | kf_S_corr | kf_in_win | feat_mp | mp_rec (64-B
// records) | flags | replaced_by | nobs | corr_ref
static size_t state_bytes(const Store& st, size_t off[10]) {
  size_t o = 0;
  auto add = [&](int i, size_t b) { off[i] = o; o += (b + 255) & ~(size_t)255; };
  add(0, sizeof(double) * 13 * st.n_kf);
  add(1, sizeof(double) * 13 * st.n_kf);
  add(2, sizeof(int32_t) * st.n_kf);
  add(3, sizeof(int32_t) * st.n_feat);
  add(4, sizeof(MpRec) * st.n_mp);
  add(5, sizeof(uint8_t) * st.n_mp);
  add(6, sizeof(int32_t) * st.n_mp);
  add(7, sizeof(int32_t) * st.n_mp);
  add(8, sizeof(int32_t) * st.n_mp);
  off[9] = o;
  return o;
}

cudaError_t launch_state_copy(lc_ctx* c, bool save, cudaStream_t s) {
  Store& st = c->st;
  size_t off[10];
  size_t need = state_bytes(st, off);
  if (save && c->sv_cap < need) {
    if (c->sv) cudaFree(c->sv);
    c->sv = nullptr;
    c->sv_cap = 0;
    cudaError_t e = cudaMalloc(&c->sv, need);
    if (e != cudaSuccess) return e;
    c->sv_cap = need;
  }
  char* b = (char*)c->sv;
  struct { void* dev; size_t o; size_t bytes; } items[] = {
      {st.kf_pose, off[0], sizeof(double) * 13 * st.n_kf},
      {st.kf_S_corr, off[1], sizeof(double) * 13 * st.n_kf},
      {st.kf_in_win, off[2], sizeof(int32_t) * st.n_kf},
      {st.feat_mp, off[3], sizeof(int32_t) * st.n_feat},
      {st.mp_rec, off[4], sizeof(MpRec) * st.n_mp},   // positions, normals, depth bounds, descriptors
      {st.mp_flags, off[5], sizeof(uint8_t) * st.n_mp},
      {st.mp_replaced_by, off[6], sizeof(int32_t) * st.n_mp},
      {st.mp_nobs, off[7], sizeof(int32_t) * st.n_mp},
      {st.mp_corr_ref, off[8], sizeof(int32_t) * st.n_mp},
  };
  for (auto& it : items) {
    if (it.bytes == 0) continue;
    cudaError_t e = save ? cudaMemcpyAsync(b + it.o, it.dev, it.bytes, cudaMemcpyDeviceToDevice, s)
                         : cudaMemcpyAsync(it.dev, b + it.o, it.bytes, cudaMemcpyDeviceToDevice, s);
    if (e != cudaSuccess) return e;
  }
  return cudaGetLastError();
}

cudaError_t launch_download_pos(lc_ctx* c, float* out, cudaStream_t s) {
  if (c->st.n_mp <= 0) return cudaSuccess;
  k_pos_gather<<<grid_for(c->st.n_mp), LC_NTHREADS, 0, s>>>(c->st.n_mp, c->st.mp_rec, out);
  c->launches++;
  return cudaGetLastError();
}
