// k_ransac.cu -- batched Sim3 RANSAC of region detection (
// PAPER.md:89 "estimating the relative pose between the new keyframe and the matched
// one", PAPER.md:200 (hypotheses evaluated in parallel); readings A41-A44;
// include/lc.h lc_sim3_ransac).
//
// CTA per problem (hypothesis pair of keyframes), thread per RANSAC iteration: Horn's
// closed-form similarity of the iteration's 3-point sample (centroids, cross-covariance,
// Horn's 4x4 N, max-eigenvalue eigenvector by cyclic Jacobi, quaternion -> R, scale,
// translation), then the symmetric reprojection inlier count over the problem's
// correspondences (staged in shared memory). Block argmax of (inliers, -iteration),
// inlier mask of the winner, optional refit on all inliers. Every fp64 expression is
// written in the oracle's order (the build uses -fmad=false), so the models, counts
// and masks are identical to oracle O13.
#include <cuda_runtime.h>

#include <algorithm>

#include "lc_internal.cuh"

namespace {

constexpr int RCAP = 512;   // correspondences staged per problem

__device__ void jacobi4(const double* A_in, double* ev, double* V) {
  double A[16];
  for (int i = 0; i < 16; ++i) { A[i] = A_in[i]; V[i] = (i % 5 == 0) ? 1.0 : 0.0; }
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
        for (int k = 0; k < 4; ++k) {
          const double akp = A[4 * k + p], akq = A[4 * k + q];
          A[4 * k + p] = c * akp - sn * akq;
          A[4 * k + q] = sn * akp + c * akq;
        }
        for (int k = 0; k < 4; ++k) {
          const double apk = A[4 * p + k], aqk = A[4 * q + k];
          A[4 * p + k] = c * apk - sn * aqk;
          A[4 * q + k] = sn * apk + c * aqk;
        }
        for (int k = 0; k < 4; ++k) {
          const double vkp = V[4 * k + p], vkq = V[4 * k + q];
          V[4 * k + p] = c * vkp - sn * vkq;
          V[4 * k + q] = sn * vkp + c * vkq;
        }
      }
  }
  for (int i = 0; i < 4; ++i) ev[i] = A[4 * i + i];
}

// Horn's similarity S12 (p1 ~ s R p2 + t) of the n correspondences idx[0..n) (A42)
template <typename PtAt>
__device__ void horn(int n, PtAt pt, int fix_scale, double* S) {
  double c1[3] = {0, 0, 0}, c2[3] = {0, 0, 0};
  for (int i = 0; i < n; ++i) {
    const double* a = pt(i, 1);
    const double* b = pt(i, 2);
    for (int j = 0; j < 3; ++j) { c1[j] = c1[j] + a[j]; c2[j] = c2[j] + b[j]; }
  }
  for (int j = 0; j < 3; ++j) { c1[j] = c1[j] / (double)n; c2[j] = c2[j] / (double)n; }
  double M[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
  for (int i = 0; i < n; ++i) {
    const double* pa = pt(i, 1);
    const double* pb = pt(i, 2);
    double a[3], b[3];
    for (int j = 0; j < 3; ++j) { a[j] = pa[j] - c1[j]; b[j] = pb[j] - c2[j]; }
    for (int r = 0; r < 3; ++r)
      for (int cc = 0; cc < 3; ++cc) M[3 * r + cc] = M[3 * r + cc] + b[r] * a[cc];
  }
  double N[16];
  N[0] = (M[0] + M[4]) + M[8];  N[1] = M[5] - M[7];          N[2] = M[6] - M[2];          N[3] = M[1] - M[3];
  N[5] = (M[0] - M[4]) - M[8];  N[6] = M[1] + M[3];          N[7] = M[6] + M[2];
  N[10] = (-M[0] + M[4]) - M[8]; N[11] = M[5] + M[7];
  N[15] = (-M[0] - M[4]) + M[8];
  N[4] = N[1]; N[8] = N[2]; N[12] = N[3]; N[9] = N[6]; N[13] = N[7]; N[14] = N[11];
  double ev[4], V[16];
  jacobi4(N, ev, V);
  int best = 0;
  for (int i = 1; i < 4; ++i) if (ev[i] > ev[best]) best = i;
  double q[4] = {V[best], V[4 + best], V[8 + best], V[12 + best]};
  int lead = 0;
  while (lead < 3 && q[lead] == 0.0) ++lead;
  if (q[lead] < 0.0) for (int i = 0; i < 4; ++i) q[i] = -q[i];
  const double w = q[0], x = q[1], y = q[2], z = q[3];
  double R[9];
  R[0] = ((w * w + x * x) - y * y) - z * z; R[1] = 2.0 * (x * y - w * z);         R[2] = 2.0 * (x * z + w * y);
  R[3] = 2.0 * (x * y + w * z);         R[4] = ((w * w - x * x) + y * y) - z * z; R[5] = 2.0 * (y * z - w * x);
  R[6] = 2.0 * (x * z - w * y);         R[7] = 2.0 * (y * z + w * x);         R[8] = ((w * w - x * x) - y * y) + z * z;
  double nom = 0.0, den = 0.0;
  for (int i = 0; i < n; ++i) {
    const double* pa = pt(i, 1);
    const double* pb = pt(i, 2);
    double a[3], b[3], rb[3];
    for (int j = 0; j < 3; ++j) { a[j] = pa[j] - c1[j]; b[j] = pb[j] - c2[j]; }
    for (int j = 0; j < 3; ++j) rb[j] = lc_row3(R + 3 * j, b);
    nom = nom + ((a[0] * rb[0] + a[1] * rb[1]) + a[2] * rb[2]);
    den = den + ((rb[0] * rb[0] + rb[1] * rb[1]) + rb[2] * rb[2]);
  }
  const double sc = fix_scale ? 1.0 : nom / den;
  for (int i = 0; i < 9; ++i) S[i] = R[i];
  for (int j = 0; j < 3; ++j) S[9 + j] = c1[j] - sc * lc_row3(R + 3 * j, c2);
  S[12] = sc;
}

struct RansacArgs {
  int n_prob, n_iter, fix_scale, refit;
  double chi2;
  const int32_t* pbeg;
  const double* P1;
  const double* P2;
  const float* uv1;
  const float* uv2;
  const float* sig1;
  const float* sig2;
  const int32_t* cam1;
  const int32_t* cam2;
  const int32_t* samples;
  const DevCam* cams;
  double* out_S;
  int32_t* out_inl;
  uint8_t* out_mask;
  unsigned long long* counts;
};

// A43: both reprojection errors below chi2 * sigma^2; behind a camera = outlier
__device__ __forceinline__ bool inlier(const DevCam& k1, const DevCam& k2, const double* S12,
                                       const double* S21, const double* p1, const double* p2,
                                       float2 u1, float2 u2, float s1, float s2, double chi2) {
  double a[3], b[3], u, v;
  lc_sim3_apply(S12, p2, a);
  if (a[2] <= 0.0) return false;
  lc_project(k1, a[0], a[1], a[2], u, v);
  double du = u - (double)u1.x, dv = v - (double)u1.y;
  if (!(du * du + dv * dv < chi2 * (double)s1)) return false;
  lc_sim3_apply(S21, p1, b);
  if (b[2] <= 0.0) return false;
  lc_project(k2, b[0], b[1], b[2], u, v);
  du = u - (double)u2.x; dv = v - (double)u2.y;
  return du * du + dv * dv < chi2 * (double)s2;
}

__global__ void __launch_bounds__(LC_NTHREADS) k_ransac(const RansacArgs a) {
  __shared__ double s_p1[RCAP][3], s_p2[RCAP][3];
  __shared__ float2 s_u1[RCAP], s_u2[RCAP];
  __shared__ float s_s1[RCAP], s_s2[RCAP];
  __shared__ unsigned long long s_best;   // (inliers << 32) | (0xFFFFFFFF - iteration)
  __shared__ double s_S[13];
  __shared__ int32_t s_sel[RCAP];
  __shared__ int s_ns;
  __shared__ DevCam s_k1, s_k2;
  const int tid = threadIdx.x;
  uint32_t c_hyp = 0;
  for (int b = blockIdx.x; b < a.n_prob; b += gridDim.x) {
    const int c0 = a.pbeg[b], nc = a.pbeg[b + 1] - c0;
    const bool staged = nc <= RCAP;
    if (tid == 0) { s_best = 0ull; s_ns = 0; s_k1 = a.cams[a.cam1[b]]; s_k2 = a.cams[a.cam2[b]]; }
    if (staged)
      for (int i = tid; i < nc; i += blockDim.x) {
        for (int j = 0; j < 3; ++j) { s_p1[i][j] = a.P1[3 * (size_t)(c0 + i) + j]; s_p2[i][j] = a.P2[3 * (size_t)(c0 + i) + j]; }
        s_u1[i] = reinterpret_cast<const float2*>(a.uv1)[c0 + i];
        s_u2[i] = reinterpret_cast<const float2*>(a.uv2)[c0 + i];
        s_s1[i] = a.sig1[c0 + i];
        s_s2[i] = a.sig2[c0 + i];
      }
    __syncthreads();
    auto P = [&](int i, int side) -> const double* {
      if (staged) return side == 1 ? s_p1[i] : s_p2[i];
      return (side == 1 ? a.P1 : a.P2) + 3 * (size_t)(c0 + i);
    };
    auto U = [&](int i, int side) -> float2 {
      if (staged) return side == 1 ? s_u1[i] : s_u2[i];
      return reinterpret_cast<const float2*>(side == 1 ? a.uv1 : a.uv2)[c0 + i];
    };
    auto SG = [&](int i, int side) -> float {
      if (staged) return side == 1 ? s_s1[i] : s_s2[i];
      return (side == 1 ? a.sig1 : a.sig2)[c0 + i];
    };
    auto count = [&](const double* S, const double* Si) {
      int n = 0;
      for (int i = 0; i < nc; ++i)
        n += inlier(s_k1, s_k2, S, Si, P(i, 1), P(i, 2), U(i, 1), U(i, 2), SG(i, 1), SG(i, 2), a.chi2);
      return n;
    };
    // (1) hypotheses
    for (int it = tid; it < a.n_iter; it += blockDim.x) {
      const int32_t* t = a.samples + 3 * ((size_t)b * a.n_iter + it);
      const int i0 = t[0], i1 = t[1], i2 = t[2];
      if (i0 < 0 || i1 < 0 || i2 < 0 || i0 >= nc || i1 >= nc || i2 >= nc || i0 == i1 || i0 == i2 || i1 == i2)
        continue;   // A41
      const int sel[3] = {i0, i1, i2};
      double S[13], Si[13];
      horn(3, [&](int i, int side) { return P(sel[i], side); }, a.fix_scale, S);
      lc_sim3_inverse(S, Si);
      ++c_hyp;
      const int n = count(S, Si);
      atomicMax(&s_best, ((unsigned long long)(uint32_t)n << 32) | (0xFFFFFFFFull - (uint32_t)it));
    }
    __syncthreads();
    const unsigned long long best = s_best;
    const bool any = best != 0ull;
    const int best_it = any ? (int)(0xFFFFFFFFull - (best & 0xFFFFFFFFull)) : -1;
    // (2) the winner's model (recomputed by thread 0: the same expressions), mask, refit
    if (tid == 0 && any) {
      const int32_t* t = a.samples + 3 * ((size_t)b * a.n_iter + best_it);
      const int sel[3] = {t[0], t[1], t[2]};
      double S[13];
      horn(3, [&](int i, int side) { return P(sel[i], side); }, a.fix_scale, S);
      for (int i = 0; i < 13; ++i) s_S[i] = S[i];
    }
    __syncthreads();
    if (!any) {
      for (int i = tid; i < nc; i += blockDim.x) a.out_mask[c0 + i] = 0;
      if (tid == 0) {
        for (int i = 0; i < 13; ++i) a.out_S[13 * (size_t)b + i] = 0.0;
        a.out_inl[b] = 0;
      }
      __syncthreads();
      continue;
    }
    double S[13], Si[13];
    for (int i = 0; i < 13; ++i) S[i] = s_S[i];
    lc_sim3_inverse(S, Si);
    for (int i = tid; i < nc; i += blockDim.x) {
      const bool in = inlier(s_k1, s_k2, S, Si, P(i, 1), P(i, 2), U(i, 1), U(i, 2), SG(i, 1), SG(i, 2), a.chi2);
      a.out_mask[c0 + i] = in ? 1 : 0;
      if (in) atomicAdd(&s_ns, 1);
    }
    __syncthreads();
    if (tid == 0) {
      const int ns = s_ns;
      a.out_inl[b] = ns;
      atomicAdd(&a.counts[LC_COUNT_RANSAC_INLIERS], (unsigned long long)ns);
      if (a.refit && ns >= 3) {   // A44: Horn on all inliers, in index order
        if (ns <= RCAP) {
          int k = 0;
          for (int i = 0; i < nc; ++i) if (a.out_mask[c0 + i]) s_sel[k++] = i;
          horn(ns, [&](int i, int side) { return P(s_sel[i], side); }, a.fix_scale, S);
        } else {   // many inliers: walk the mask for every access (same order, slower)
          auto nth = [&](int r) { int k = -1; for (int i = 0; i < nc; ++i) if (a.out_mask[c0 + i] && ++k == r) return i; return 0; };
          horn(ns, [&](int i, int side) { return P(nth(i), side); }, a.fix_scale, S);
        }
      }
      for (int i = 0; i < 13; ++i) a.out_S[13 * (size_t)b + i] = S[i];
    }
    __syncthreads();
  }
  // hypotheses evaluated
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) c_hyp += __shfl_down_sync(0xffffffffu, c_hyp, o);
  if ((tid & 31) == 0 && c_hyp) atomicAdd(&a.counts[LC_COUNT_RANSAC_HYP], (unsigned long long)c_hyp);
}

// ---------------------------------------------------------------------------
// Sim3 refinement (readings A45-A48): Gauss-Newton with central-difference Jacobians,
// Huber weights, outlier removal between the two phases. Per step: threads compute
// each correspondence's residuals / Jacobians / weights into shared memory (chunks
// of RCH), then 35 threads -- one per entry of H (lower 28) and g (7) -- accumulate in
// the oracle's (correspondence, residual) order, so every sum, the fixed-order 7x7
// Cholesky (thread 0) and the retraction are the oracle's bits.
// ---------------------------------------------------------------------------
constexpr int RCH = 64;

__device__ __forceinline__ void retract(const double* d, const double* S, double* out) {   // A45
  const double a = d[0], b = d[1], c = d[2];
  const double n2 = (a * a + b * b) + c * c;
  const double k = 1.0 / (1.0 + n2);
  double D[13];
  D[0] = ((1.0 + a * a) - b * b - c * c) * k;  D[1] = 2.0 * (a * b - c) * k;          D[2] = 2.0 * (a * c + b) * k;
  D[3] = 2.0 * (a * b + c) * k;          D[4] = ((1.0 - a * a) + b * b - c * c) * k;  D[5] = 2.0 * (b * c - a) * k;
  D[6] = 2.0 * (a * c - b) * k;          D[7] = 2.0 * (b * c + a) * k;          D[8] = ((1.0 - a * a) - b * b + c * c) * k;
  D[9] = d[3]; D[10] = d[4]; D[11] = d[5]; D[12] = 1.0 + d[6];
  lc_sim3_compose(D, S, out);
}

__device__ __forceinline__ bool residuals(const DevCam& k1, const DevCam& k2, const double* S, const double* p1,
                                          const double* p2, float2 u1, float2 u2, double* r) {
  double Si[13], a[3], b[3], u, v;
  lc_sim3_inverse(S, Si);
  lc_sim3_apply(S, p2, a);
  lc_sim3_apply(Si, p1, b);
  if (a[2] <= 0.0 || b[2] <= 0.0) return false;
  lc_project(k1, a[0], a[1], a[2], u, v);
  r[0] = u - (double)u1.x; r[1] = v - (double)u1.y;
  lc_project(k2, b[0], b[1], b[2], u, v);
  r[2] = u - (double)u2.x; r[3] = v - (double)u2.y;
  return true;
}

__device__ __forceinline__ double huber_w(double e2, double delta) {
  const double e = sqrt(e2);
  return e <= delta ? 1.0 : delta / e;
}

struct RefineArgs {
  int n_prob, max_iter;
  double th2, lambda;
  const int32_t* pbeg;
  const double* P1;
  const double* P2;
  const float* uv1;
  const float* uv2;
  const float* sig1;
  const float* sig2;
  const int32_t* cam1;
  const int32_t* cam2;
  const double* S_in;
  const DevCam* cams;
  double* out_S;
  int32_t* out_inl;
  uint8_t* out_mask;   // also the active flags during the refinement
  unsigned long long* counts;
};

__global__ void __launch_bounds__(LC_NTHREADS) k_refine(const RefineArgs a) {
  __shared__ double s_J[RCH][4][7], s_r[RCH][4], s_w[RCH][2];
  __shared__ uint8_t s_ok[RCH], s_okj[RCH][7];
  __shared__ double s_H[49], s_g[7], s_S[13], s_dn;
  __shared__ int s_spd, s_ninl;
  __shared__ DevCam s_k1, s_k2;
  const int tid = threadIdx.x;
  const double delta = sqrt(a.th2), h = 1e-6;
  uint32_t c_it = 0, c_inl = 0;
  for (int b = blockIdx.x; b < a.n_prob; b += gridDim.x) {
    const int c0 = a.pbeg[b], nc = a.pbeg[b + 1] - c0;
    if (tid == 0) {
      for (int i = 0; i < 13; ++i) s_S[i] = a.S_in[13 * (size_t)b + i];
      s_k1 = a.cams[a.cam1[b]];
      s_k2 = a.cams[a.cam2[b]];
      s_ninl = 0;
    }
    for (int i = tid; i < nc; i += blockDim.x) a.out_mask[c0 + i] = 1;   // active
    __syncthreads();
    auto P = [&](int i, int side) { return (side == 1 ? a.P1 : a.P2) + 3 * (size_t)(c0 + i); };
    auto U = [&](int i, int side) { return reinterpret_cast<const float2*>(side == 1 ? a.uv1 : a.uv2)[c0 + i]; };
    auto chi2 = [&](const double* S, int i, double& e1, double& e2) -> bool {
      double r[4];
      if (!residuals(s_k1, s_k2, S, P(i, 1), P(i, 2), U(i, 1), U(i, 2), r)) return false;
      e1 = (r[0] * r[0] + r[1] * r[1]) / (double)a.sig1[c0 + i];
      e2 = (r[2] * r[2] + r[3] * r[3]) / (double)a.sig2[c0 + i];
      return true;
    };
    for (int phase = 0; phase < 2; ++phase) {
      const int n_it = phase == 0 ? min(a.max_iter, 5) : a.max_iter;
      for (int it = 0; it < n_it; ++it) {
        double S[13];
        for (int i = 0; i < 13; ++i) S[i] = s_S[i];
        if (tid < 49) s_H[tid] = 0.0;
        if (tid < 7) s_g[tid] = 0.0;
        __syncthreads();
        for (int ch = 0; ch < nc; ch += RCH) {
          const int n = min(RCH, nc - ch);
          // one work item per (correspondence, Jacobian column): the 14 perturbed residual
          // evaluations of a correspondence run on 7 threads (the values are the same as
          // a thread per correspondence would compute; only the assignment changes)
          for (int wk = tid; wk < n * 7; wk += blockDim.x) {
            const int l = wk / 7, j = wk - 7 * l, i = ch + l;
            bool ok = a.out_mask[c0 + i] != 0;
            if (j == 0) {
              double r[4];
              const bool ok0 = ok && residuals(s_k1, s_k2, S, P(i, 1), P(i, 2), U(i, 1), U(i, 2), r);
              s_ok[l] = ok0 ? 1 : 0;
              if (ok0) {
                const double s1 = (double)a.sig1[c0 + i], s2 = (double)a.sig2[c0 + i];
                const double e1 = (r[0] * r[0] + r[1] * r[1]) / s1, e2 = (r[2] * r[2] + r[3] * r[3]) / s2;
                for (int q = 0; q < 4; ++q) s_r[l][q] = r[q];
                s_w[l][0] = huber_w(e1, delta) / s1;
                s_w[l][1] = huber_w(e2, delta) / s2;
              }
            }
            if (ok) {
              double dp[7] = {0, 0, 0, 0, 0, 0, 0}, dm[7] = {0, 0, 0, 0, 0, 0, 0};
              dp[j] = h; dm[j] = -h;
              double Sp[13], Sm[13], rp[4], rm[4];
              retract(dp, S, Sp);
              retract(dm, S, Sm);
              ok = residuals(s_k1, s_k2, Sp, P(i, 1), P(i, 2), U(i, 1), U(i, 2), rp) &&
                   residuals(s_k1, s_k2, Sm, P(i, 1), P(i, 2), U(i, 1), U(i, 2), rm);
              for (int q = 0; q < 4; ++q) s_J[l][q][j] = (rp[q] - rm[q]) / (2.0 * h);
            }
            s_okj[l][j] = ok ? 1 : 0;
          }
          __syncthreads();
          for (int l = tid; l < n; l += blockDim.x) {   // usable iff every evaluation succeeded
            uint8_t all = s_ok[l];
            for (int j = 0; j < 7; ++j) all &= s_okj[l][j];
            s_ok[l] = all;
          }
          __syncthreads();
          if (tid < 35) {   // one entry per thread, accumulated in (correspondence, residual) order
            int x, y;
            if (tid < 28) { x = 0; while ((x + 1) * (x + 2) / 2 <= tid) ++x; y = tid - x * (x + 1) / 2; }
            else { x = tid - 28; y = -1; }
            double acc = y >= 0 ? s_H[7 * x + y] : s_g[x];
            // branch-free so the products of later correspondences are formed while the
            // ordered additions run: a skipped correspondence adds +0.0, which leaves the
            // accumulator's bits unchanged (it starts at +0.0 and never becomes -0.0)
#pragma unroll 4
            for (int l = 0; l < n; ++l) {
              const bool okl = s_ok[l] != 0;
#pragma unroll
              for (int q = 0; q < 4; ++q) {
                const double wq = q < 2 ? s_w[l][0] : s_w[l][1];
                const double other = y >= 0 ? s_J[l][q][y] : s_r[l][q];
                const double prod = wq * s_J[l][q][x] * other;
                acc = acc + (okl ? prod : 0.0);
              }
            }
            if (y >= 0) s_H[7 * x + y] = acc; else s_g[x] = acc;
          }
          __syncthreads();
        }
        if (tid == 0) {   // H + lambda diag(H) = L L^T, H d = -g, S <- retract(d) S
          double L[49];
          for (int x = 0; x < 7; ++x)
            for (int y = 0; y <= x; ++y) L[7 * x + y] = s_H[7 * x + y] + (x == y ? a.lambda * s_H[7 * x + x] : 0.0);
          int spd = 1;
          for (int x = 0; x < 7 && spd; ++x)
            for (int y = 0; y <= x; ++y) {
              double acc = L[7 * x + y];
              for (int k = 0; k < y; ++k) acc = acc - L[7 * x + k] * L[7 * y + k];
              if (x == y) {
                if (!(acc > 0.0)) { spd = 0; break; }
                L[7 * x + x] = sqrt(acc);
              } else {
                L[7 * x + y] = acc / L[7 * y + y];
              }
            }
          s_spd = spd;
          if (spd) {
            double z[7], d[7];
            for (int x = 0; x < 7; ++x) {
              double acc = -s_g[x];
              for (int k = 0; k < x; ++k) acc = acc - L[7 * x + k] * z[k];
              z[x] = acc / L[7 * x + x];
            }
            for (int x = 6; x >= 0; --x) {
              double acc = z[x];
              for (int k = x + 1; k < 7; ++k) acc = acc - L[7 * k + x] * d[k];
              d[x] = acc / L[7 * x + x];
            }
            double S2[13];
            retract(d, S, S2);
            for (int i = 0; i < 13; ++i) s_S[i] = S2[i];
            double dn = 0.0;
            for (int x = 0; x < 7; ++x) dn = dn + d[x] * d[x];
            s_dn = dn;
            ++c_it;
          }
        }
        __syncthreads();
        if (!s_spd || s_dn < 1e-20) break;
      }
      if (phase == 0) {   // drop correspondences with a chi2 >= th2 (EXT OptimizeSim3)
        double S[13];
        for (int i = 0; i < 13; ++i) S[i] = s_S[i];
        for (int i = tid; i < nc; i += blockDim.x) {
          double e1, e2;
          const bool in = chi2(S, i, e1, e2) && e1 < a.th2 && e2 < a.th2;
          a.out_mask[c0 + i] = in ? 1 : 0;
        }
        __syncthreads();
      }
    }
    double S[13];
    for (int i = 0; i < 13; ++i) S[i] = s_S[i];
    for (int i = tid; i < nc; i += blockDim.x) {
      double e1, e2;
      const bool in = chi2(S, i, e1, e2) && e1 < a.th2 && e2 < a.th2;
      a.out_mask[c0 + i] = in ? 1 : 0;
      if (in) atomicAdd(&s_ninl, 1);
    }
    __syncthreads();
    if (tid == 0) {
      a.out_inl[b] = s_ninl;
      c_inl += (uint32_t)s_ninl;
      for (int i = 0; i < 13; ++i) a.out_S[13 * (size_t)b + i] = s_S[i];
    }
    __syncthreads();
  }
  if (tid == 0 && (c_it || c_inl)) {
    atomicAdd(&a.counts[LC_COUNT_REFINE_ITERS], (unsigned long long)c_it);
    atomicAdd(&a.counts[LC_COUNT_REFINE_INLIERS], (unsigned long long)c_inl);
  }
}

}  // namespace

cudaError_t launch_refine(lc_ctx* c, int n_prob, const int32_t* d_pbeg, const double* P1, const double* P2,
                          const float* uv1, const float* uv2, const float* sig1, const float* sig2,
                          const int32_t* d_cam1, const int32_t* d_cam2, const double* S_in, int max_iter,
                          double th2, double lambda, double* out_S, int32_t* out_inl, uint8_t* out_mask,
                          unsigned long long* counts, cudaStream_t s) {
  if (n_prob <= 0) return cudaSuccess;
  RefineArgs a;
  a.n_prob = n_prob; a.max_iter = max_iter; a.th2 = th2; a.lambda = lambda;
  a.pbeg = d_pbeg; a.P1 = P1; a.P2 = P2; a.uv1 = uv1; a.uv2 = uv2; a.sig1 = sig1; a.sig2 = sig2;
  a.cam1 = d_cam1; a.cam2 = d_cam2; a.S_in = S_in; a.cams = c->st.cams;
  a.out_S = out_S; a.out_inl = out_inl; a.out_mask = out_mask; a.counts = counts;
  k_refine<<<std::min(n_prob, 148 * 8), LC_NTHREADS, 0, s>>>(a);
  c->launches++;
  return cudaGetLastError();
}

cudaError_t launch_ransac(lc_ctx* c, int n_prob, const int32_t* d_pbeg, const double* P1, const double* P2,
                          const float* uv1, const float* uv2, const float* sig1, const float* sig2,
                          const int32_t* d_cam1, const int32_t* d_cam2, const int32_t* samples, int n_iter,
                          double chi2, int fix_scale, int refit, double* out_S, int32_t* out_inl,
                          uint8_t* out_mask, unsigned long long* counts, cudaStream_t s) {
  if (n_prob <= 0) return cudaSuccess;
  RansacArgs a;
  a.n_prob = n_prob; a.n_iter = n_iter; a.fix_scale = fix_scale; a.refit = refit; a.chi2 = chi2;
  a.pbeg = d_pbeg; a.P1 = P1; a.P2 = P2; a.uv1 = uv1; a.uv2 = uv2; a.sig1 = sig1; a.sig2 = sig2;
  a.cam1 = d_cam1; a.cam2 = d_cam2; a.samples = samples; a.cams = c->st.cams;
  a.out_S = out_S; a.out_inl = out_inl; a.out_mask = out_mask; a.counts = counts;
  k_ransac<<<std::min(n_prob, 148 * 8), LC_NTHREADS, 0, s>>>(a);
  c->launches++;
  return cudaGetLastError();
}
