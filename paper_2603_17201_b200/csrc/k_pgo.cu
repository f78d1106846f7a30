// k_pgo.cu -- essential-graph Sim3 pose-graph optimisation on the device (SURVEY.md
// §8(f) f1; §IV.F: "essential (pose) graph optimization to propagate
// the loop correction", Jacobians by "automatic differentiation"; Conclusion:
// "Levenberg-Marquardt"). Readings A49-A54.
//
// One persistent cooperative kernel runs the whole Levenberg-Marquardt loop: no host
// round trip per iteration or per linear-solver step. Phases are separated by a
// grid-wide barrier; every CTA reduces the same per-CTA partials in the same order,
// so all CTAs take identical control decisions (accept / reject / stop) and the
// result is deterministic for a given grid size.
//
//   linearise   16-lane group per edge: lane k < 14 evaluates the residual
//               e = log(M o S_i o S_j^-1) on a forward-mode dual number seeded with
//               tangent direction k of vertex i (k < 7) or j (k >= 7) (A50), i.e. one
//               Jacobian column per lane; the group forms J^T J and J^T e blocks in
//               shared memory and writes one 1.7-KB record per edge.
//   assemble    warp per vertex: diagonal block and gradient summed over the vertex's
//               incident edges in ascending edge order (the oracle's order).
//   solve       (H + lambda diag(H)) delta = -b by block-Jacobi preconditioned CG
//               (A54: the paper's LDLT is a CPU library solve; CG on the block-sparse
//               matrix is the data-parallel equivalent); 8-lane group per vertex.
//   trial       S_v' = exp(delta_v) o S_v, chi2' by thread per edge; accept iff it
//               decreases (A52/A53).
#include <cooperative_groups.h>

#include "lc_internal.cuh"

namespace {

constexpr int kT = 256;        // threads per CTA
constexpr int kRec = 212;      // doubles per edge record
// record layout: Hii [0,49) Hjj [49,98) Hij [98,147) Hji [147,196) bi [196,203) bj [203,210) chi2 [210]
constexpr int kOffHii = 0, kOffHjj = 49, kOffHij = 98, kOffHji = 147, kOffBi = 196, kOffBj = 203;
constexpr int kVD = 56;        // per-vertex diagonal block (49) + gradient (7)
constexpr int kVL = 28;        // per-vertex Cholesky factor of the damped diagonal block
constexpr int kVec = 8;        // padded 7-vectors
constexpr int kBWMax = 28;     // largest block bandwidth of the banded direct solve (435-block window)

// ---------------------------------------------------------------------------
// forward-mode dual number with one partial (A50): value and derivative along one seed
// ---------------------------------------------------------------------------
struct dd {
  double v, d;
};
__device__ __forceinline__ dd operator+(dd a, dd b) { return {a.v + b.v, a.d + b.d}; }
__device__ __forceinline__ dd operator-(dd a, dd b) { return {a.v - b.v, a.d - b.d}; }
__device__ __forceinline__ dd operator*(dd a, dd b) { return {a.v * b.v, a.d * b.v + a.v * b.d}; }
__device__ __forceinline__ dd operator/(dd a, dd b) { return {a.v / b.v, (a.d * b.v - a.v * b.d) / (b.v * b.v)}; }
__device__ __forceinline__ dd scl(dd a, double c) { return {a.v * c, a.d * c}; }
__device__ __forceinline__ dd addc(dd a, double c) { return {a.v + c, a.d}; }
__device__ __forceinline__ dd neg(dd a) { return {-a.v, -a.d}; }
__device__ __forceinline__ double val(dd a) { return a.v; }
__device__ __forceinline__ dd vsqrt(dd a) { const double s = sqrt(a.v); return {s, (0.5 / s) * a.d}; }
__device__ __forceinline__ dd vsin(dd a) { return {sin(a.v), cos(a.v) * a.d}; }
__device__ __forceinline__ dd vcos(dd a) { return {cos(a.v), -sin(a.v) * a.d}; }
__device__ __forceinline__ dd vexp(dd a) { const double e = exp(a.v); return {e, e * a.d}; }
__device__ __forceinline__ dd vexpm1(dd a) { return {expm1(a.v), exp(a.v) * a.d}; }
__device__ __forceinline__ dd vlog(dd a) { return {log(a.v), (1.0 / a.v) * a.d}; }
__device__ __forceinline__ dd vatan2(dd y, dd x) {
  const double den = x.v * x.v + y.v * y.v;
  return {atan2(y.v, x.v), (x.v * y.d - y.v * x.d) / den};
}
// plain doubles
__device__ __forceinline__ double scl(double a, double c) { return a * c; }
__device__ __forceinline__ double addc(double a, double c) { return a + c; }
__device__ __forceinline__ double neg(double a) { return -a; }
__device__ __forceinline__ double val(double a) { return a; }
__device__ __forceinline__ double vsqrt(double a) { return sqrt(a); }
__device__ __forceinline__ double vsin(double a) { return sin(a); }
__device__ __forceinline__ double vcos(double a) { return cos(a); }
__device__ __forceinline__ double vexp(double a) { return exp(a); }
__device__ __forceinline__ double vexpm1(double a) { return expm1(a); }
__device__ __forceinline__ double vlog(double a) { return log(a); }
__device__ __forceinline__ double vatan2(double y, double x) { return atan2(y, x); }
template <class T> __device__ __forceinline__ T zero();
template <> __device__ __forceinline__ double zero<double>() { return 0.0; }
template <> __device__ __forceinline__ dd zero<dd>() { return {0.0, 0.0}; }

template <class T>
__device__ __forceinline__ T dot3(const T* a, const T* b) {
  return (a[0] * b[0] + a[1] * b[1]) + a[2] * b[2];
}
template <class T>
__device__ __forceinline__ void cross3(const T* a, const T* b, T* o) {
  const T r0 = a[1] * b[2] - a[2] * b[1];
  const T r1 = a[2] * b[0] - a[0] * b[2];
  const T r2 = a[0] * b[1] - a[1] * b[0];
  o[0] = r0; o[1] = r1; o[2] = r2;
}

// A49: W(omega, sigma) = A I + B Omega + C Omega^2 coefficients (th2 = |omega|^2)
template <class T>
__device__ __forceinline__ void w_coef(T th2, T sg, T& A, T& B, T& C) {
  const bool ssmall = fabs(val(sg)) < 1e-3;
  if (ssmall) A = addc(sg * addc(sg * addc(scl(sg, 1.0 / 24.0), 1.0 / 6.0), 0.5), 1.0);
  else A = vexpm1(sg) / sg;
  if (val(th2) < 1e-8) {
    if (ssmall) {
      B = addc(sg * addc(sg * addc(scl(sg, 1.0 / 30.0), 1.0 / 8.0), 1.0 / 3.0), 0.5);
      C = addc(sg * addc(sg * addc(scl(sg, 1.0 / 72.0), 1.0 / 20.0), 1.0 / 8.0), 1.0 / 6.0);
    } else {
      const T es = vexp(sg), s2 = sg * sg;
      B = addc(addc(sg, -1.0) * es, 1.0) / s2;
      C = addc(addc(s2 - scl(sg, 2.0), 2.0) * es, -2.0) / scl(s2 * sg, 2.0);
    }
    return;
  }
  const T th = vsqrt(th2), sn = vsin(th), cs = vcos(th), h = vsin(scl(th, 0.5));
  const T es = vexp(sg), em = vexpm1(sg);
  const T h2 = scl(h * h, 2.0);
  const T den = sg * sg + th2;
  const T nb = (es * sg) * sn + th * (h2 - em * cs);
  B = nb / (th * den);
  const T nc = (em * cs - h2) * sg + (es * sn) * th;
  C = (A - nc / den) / th2;
}

// A49: Sim3 log -> x = (omega, upsilon, sigma); R row-major, p' = s R p + t
template <class T>
__device__ __forceinline__ void sim3_log(const T* R, const T* t, T s, T* x) {
  const T v[3] = {R[7] - R[5], R[2] - R[6], R[3] - R[1]};
  const T c = scl(addc((R[0] + R[4]) + R[8], -1.0), 0.5);
  const T n2 = dot3(v, v);
  T w[3];
  if (val(n2) < 4e-8 && val(c) > 0.0) {
    const T f = addc(scl(n2, 1.0 / 48.0), 0.5);
#pragma unroll
    for (int i = 0; i < 3; ++i) w[i] = f * v[i];
  } else {
    const T nv = vsqrt(n2);
    const T th = vatan2(scl(nv, 0.5), c);
    const T f = th / nv;
#pragma unroll
    for (int i = 0; i < 3; ++i) w[i] = f * v[i];
  }
  const T sg = vlog(s);
  const T th2 = dot3(w, w);
  T A, B, C;
  w_coef(th2, sg, A, B, C);
  const T z = zero<T>();
  const T O[9] = {z, neg(w[2]), w[1], w[2], z, neg(w[0]), neg(w[1]), w[0], z};
  T W[9];
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j) {
      T o2 = w[i] * w[j];
      if (i == j) o2 = o2 - th2;
      T e = B * O[3 * i + j] + C * o2;
      if (i == j) e = e + A;
      W[3 * i + j] = e;
    }
  const T det = (W[0] * (W[4] * W[8] - W[5] * W[7]) - W[1] * (W[3] * W[8] - W[5] * W[6])) +
                W[2] * (W[3] * W[7] - W[4] * W[6]);
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    T Wk[9];
#pragma unroll
    for (int i = 0; i < 9; ++i) Wk[i] = W[i];
#pragma unroll
    for (int i = 0; i < 3; ++i) Wk[3 * i + k] = t[i];
    const T dk = (Wk[0] * (Wk[4] * Wk[8] - Wk[5] * Wk[7]) - Wk[1] * (Wk[3] * Wk[8] - Wk[5] * Wk[6])) +
                 Wk[2] * (Wk[3] * Wk[7] - Wk[4] * Wk[6]);
    x[3 + k] = dk / det;
  }
  x[0] = w[0]; x[1] = w[1]; x[2] = w[2];
  x[6] = sg;
}

// A49: Sim3 exp of x (plain doubles; the trial update S' = exp(delta) o S)
__device__ __forceinline__ void sim3_exp(const double* x, double* S) {
  const double* w = x;
  const double* u = x + 3;
  const double th2 = dot3(w, w);
  double a, b;
  if (th2 < 1e-8) {
    a = th2 * (-1.0 / 6.0) + 1.0;
    b = th2 * (-1.0 / 24.0) + 0.5;
  } else {
    const double th = sqrt(th2), hh = sin(th * 0.5);
    a = sin(th) / th;
    b = ((hh * hh) * 2.0) / th2;
  }
  const double O[9] = {0.0, -w[2], w[1], w[2], 0.0, -w[0], -w[1], w[0], 0.0};
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j) {
      double o2 = w[i] * w[j];
      if (i == j) o2 = o2 - th2;
      double e = a * O[3 * i + j] + b * o2;
      if (i == j) e = e + 1.0;
      S[3 * i + j] = e;
    }
  double A, B, C, wu[3], wwu[3];
  w_coef(th2, x[6], A, B, C);
  cross3(w, u, wu);
  cross3(w, wu, wwu);
#pragma unroll
  for (int i = 0; i < 3; ++i) S[9 + i] = (A * u[i] + B * wu[i]) + C * wwu[i];
  S[12] = exp(x[6]);
}

// residual value of edge (M, S_i, S_j): e = log((M o S_i) o S_j^-1)
__device__ __forceinline__ void edge_value(const double* M, const double* Si, const double* Sj, double* Q,
                                           double* e) {
  double T1[13], Sji[13];
  lc_sim3_compose(M, Si, T1);
  lc_sim3_inverse(Sj, Sji);
  lc_sim3_compose(T1, Sji, Q);
  sim3_log<double>(Q, Q + 9, Q[12], e);
}

struct PgoArgs {
  int n_v, n_e, max_iter, cg_max;
  double lambda0, eps_dx, eps_chi2, cg_tol;
  const int32_t* eij;      // [n_e][2]
  const double* M;         // [n_e][13]
  const double* S_in;      // [n_v][13]
  const uint8_t* fixed;    // [n_v]
  const int32_t* vbeg;     // [n_v+1] incidence CSR
  const int2* vinc2;       // [2 n_e] ((edge << 1) | role (0: vertex is i, 1: j), other vertex), ascending edge
  double* S_out;           // [n_v][13] estimate (buffer 0)
  double* S_tmp;           // [n_v][13] (buffer 1)
  double* rec;             // [n_e][kRec]
  double* vd;              // [n_v][kVD]
  double* vl;              // [n_v][kVL]
  double* vx;              // 6 vectors [n_v][kVec]: x, r, u, w, p, s
  double* part;            // [gridDim][4] per-CTA partial sums
  // banded direct solve (A54): bw >= 0 selects it; pos/ord the host's reverse Cuthill-McKee
  // ordering (free vertices first), bw its block bandwidth
  int bw;
  const int32_t* pos;      // [n_v] vertex -> position
  const int32_t* ord;      // [n_v] position -> vertex
  double* band;            // [n_v][bw+1][49] assembled H in band storage: (p + d, p) blocks
  double* lband;           // [n_v][bw+1][49] Cholesky factor, same layout
  double* yb;              // [n_v][8] forward-substitution result
  double* bres;            // [8] fail flag, |delta|^2 (banded); [2 + parity] cyclic-reduction fail flags
  // block cyclic reduction (A54b): cr_s > 0 selects it; super-blocks of cr_s positions
  int cr_s, cr_N, cr_levels;
  double* crA;             // [cr_N][D][D] damped diagonal super-blocks, then their Cholesky factors
  double* crC;             // [cr_N][D][D] coupling with the current left neighbour, then X_l
  double* crX;             // [cr_N][D][D] X_r of an eliminated super-block
  double* cry;             // [cr_N][D] right-hand side, then L^-1 (rhs)
  double* crx;             // [cr_N][D] solution
  long long* ctim;         // LC_PGO_TIMING: [8] elimination sub-phase cycles (CTA 0)
  unsigned int* bar;       // grid barrier counter (zeroed before launch)
  double* trace;           // [max_iter][6] or null
  double* chi2_out;        // [2] or null
  unsigned long long* counts;
};

// grid-wide barrier (all CTAs co-resident: cooperative launch); monotone counter
__device__ __forceinline__ void grid_barrier(unsigned int* bar, unsigned int& target) {
  __syncthreads();
  target += gridDim.x;
  if (threadIdx.x == 0) {
    __threadfence();
    atomicAdd(bar, 1u);
    unsigned int v;
    for (;;) {
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(bar) : "memory");
      if ((int)(v - target) >= 0) break;
      __nanosleep(32);
    }
    __threadfence();
  }
  __syncthreads();
}

// deterministic CTA reduction of 4 partials -> part[blockIdx]; then every CTA sums the
// gridDim partials in the same fixed order (after the barrier)
__device__ __forceinline__ void cta_partial(double a0, double a1, double a2, double a3, double* part,
                                            double (*sh)[4]) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  double a[4] = {a0, a1, a2, a3};
#pragma unroll
  for (int k = 0; k < 4; ++k)
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) a[k] += __shfl_xor_sync(0xffffffffu, a[k], o);
  if (lane == 0)
#pragma unroll
    for (int k = 0; k < 4; ++k) sh[wid][k] = a[k];
  __syncthreads();
  if (threadIdx.x < 4) {
    double s = 0.0;
    for (int w = 0; w < kT / 32; ++w) s += sh[w][threadIdx.x];
    part[4 * blockIdx.x + threadIdx.x] = s;
  }
  __syncthreads();
}

__device__ __forceinline__ void grid_total(const double* part, double* out4, double (*sh)[4]) {
  if (threadIdx.x < 32) {
    double a[4] = {0.0, 0.0, 0.0, 0.0};
    for (int b = threadIdx.x; b < (int)gridDim.x; b += 32)
#pragma unroll
      for (int k = 0; k < 4; ++k) a[k] += __ldcg(part + 4 * b + k);
#pragma unroll
    for (int k = 0; k < 4; ++k)
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) a[k] += __shfl_xor_sync(0xffffffffu, a[k], o);
    if (threadIdx.x == 0)
#pragma unroll
      for (int k = 0; k < 4; ++k) sh[0][k] = a[k];
  }
  __syncthreads();
#pragma unroll
  for (int k = 0; k < 4; ++k) out4[k] = sh[0][k];
  __syncthreads();
}

// chi2 partial of this thread: thread per edge, value-only residuals at estimate S
__device__ __forceinline__ double chi2_part(const PgoArgs& a, const double* S) {
  double acc = 0.0;
  for (int e = blockIdx.x * kT + threadIdx.x; e < a.n_e; e += gridDim.x * kT) {
    const int i = a.eij[2 * e], j = a.eij[2 * e + 1];
    double M[13], Si[13], Sj[13], Q[13], r[7];
#pragma unroll
    for (int k = 0; k < 13; ++k) {
      M[k] = a.M[13 * (size_t)e + k];
      Si[k] = __ldcg(S + 13 * (size_t)i + k);
      Sj[k] = __ldcg(S + 13 * (size_t)j + k);
    }
    edge_value(M, Si, Sj, Q, r);
    double c = 0.0;
#pragma unroll
    for (int k = 0; k < 7; ++k) c += r[k] * r[k];
    acc += c;
  }
  return acc;
}

// hat(g) for the 3-vector g
__device__ __forceinline__ void hat3(const double* g, double* H) {
  H[0] = 0.0; H[1] = -g[2]; H[2] = g[1];
  H[3] = g[2]; H[4] = 0.0; H[5] = -g[0];
  H[6] = -g[1]; H[7] = g[0]; H[8] = 0.0;
}
__device__ __forceinline__ void mat3(const double* A, const double* B, double* o) {
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j) o[3 * i + j] = (A[3 * i] * B[j] + A[3 * i + 1] * B[3 + j]) + A[3 * i + 2] * B[6 + j];
}

// linearise: 16-lane group per edge -> record
__device__ void linearise(const PgoArgs& a, const double* S, double* shJ) {
  const int lane16 = threadIdx.x & 15;
  const int grp = (blockIdx.x * kT + threadIdx.x) >> 4, ngrp = (gridDim.x * kT) >> 4;
  double* J = shJ + (threadIdx.x >> 4) * 112;   // [14][7] columns + e[7]
  const unsigned mask = 0xffffu << (threadIdx.x & 16);
  for (int e = grp; e < a.n_e; e += ngrp) {
    const int i = a.eij[2 * e], j = a.eij[2 * e + 1];
    double M[13], Si[13], Sj[13], Q[13], P[13], Sji[13], T1[13];
#pragma unroll
    for (int k = 0; k < 13; ++k) {
      M[k] = a.M[13 * (size_t)e + k];
      Si[k] = __ldcg(S + 13 * (size_t)i + k);
      Sj[k] = __ldcg(S + 13 * (size_t)j + k);
    }
    lc_sim3_compose(M, Si, T1);
    lc_sim3_inverse(Sj, Sji);
    lc_sim3_compose(T1, Sji, Q);
    if (lane16 < 14) {
      const int k = lane16 < 7 ? lane16 : lane16 - 7;
      const bool fixed_v = a.fixed[lane16 < 7 ? i : j] != 0;
      double g[7] = {0, 0, 0, 0, 0, 0, 0};
      g[k] = 1.0;
      double Hg[9], dR[9], dt[3], ds;
      hat3(g, Hg);
      if (lane16 < 7) {
        // d/d delta_i of M o exp(delta) o P, P = S_i o S_j^-1
        lc_sim3_compose(Si, Sji, P);
        double tmp[9];
        mat3(M, Hg, tmp);
        mat3(tmp, P, dR);
        double u[3];
#pragma unroll
        for (int r = 0; r < 3; ++r) u[r] = ((g[6] * P[9 + r] + lc_row3(Hg + 3 * r, P + 9)) + g[3 + r]);
#pragma unroll
        for (int r = 0; r < 3; ++r) dt[r] = M[12] * lc_row3(M + 3 * r, u);
        ds = (M[12] * g[6]) * P[12];
      } else {
        // d/d delta_j of Q o exp(-delta)
#pragma unroll
        for (int r = 0; r < 9; ++r) dR[r] = 0.0;
        double tmp[9];
        mat3(Q, Hg, tmp);
#pragma unroll
        for (int r = 0; r < 9; ++r) dR[r] = -tmp[r];
#pragma unroll
        for (int r = 0; r < 3; ++r) dt[r] = -(Q[12] * lc_row3(Q + 3 * r, g + 3));
        ds = -(Q[12] * g[6]);
      }
      dd R[9], t[3], x[7];
#pragma unroll
      for (int r = 0; r < 9; ++r) R[r] = {Q[r], dR[r]};
#pragma unroll
      for (int r = 0; r < 3; ++r) t[r] = {Q[9 + r], dt[r]};
      sim3_log<dd>(R, t, dd{Q[12], ds}, x);
#pragma unroll
      for (int r = 0; r < 7; ++r) J[7 * lane16 + r] = fixed_v ? 0.0 : x[r].d;
      if (lane16 == 0)
#pragma unroll
        for (int r = 0; r < 7; ++r) J[98 + r] = x[r].v;
    }
    __syncwarp(mask);
    double* R = a.rec + (size_t)e * kRec;
    for (int o = lane16; o < 211; o += 16) {
      double v = 0.0;
      if (o < 196) {
        const int blk = o / 49, ab = o - 49 * blk, r = ab / 7, c = ab - 7 * r;
        // Hii: (i, i); Hjj: (j, j); Hij: (i row, j col); Hji: (j row, i col)
        const int cr = (blk == 0 || blk == 2) ? r : 7 + r;
        const int cc = (blk == 0 || blk == 3) ? c : 7 + c;
#pragma unroll
        for (int q = 0; q < 7; ++q) v += J[7 * cr + q] * J[7 * cc + q];
      } else if (o < 210) {
        const int col = o - 196;   // 0..6 vertex i, 7..13 vertex j
#pragma unroll
        for (int q = 0; q < 7; ++q) v += J[7 * col + q] * J[98 + q];
      } else {
#pragma unroll
        for (int q = 0; q < 7; ++q) v += J[98 + q] * J[98 + q];
      }
      R[o] = v;
    }
    __syncwarp(mask);
  }
}

__device__ __forceinline__ double vget(const double* base, int v, int r) {
  return __ldcg(base + (size_t)v * kVec + r);
}

// z = (L L^T)^-1 r for vertex v, every lane of the group computes all 7 and keeps its own
__device__ __forceinline__ double precond(const double* L, const double* rv, int lane) {
  double y[7];
#pragma unroll
  for (int i = 0; i < 7; ++i) {
    double s = rv[i];
#pragma unroll
    for (int k = 0; k < i; ++k) s -= L[i * (i + 1) / 2 + k] * y[k];
    y[i] = s / L[i * (i + 1) / 2 + i];
  }
#pragma unroll
  for (int i = 6; i >= 0; --i) {
    double s = y[i];
#pragma unroll
    for (int k = i + 1; k < 7; ++k) s -= L[k * (k + 1) / 2 + i] * y[k];
    y[i] = s / L[i * (i + 1) / 2 + i];
  }
  double out = 0.0;
#pragma unroll
  for (int i = 0; i < 7; ++i) out = (lane == i) ? y[i] : out;
  return out;
}

// row lane8 of (H + lambda diag H) y at vertex v: diagonal block, then the off-diagonal
// blocks of the incident edges in ascending edge order (incidences loaded 4 at a time so
// their block-row and neighbour loads are in flight together)
__device__ __forceinline__ double spmv_row(const PgoArgs& a, int v, int lane8, const double* y, double lambda) {
  const double* D = a.vd + (size_t)v * kVD + 7 * lane8;
  double s = 0.0;
#pragma unroll
  for (int c = 0; c < 7; ++c) s += __ldcg(D + c) * vget(y, v, c);
  s += lambda * __ldcg(D + lane8) * vget(y, v, lane8);
  if (a.fixed[v]) return s;
  const int b0 = a.vbeg[v], b1 = a.vbeg[v + 1];
  for (int q0 = b0; q0 < b1; q0 += 4) {
    int2 w[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) w[u] = q0 + u < b1 ? __ldcg(a.vinc2 + q0 + u) : make_int2(-1, 0);
    double t[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      t[u] = 0.0;
      if (w[u].x >= 0) {
        const double* B = a.rec + (size_t)(w[u].x >> 1) * kRec + ((w[u].x & 1) ? kOffHji : kOffHij) + 7 * lane8;
#pragma unroll
        for (int c = 0; c < 7; ++c) t[u] += __ldcg(B + c) * vget(y, w[u].y, c);
      }
    }
#pragma unroll
    for (int u = 0; u < 4; ++u)
      if (w[u].x >= 0) s += t[u];
  }
  return s;
}

// ---------------------------------------------------------------------------
// banded direct solve (A54). Positions p = pos[v] come from a reverse Cuthill-McKee
// ordering with block bandwidth bw, so the damped matrix is block-banded: block (p+d, p)
// nonzero only for d <= bw. band[p][d] holds it (d = 0: the vertex's diagonal block).
// ---------------------------------------------------------------------------
__device__ void band_assemble(const PgoArgs& a) {
  const int NB = a.bw + 1;
  const int lane = threadIdx.x & 31;
  const int warp = (blockIdx.x * kT + threadIdx.x) >> 5, nwarp = (gridDim.x * kT) >> 5;
  for (int p = warp; p < a.n_v; p += nwarp) {
    const int v = a.ord[p];
    double* Ab = a.band + (size_t)p * NB * 49;
    for (int o = lane; o < NB * 49; o += 32) Ab[o] = o < 49 ? __ldcg(a.vd + (size_t)v * kVD + o) : 0.0;
    __syncwarp();
    if (a.fixed[v]) continue;
    const int b0 = a.vbeg[v], b1 = a.vbeg[v + 1];
    for (int q = b0; q < b1; ++q) {
      const int2 w = __ldg(a.vinc2 + q);
      if (a.fixed[w.y]) continue;
      const int d = a.pos[w.y] - p;
      if (d < 1) continue;
      // block (rows other, cols v): Hji when v is i (role 0), Hij when v is j
      const double* B = a.rec + (size_t)(w.x >> 1) * kRec + ((w.x & 1) ? kOffHij : kOffHji);
      for (int o = lane; o < 49; o += 32) Ab[d * 49 + o] += __ldcg(B + o);
      __syncwarp();
    }
  }
}

// CTA-wide: Cholesky of the damped band matrix, forward substitution fused; then back
// substitution. The active window -- positions j..j+bw, lower-triangular blocks -- lives
// in shared memory; a block (r, c), r >= c, sits at the unordered slot pair
// (r mod NB, c mod NB), so the window needs NB (NB + 1) / 2 blocks and the position
// that retires at step j frees exactly the slots the entering position j + NB takes.
// x -> X (vertex order); writes bres = (fail, |x|^2).
__device__ __forceinline__ int tri_slot(int a, int b) {
  const int hi = a > b ? a : b, lo = a > b ? b : a;
  return hi * (hi + 1) / 2 + lo;
}
__device__ __forceinline__ int wslot(int r, int c, int NB) { return tri_slot(r % NB, c % NB); }

#ifdef LC_PGO_TIMING
#define PGO_TIC(k) do { if (t == 0) { const long long c_ = clock64(); tim[k] += c_ - tlast; tlast = c_; } } while (0)
#else
#define PGO_TIC(k) do { } while (0)
#endif

__device__ void band_solve(const PgoArgs& a, double lambda, double* sm, double* X) {
  const int n = a.n_v, BW = a.bw, NB = BW + 1, t = threadIdx.x;
  const int nw = NB * (NB + 1) / 2;
  double* Wn = sm;                        // [nw][49] window blocks
  double* Yw = Wn + (size_t)nw * 49;      // [NB][8]
  double* Xs = Yw + NB * 8;               // [NB][8] back-substitution window
  double* Lc = Xs + NB * 8;               // [NB][49] one factor column (back substitution)
  double* part = Lc + NB * 49;            // [NB + 2][8]
  unsigned short* pairs = (unsigned short*)(part + NB * 8 + 16);   // [BW (BW + 1) / 2] (d1, d2)
  __shared__ int s_fail;
#ifdef LC_PGO_TIMING
  long long tim[8] = {0, 0, 0, 0, 0, 0, 0, 0}, tlast = clock64();
#endif
  if (t == 0) {
    s_fail = 0;
    int k = 0;
    for (int d1 = 1; d1 <= BW; ++d1)
      for (int d2 = d1; d2 <= BW; ++d2) pairs[k++] = (unsigned short)(d1 | (d2 << 8));
  }
  // block (r, c) of the damped matrix, entry e (0 if outside the matrix)
  auto blk_val = [&](int r, int c, int e) -> double {
    if (r >= n) return 0.0;
    double v = __ldcg(a.band + ((size_t)c * NB + (r - c)) * 49 + e);
    if (r == c && (e / 7) == (e % 7)) v = v + lambda * v;
    return v;
  };
  auto grad_val = [&](int q, int r) -> double {   // b (the right-hand side is -b)
    return q < n ? __ldcg(a.vd + (size_t)a.ord[q] * kVD + 49 + r) : 0.0;
  };
  for (int idx = t; idx < nw * 49; idx += kT) {
    const int blk = idx / 49, e = idx - 49 * blk;
    int r = 0;
    while ((r + 1) * (r + 2) / 2 <= blk) ++r;
    const int c = blk - r * (r + 1) / 2;    // initial window: positions 0..BW, slot = position
    Wn[(size_t)blk * 49 + e] = r < NB ? blk_val(r, c, e) : 0.0;
  }
  if (t < NB * 8) Yw[t] = (t % 8) < 7 ? -grad_val(t / 8, t % 8) : 0.0;
  __syncthreads();
  const int per = (NB * 49 + kT - 1) / kT;
  double pf[8];   // prefetched blocks of the entering position
  // Diagonal-block Cholesky by one thread with the block in registers (shuffle latency
  // made a warp-parallel version slower), then y_jd = L^-1 y_jd. The pivots'
  // reciprocals go to the unused upper triangle: invd[0] -> (1, 2), invd[k] -> (0, k).
  // Look-ahead: block (j+1, j+1) only needs pair (1, 1) of the update of step j, so the
  // last warp applies that pair with all its lanes and factors the block while the other
  // warps apply the remaining pairs (the Cholesky leaves the critical path).
  auto chol_diag = [&](int jd) {   // one thread
    double* A0 = Wn + (size_t)wslot(jd, jd, NB) * 49;
    {
      double L[28], inv[7];
#pragma unroll
      for (int i = 0; i < 7; ++i)
#pragma unroll
        for (int k = 0; k <= i; ++k) L[i * (i + 1) / 2 + k] = A0[7 * i + k];
      bool okc = true;
#pragma unroll
      for (int k = 0; k < 7; ++k) {
        const double akk = L[k * (k + 1) / 2 + k];
        if (!(akk > 0.0)) { okc = false; break; }
        inv[k] = rsqrt(akk);
        L[k * (k + 1) / 2 + k] = akk * inv[k];
#pragma unroll
        for (int i = k + 1; i < 7; ++i) L[i * (i + 1) / 2 + k] *= inv[k];
#pragma unroll
        for (int i = k + 1; i < 7; ++i)
#pragma unroll
          for (int jj = k + 1; jj <= i; ++jj) L[i * (i + 1) / 2 + jj] -= L[i * (i + 1) / 2 + k] * L[jj * (jj + 1) / 2 + k];
      }
      if (!okc) {
        s_fail = 1;
      } else {
#pragma unroll
        for (int i = 0; i < 7; ++i)
#pragma unroll
          for (int k = 0; k <= i; ++k) A0[7 * i + k] = L[i * (i + 1) / 2 + k];
        A0[9] = inv[0];
#pragma unroll
        for (int k = 1; k < 7; ++k) A0[k] = inv[k];
        double* yv = Yw + (jd % NB) * 8;
        double y[7];
#pragma unroll
        for (int r = 0; r < 7; ++r) {
          double sacc = yv[r];
#pragma unroll
          for (int m = 0; m < r; ++m) sacc -= L[r * (r + 1) / 2 + m] * y[m];
          y[r] = sacc * inv[r];
        }
#pragma unroll
        for (int r = 0; r < 7; ++r) yv[r] = y[r];
      }
    }
  };
  if (t == 0 && n > 0) chol_diag(0);
  __syncthreads();
  int ordq = (t >= kT - 32 && t < kT - 25 && NB < n) ? __ldg(a.ord + NB) : 0;
  for (int j = 0; j < n; ++j) {
    const int q = j + NB;
    // the entering gradient: a dependent load pair (ord, then vd), issued by the last warp,
    // which has no work in steps (1)-(2) and little in (3), so the Cholesky warp never waits on it
    const int tr = t - (kT - 32);
    // (ord[q] was loaded one step earlier, so the gradient load does not wait on it)
    const double pfr = (tr >= 0 && tr < 7 && q < n) ? __ldcg(a.vd + (size_t)ordq * kVD + 49 + tr) : 0.0;
    ordq = (tr >= 0 && tr < 7 && q + 1 < n) ? __ldg(a.ord + q + 1) : 0;
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int idx = t + u * kT;
      pf[u] = 0.0;
      if (u < per && idx < NB * 49) {
        const int c = q - BW + idx / 49;   // blocks (q, c), c = j+1 .. q (damping added at store)
        if (q < n) pf[u] = __ldcg(a.band + ((size_t)c * NB + (q - c)) * 49 + idx % 49);
      }
    }
    double* A0 = Wn + (size_t)wslot(j, j, NB) * 49;
    // (1) the diagonal block was factored by the look-ahead of the previous step (with
    //     bw = 0 position j enters the window only at the end of step j - 1: factor here)
    if (BW == 0 && t == 0 && j > 0) chol_diag(j);
    __syncthreads();
    PGO_TIC(0);
    if (s_fail) break;
    // (2) panel: L_{j+d, j} = A_{j+d, j} L_jj^-T (thread per scalar row); y_{j+d} -= L y_j
    if (t < 7 * BW) {
      const int d = 1 + t / 7, r = t % 7;
      if (j + d < n) {
        double* Ar = Wn + (size_t)wslot(j + d, j, NB) * 49 + 7 * r;
        double x[7];
#pragma unroll
        for (int k = 0; k < 7; ++k) {
          double s = Ar[k];
#pragma unroll
          for (int m = 0; m < k; ++m) s -= x[m] * A0[7 * k + m];
          x[k] = s * A0[k == 0 ? 9 : k];
        }
        const double* yj = Yw + (j % NB) * 8;
        double acc = 0.0;
#pragma unroll
        for (int k = 0; k < 7; ++k) { Ar[k] = x[k]; acc += x[k] * yj[k]; }
        Yw[((j + d) % NB) * 8 + r] -= acc;
      }
    }
    __syncthreads();
    PGO_TIC(1);
    // (3) trailing update of the window: block (j+d2, j+d1) -= L_{j+d2, j} L_{j+d1, j}^T,
    //     thread per block pair (L_{j+d1, j} held in registers: 98 shared loads per 343
    //     FMAs; a thread per (pair, row) re-reads L_{j+d1, j} 7 times and measured slower).
    //     Pair (1, 1) belongs to the look-ahead warp.
    {
      const int nblk = BW * (BW + 1) / 2, jm = j % NB;
      if (t >= kT - 32) {
        const int lane = t - (kT - 32);
        if (BW > 0 && j + 1 < n) {
          int s1 = jm + 1;
          if (s1 >= NB) s1 -= NB;
          const double* L1 = Wn + (size_t)tri_slot(s1, jm) * 49;
          double* T = Wn + (size_t)tri_slot(s1, s1) * 49;
          for (int e = lane; e < 49; e += 32) {
            const int r = e / 7, c = e - 7 * r;
            double acc = 0.0;
#pragma unroll
            for (int m = 0; m < 7; ++m) acc += L1[7 * r + m] * L1[7 * c + m];
            T[e] -= acc;
          }
          __syncwarp();
          if (lane == 0) chol_diag(j + 1);
        }
      } else {
        for (int b = 1 + t; b < nblk; b += kT - 32) {
          const int pr = pairs[b], d1 = pr & 0xff, d2 = pr >> 8;
          if (j + d2 >= n) continue;
          int s2 = jm + d2, s1 = jm + d1;
          if (s2 >= NB) s2 -= NB;
          if (s1 >= NB) s1 -= NB;
          const double* L2 = Wn + (size_t)tri_slot(s2, jm) * 49;
          const double* L1 = Wn + (size_t)tri_slot(s1, jm) * 49;
          double* T = Wn + (size_t)tri_slot(s2, s1) * 49;
          double l1[49];
#pragma unroll
          for (int k = 0; k < 49; ++k) l1[k] = L1[k];
#pragma unroll
          for (int r = 0; r < 7; ++r) {
            double l2[7];
#pragma unroll
            for (int m = 0; m < 7; ++m) l2[m] = L2[7 * r + m];
#pragma unroll
            for (int c = 0; c < 7; ++c) {
              double acc = 0.0;
#pragma unroll
              for (int m = 0; m < 7; ++m) acc += l2[m] * l1[7 * c + m];
              T[7 * r + c] -= acc;
            }
          }
        }
      }
    }
    __syncthreads();
    PGO_TIC(2);
    // (4) retire position j (factor column + y_j to global) and let position j + NB enter:
    //     the entering block (q, j+1+d') takes the slot of the retiring block (j+d'+1, j)
    //     (d' = bw: the diagonal (q, q) takes (j, j)), so each thread moves its own entries
    {
      const int jm = j % NB;
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int idx = t + u * kT;
        if (u < per && idx < NB * 49) {
          const int dp = idx / 49, e = idx - 49 * dp;
          const int d = dp == BW ? 0 : dp + 1;       // retiring block (j + d, j)
          int sc = jm + 1 + dp;
          if (sc >= NB) sc -= NB;
          double* slot = Wn + (size_t)tri_slot(jm, sc) * 49 + e;
          a.lband[(size_t)j * NB * 49 + d * 49 + e] = (j + d < n) ? *slot : 0.0;
          double v = pf[u];
          if (dp == BW && (e / 7) == (e % 7)) v = v + lambda * v;
          *slot = v;
        }
      }
      if (tr >= 0 && tr < 8) {
        a.yb[(size_t)j * 8 + tr] = Yw[jm * 8 + tr];
        Yw[jm * 8 + tr] = tr < 7 ? -pfr : 0.0;
      }
    }
    __syncthreads();
    PGO_TIC(4);
  }
  double xx = 0.0;
  if (!s_fail) {
    // back substitution: x_j = L_jj^-T (y_j - sum_d L_{j+d,j}^T x_{j+d}), two barriers per
    // position. Warps 0-6 = rows r of the 7-vector, lane d-1 = block d: each thread holds
    // the 7 factor entries L_{j+d,j}[m][r] it needs (prefetched one position ahead), the
    // warp's butterfly sums over d; the last warp holds the diagonal block (2 entries per
    // lane), y_j and the vertex index, and its lane 0 solves the 7x7 triangle.
    const int r = t >> 5, dl = t & 31, d = dl + 1;
    const bool part_thr = t < kT - 32 && d <= BW;
    const int lw = t - (kT - 32);   // lane in the last warp, < 0 elsewhere
    const size_t col = (size_t)NB * 49;
    double pf[7], pd0 = 0.0, pd1 = 0.0, pfy = 0.0;
    int vnext = 0;
    auto prefetch = [&](int jj) {
      if (part_thr) {
#pragma unroll
        for (int m = 0; m < 7; ++m) pf[m] = __ldcg(a.lband + jj * col + d * 49 + 7 * m + r);
      }
      if (lw >= 0) {
        pd0 = __ldcg(a.lband + jj * col + lw);
        pd1 = lw + 32 < 49 ? __ldcg(a.lband + jj * col + lw + 32) : 0.0;
        pfy = lw < 7 ? __ldcg(a.yb + (size_t)jj * 8 + lw) : 0.0;
        if (lw == 0) vnext = a.ord[jj];
      }
    };
    prefetch(n - 1);
    double* Dg = Lc;          // diagonal block of the current position
    double* ssum = part;      // [8] sum over d
    double* sy = part + 8;    // [8] y_j
    for (int j = n - 1; j >= 0; --j) {
      double cur[7];
#pragma unroll
      for (int m = 0; m < 7; ++m) cur[m] = pf[m];
      const double c0 = pd0, c1 = pd1, cy = pfy;
      const int vcur = vnext;
      if (j > 0) prefetch(j - 1);
      if (t < kT - 32) {
        double sacc = 0.0;
        if (part_thr && j + d < n) {
          const double* xd = Xs + ((j + d) % NB) * 8;
#pragma unroll
          for (int m = 0; m < 7; ++m) sacc += cur[m] * xd[m];
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) sacc += __shfl_xor_sync(0xffffffffu, sacc, o);
        if (dl == 0) ssum[r] = sacc;
      } else {
        Dg[lw] = c0;
        if (lw + 32 < 49) Dg[lw + 32] = c1;
        if (lw < 7) sy[lw] = cy;
      }
      __syncthreads();
      if (lw == 0) {
        double x[7];
#pragma unroll
        for (int q = 0; q < 7; ++q) x[q] = sy[q] - ssum[q];
#pragma unroll
        for (int q = 6; q >= 0; --q) {
          double sacc = x[q];
#pragma unroll
          for (int m = q + 1; m < 7; ++m) sacc -= Dg[7 * m + q] * x[m];
          x[q] = sacc * Dg[q == 0 ? 9 : q];
        }
#pragma unroll
        for (int q = 0; q < 7; ++q) {
          Xs[(j % NB) * 8 + q] = x[q];
          X[(size_t)vcur * kVec + q] = x[q];
          xx += x[q] * x[q];
        }
      }
      __syncthreads();
    }
  }
  PGO_TIC(5);
  if (t == kT - 32) {   // the back substitution's solving thread holds |x|^2
    a.bres[0] = s_fail ? 1.0 : 0.0;
    a.bres[1] = xx;
  }
#ifdef LC_PGO_TIMING
  if (t == 0) {
    for (int k = 0; k < 6; ++k) a.counts[k] += (unsigned long long)tim[k];
    a.counts[6] += n;
  }
#endif
}

// ---------------------------------------------------------------------------
// Block cyclic reduction (A54b). The damped band matrix (block bandwidth bw, RCM order)
// is cut into N super-blocks of s = max(bw, 1) consecutive positions (D = 7 s unknowns;
// positions past n_v are identity padding). Super-blocks I and I + 2 share no nonzero,
// so the matrix is block tridiagonal and odd-even elimination applies: at stride st the
// super-blocks i = st (2k + 1) are eliminated, each independently (one CTA: dense
// Cholesky of A_i in shared memory, X_l = L_i^-1 A_il, X_r = L_i^-1 A_ir, y_i = L_i^-1 b_i),
// then every survivor J = 2 st k takes its Schur update (one CTA: A_J -= X^T X from both
// eliminated neighbours, the new left coupling -X_r^T X_l, b_J -= X^T y). log2 N levels
// replace the n_v-step chain of the banded factorisation and spread over the SMs; the back
// substitution x_i = L_i^-T (y_i - X_l x_l - X_r x_r) runs the levels in reverse. This is
// the Cholesky factorisation of the same matrix in the odd-even order of its super-blocks
// (no pivoting; a non-positive pivot fails the solve, as in the banded path).
// ---------------------------------------------------------------------------
constexpr int kCrPC = 64;      // column panel of the triangular solves and products
constexpr int kCrSMax = 18;    // largest super-block (positions): D <= 126

// entry (r, c) of block (P1, P2) of the damped matrix; positions >= n_v are identity padding
__device__ __forceinline__ double cr_entry(const PgoArgs& a, double lambda, int P1, int P2, int r, int c) {
  if (P1 >= a.n_v || P2 >= a.n_v) return (P1 == P2 && r == c) ? 1.0 : 0.0;
  if (P1 < P2) {
    const int tp = P1; P1 = P2; P2 = tp;
    const int tr = r; r = c; c = tr;
  }
  const int d = P1 - P2;
  if (d > a.bw) return 0.0;
  double v = __ldcg(a.band + ((size_t)P2 * (a.bw + 1) + d) * 49 + 7 * r + c);
  if (d == 0 && r == c) v = v + lambda * v;
  return v;
}

// grid-wide: dense super-blocks and right-hand side from band storage (warp per row)
__device__ void cr_assemble(const PgoArgs& a, double lambda) {
  const int s = a.cr_s, N = a.cr_N, D = 7 * s;
  const int lane = threadIdx.x & 31;
  const int warp = (blockIdx.x * kT + threadIdx.x) >> 5, nwarp = (gridDim.x * kT) >> 5;
  for (int task = warp; task < N * D; task += nwarp) {
    const int I = task / D, ra = task - I * D;
    const int P1 = I * s + ra / 7, r = ra % 7;
    double* Ar = a.crA + ((size_t)I * D + ra) * D;
    double* Cr = a.crC + ((size_t)I * D + ra) * D;
    for (int cb = lane; cb < D; cb += 32) {
      const int P2 = I * s + cb / 7, c = cb % 7;
      Ar[cb] = cr_entry(a, lambda, P1, P2, r, c);
      Cr[cb] = I > 0 ? cr_entry(a, lambda, P1, P2 - s, r, c) : 0.0;
    }
    if (lane == 0) a.cry[(size_t)I * D + ra] = P1 < a.n_v ? -__ldcg(a.vd + (size_t)a.ord[P1] * kVD + 49 + r) : 0.0;
  }
}

// CTA: in-place Cholesky of the D x D matrix in shared memory (pitch D, lower triangle).
// Step k updates the trailing triangle with the unscaled column k (A_ij -= A_ik A_jk / d_k,
// one barrier per step); the thread that updates A_{k+1,k+1} also stores its reciprocal,
// so no step waits on a division. The columns are scaled at the end (L_ik = A_ik / sqrt(d_k)).
// Outputs for the triangular solves: inv[k] = 1 / L_kk and, per 7 x 7 diagonal block q,
// its inverse Binv[q] (lower triangular, row-major 49). rcp: D scratch doubles.
// Returns false (CTA-uniform) on a non-positive pivot.
__device__ bool cr_chol(double* A, int D, double* inv, double* Binv, double* rcp) {
  const int t = threadIdx.x, ty = t >> 4, tx = t & 15;
  if (t == 0) rcp[0] = 1.0 / A[0];
  __syncthreads();
  for (int k = 0; k < D; ++k) {
    const double dk = A[k * D + k];
    if (!(dk > 0.0)) return false;
    const double rk = rcp[k];
    for (int i = k + 1 + ty; i < D; i += 16) {
      const double f = A[i * D + k] * rk;
      for (int j = k + 1 + tx; j <= i; j += 16) {
        const double v = A[i * D + j] - f * A[j * D + k];
        A[i * D + j] = v;
        if (i == k + 1 && j == k + 1) rcp[k + 1] = 1.0 / v;
      }
    }
    __syncthreads();
  }
  for (int k = t; k < D; k += kT) {
    const double l = sqrt(A[k * D + k]);
    inv[k] = 1.0 / l;
    A[k * D + k] = l;
  }
  __syncthreads();
  for (int e = t; e < D * D; e += kT) {
    const int i = e / D, k = e - i * D;
    if (k < i) A[e] = A[e] * inv[k];
  }
  __syncthreads();
  // inverse of each diagonal 7 x 7 block: thread per (block, column), forward substitution
  for (int w = t; w < D; w += kT) {
    const int q = w / 7, c = w - 7 * q, o = 7 * q;
    double y[7];
#pragma unroll
    for (int r = 0; r < 7; ++r) {
      double sacc = r == c ? 1.0 : 0.0;
#pragma unroll
      for (int m = 0; m < r; ++m) sacc -= A[(o + r) * D + o + m] * y[m];
      y[r] = r < c ? 0.0 : sacc * inv[o + r];
    }
#pragma unroll
    for (int r = 0; r < 7; ++r) Binv[49 * q + 7 * r + c] = y[r];
  }
  __syncthreads();
  return true;
}

#ifndef LC_CR_BLOCKED
#define LC_CR_BLOCKED 1
#endif
// Blocked (7-wide block columns) right-looking Cholesky of the D x D SPD super-block, same
// outputs as cr_chol: per block column K (o = 7K) -- (1) warp 0 factors the 7 x 7 diagonal
// block in registers (lane r = row r, pivots and columns by shuffle) and forms its inverse
// Binv_K; (2) thread per row i >= o + 7: L_iK = A_iK Binv_K^T; (3) the trailing lower
// triangle A_ij -= sum_m L_im L_jm over 4 x 4 register tiles (the 7-term products summed
// in registers: 0.8 shared-memory accesses per FMA instead of 3) -- three barriers per
// block column instead of one per column. Returns false (CTA-uniform) on a non-positive pivot.
__device__ bool cr_chol_blocked(double* A, int D, double* inv, double* Binv, int* bad) {
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const int nb = D / 7;
  if (t == 0) *bad = 0;
  __syncthreads();
  for (int K = 0; K < nb; ++K) {
    const int o = 7 * K;
    if (warp == 0) {   // (1) diagonal block
      double row[7];
#pragma unroll
      for (int c = 0; c < 7; ++c) row[c] = (lane < 7 && c <= lane) ? A[(o + lane) * D + o + c] : 0.0;
      double il[7];
#pragma unroll
      for (int c = 0; c < 7; ++c) {
        const double piv = __shfl_sync(0xffffffffu, row[c], c);
        if (!(piv > 0.0) && lane == 0) *bad = 1;
        const double l = sqrt(piv);
        il[c] = 1.0 / l;
        if (lane == c) row[c] = l;
        else if (lane > c && lane < 7) row[c] *= il[c];
#pragma unroll
        for (int j = c + 1; j < 7; ++j) {
          const double ljc = __shfl_sync(0xffffffffu, row[c], j);
          if (lane < 7 && lane >= j) row[j] -= row[c] * ljc;
        }
      }
      if (lane < 7) {
#pragma unroll
        for (int c = 0; c < 7; ++c)
          if (c <= lane) A[(o + lane) * D + o + c] = row[c];
#pragma unroll
        for (int c = 0; c < 7; ++c)
          if (c == lane) inv[o + c] = il[c];
      }
      // Binv_K: lane c (< 7) forms column c of L_KK^-1 by forward substitution
      double y[7];
#pragma unroll
      for (int r = 0; r < 7; ++r) {
        double sacc = (r == lane) ? 1.0 : 0.0;
#pragma unroll
        for (int m = 0; m < r; ++m) sacc -= __shfl_sync(0xffffffffu, row[m], r) * y[m];
        y[r] = r < lane ? 0.0 : sacc * il[r];
      }
      if (lane < 7) {
#pragma unroll
        for (int r = 0; r < 7; ++r) Binv[49 * K + 7 * r + lane] = y[r];
      }
    }
    __syncthreads();
    if (*bad) return false;
    const int n = D - o - 7;
    if (n <= 0) break;
    // (2) panel: L_iK = A_iK Binv_K^T (lower-triangular Binv: m <= c)
    for (int i = o + 7 + t; i < D; i += kT) {
      double av[7];
#pragma unroll
      for (int m = 0; m < 7; ++m) av[m] = A[i * D + o + m];
      const double* Bi = Binv + 49 * K;
#pragma unroll
      for (int c = 0; c < 7; ++c) {
        double sacc = 0.0;
#pragma unroll
        for (int m = 0; m <= c; ++m) sacc += av[m] * Bi[7 * c + m];
        A[i * D + o + c] = sacc;
      }
    }
    __syncthreads();
    // (3) trailing update over 4 x 4 tiles (ti >= tj), rows / columns >= o + 7
    const int T = (n + 3) >> 2;
    const int npair = T * (T + 1) / 2;
    for (int pi = t; pi < npair; pi += kT) {
      int ti = (int)((sqrtf(8.0f * (float)pi + 1.0f) - 1.0f) * 0.5f);   // pi = ti (ti + 1) / 2 + tj
      while ((ti + 1) * (ti + 2) / 2 <= pi) ++ti;
      while (ti * (ti + 1) / 2 > pi) --ti;
      const int tj = pi - ti * (ti + 1) / 2;
      const int i0 = o + 7 + 4 * ti, j0 = o + 7 + 4 * tj;
      double li[4][7], lj[4][7];
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int m = 0; m < 7; ++m) {
          li[u][m] = i0 + u < D ? A[(i0 + u) * D + o + m] : 0.0;
          lj[u][m] = j0 + u < D ? A[(j0 + u) * D + o + m] : 0.0;
        }
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int v = 0; v < 4; ++v) {
          const int i = i0 + u, j = j0 + v;
          if (i < D && j <= i) {
            double sacc = 0.0;
#pragma unroll
            for (int m = 0; m < 7; ++m) sacc += li[u][m] * lj[v][m];
            A[i * D + j] -= sacc;
          }
        }
    }
    __syncthreads();
  }
  return true;
}

// CTA: B <- L^-1 B for a D x pc panel (pitch kCrPC) in shared memory, L lower (pitch D),
// Binv the inverses of its 7 x 7 diagonal blocks: per 7-row block, X_q = Binv_q B_q (thread
// per column), then the rank-7 update of the rows below (thread per (row, column) tile)
__device__ void cr_trsm(const double* L, const double* Binv, int D, double* B, int pc) {
  const int t = threadIdx.x, ty = t >> 4, tx = t & 15;
  for (int q = 0; q < D; q += 7) {
    if (t < pc) {
      double b[7];
#pragma unroll
      for (int r = 0; r < 7; ++r) b[r] = B[(q + r) * kCrPC + t];
      const double* Bi = Binv + 7 * q;   // 49 (q / 7)
#pragma unroll
      for (int r = 0; r < 7; ++r) {
        double sacc = 0.0;
#pragma unroll
        for (int m = 0; m <= r; ++m) sacc += Bi[7 * r + m] * b[m];
        B[(q + r) * kCrPC + t] = sacc;
      }
    }
    __syncthreads();
    if (q + 7 < D) {
      double xv[4][7];
#pragma unroll
      for (int v = 0; v < 4; ++v)
#pragma unroll
        for (int m = 0; m < 7; ++m) xv[v][m] = (tx + 16 * v < pc) ? B[(q + m) * kCrPC + tx + 16 * v] : 0.0;
      for (int row = q + 7 + ty; row < D; row += 16) {
        double l[7];
#pragma unroll
        for (int m = 0; m < 7; ++m) l[m] = L[row * D + q + m];
#pragma unroll
        for (int v = 0; v < 4; ++v) {
          const int c = tx + 16 * v;
          if (c < pc) {
            double sacc = B[row * kCrPC + c];
#pragma unroll
            for (int m = 0; m < 7; ++m) sacc -= l[m] * xv[v][m];
            B[row * kCrPC + c] = sacc;
          }
        }
      }
    }
    __syncthreads();
  }
}

// CTA: acc[u][v] = sum_m P[m][a_u] Q[m][c_v], a_u = ty + 16 u (< D), c_v = tx + 16 v (< pc)
__device__ __forceinline__ void cr_gemm_tn(const double* P, int ldp, const double* Q, int ldq, int D, int pc,
                                           double (&acc)[8][4]) {
  const int ty = threadIdx.x >> 4, tx = threadIdx.x & 15;
#pragma unroll
  for (int u = 0; u < 8; ++u)
#pragma unroll
    for (int v = 0; v < 4; ++v) acc[u][v] = 0.0;
  int au[8], cv[4];
#pragma unroll
  for (int u = 0; u < 8; ++u) au[u] = min(ty + 16 * u, D - 1);
#pragma unroll
  for (int v = 0; v < 4; ++v) cv[v] = min(tx + 16 * v, pc - 1);
#pragma unroll 2
  for (int m = 0; m < D; ++m) {
    double p[8], q[4];
#pragma unroll
    for (int u = 0; u < 8; ++u) p[u] = P[m * ldp + au[u]];
#pragma unroll
    for (int v = 0; v < 4; ++v) q[v] = Q[m * ldq + cv[v]];
#pragma unroll
    for (int u = 0; u < 8; ++u)
#pragma unroll
      for (int v = 0; v < 4; ++v) acc[u][v] += p[u] * q[v];
  }
}

// CTA: z <- L^-T z (L lower in shared memory, pitch D, inv = 1 / diag; z in shared
// memory), one warp, right-looking: lane owns z_m for m = lane mod 32 in registers; x_r from
// its owner by shuffle, then every lane subtracts L_rm x_r from its z_m (m < r)
__device__ void cr_ltsolve(const double* L, const double* inv, int D, double* z) {
  if (threadIdx.x < 32) {
    const int lane = threadIdx.x;
    double zr[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) zr[u] = lane + 32 * u < D ? z[lane + 32 * u] : 0.0;
    for (int r = D - 1; r >= 0; --r) {
      const int u0 = r >> 5;
      double own = zr[0];
#pragma unroll
      for (int u = 1; u < 4; ++u) own = u == u0 ? zr[u] : own;
      const double xr = __shfl_sync(0xffffffffu, own, r & 31) * inv[r];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int m = lane + 32 * u;
        if (m < r) zr[u] -= L[r * D + m] * xr;
        else if (m == r) zr[u] = xr;
      }
    }
#pragma unroll
    for (int u = 0; u < 4; ++u)
      if (lane + 32 * u < D) z[lane + 32 * u] = zr[u];
  }
  __syncthreads();
}

// global (L2) -> shared, 8 loads in flight per thread
__device__ __forceinline__ void cr_load(double* dst, const double* src, int n) {
  for (int e0 = threadIdx.x; e0 < n; e0 += 8 * kT) {
    double v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) v[u] = e0 + u * kT < n ? __ldcg(src + e0 + u * kT) : 0.0;
#pragma unroll
    for (int u = 0; u < 8; ++u)
      if (e0 + u * kT < n) dst[e0 + u * kT] = v[u];
  }
}

// eliminate super-block i at stride st (CTA); false on a non-positive pivot
__device__ bool cr_eliminate(const PgoArgs& a, int i, int st, double* sm, long long* et) {
#ifdef LC_PGO_TIMING
  long long tl = clock64();
#define CE_TIC(k) do { if (et && threadIdx.x == 0) { const long long c_ = clock64(); et[k] += c_ - tl; tl = c_; } } while (0)
#else
#define CE_TIC(k) do { (void)et; } while (0)
#endif
  const int D = 7 * a.cr_s, N = a.cr_N, r = i + st;
  const size_t DD = (size_t)D * D;
  double* sL = sm;
  double* sB = sm + DD;
  double* sInv = sB + (size_t)D * kCrPC;
  double* sBinv = sInv + D;   // [D / 7][49]
  double* sRcp = sBinv + 7 * D;
  cr_load(sL, a.crA + i * DD, (int)DD);
  __syncthreads();
  CE_TIC(0);
#if LC_CR_BLOCKED
  if (!cr_chol_blocked(sL, D, sInv, sBinv, (int*)sRcp)) return false;
#else
  if (!cr_chol(sL, D, sInv, sBinv, sRcp)) return false;
#endif
  CE_TIC(1);
  for (int e = threadIdx.x; e < (int)DD; e += kT) a.crA[i * DD + e] = sL[e];
  const int ncol = D + (r < N ? D : 0) + 1;   // [A_il | A_ir | b_i]
  double* Ci = a.crC + i * DD;
  const double* Cr = a.crC + (size_t)r * DD;  // A_ri (rows r, cols i): A_ir = Cr^T
  double* Xi = a.crX + i * DD;
  double* yi = a.cry + (size_t)i * D;
  for (int c0 = 0; c0 < ncol; c0 += kCrPC) {
    const int pc = min(kCrPC, ncol - c0);
    // 8 loads in flight per thread; A_il and b_i row-major, A_ir = A_ri^T read along A_ri's rows
    for (int e0 = threadIdx.x; e0 < D * pc; e0 += 8 * kT) {
      double v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int e = e0 + u * kT;
        v[u] = 0.0;
        if (e < D * pc) {
          const int ra = e / pc, c = e - ra * pc, g = c0 + c;
          if (g < D) v[u] = __ldcg(Ci + (size_t)ra * D + g);
          else if (g == ncol - 1) v[u] = __ldcg(yi + ra);
        }
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int e = e0 + u * kT;
        if (e < D * pc) {
          const int ra = e / pc, c = e - ra * pc, g = c0 + c;
          if (g < D || g == ncol - 1) sB[ra * kCrPC + c] = v[u];
        }
      }
    }
    for (int e0 = threadIdx.x; e0 < D * pc; e0 += 8 * kT) {
      double v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int e = e0 + u * kT;
        v[u] = 0.0;
        if (e < D * pc) {
          const int c = e / D, ra = e - c * D, g = c0 + c;
          if (g >= D && g < ncol - 1) v[u] = __ldcg(Cr + (size_t)(g - D) * D + ra);
        }
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int e = e0 + u * kT;
        if (e < D * pc) {
          const int c = e / D, ra = e - c * D, g = c0 + c;
          if (g >= D && g < ncol - 1) sB[ra * kCrPC + c] = v[u];
        }
      }
    }
    __syncthreads();
    CE_TIC(2);
    cr_trsm(sL, sBinv, D, sB, pc);
    CE_TIC(3);
    for (int e = threadIdx.x; e < D * pc; e += kT) {
      const int ra = e / pc, c = e - ra * pc, g = c0 + c;
      const double v = sB[ra * kCrPC + c];
      if (g < D) Ci[(size_t)ra * D + g] = v;
      else if (g < ncol - 1) Xi[(size_t)ra * D + (g - D)] = v;
      else yi[ra] = v;
    }
    __syncthreads();
  }
  CE_TIC(4);
#undef CE_TIC
  return true;
}

// Schur update of survivor J at stride st (CTA)
__device__ void cr_update(const PgoArgs& a, int J, int st, double* sm) {
  const int D = 7 * a.cr_s, N = a.cr_N;
  const size_t DD = (size_t)D * D;
  const int ty = threadIdx.x >> 4, tx = threadIdx.x & 15;
  double* sP = sm;
  double* sQ = sm + DD;
  double* sy = sQ + (size_t)D * kCrPC;
  double* AJ = a.crA + (size_t)J * DD;
  double* bJ = a.cry + (size_t)J * D;
  for (int side = 0; side < 2; ++side) {
    const int i = side == 0 ? J - st : J + st;   // eliminated neighbour: left (J is its r) or right (J is its l)
    if (i < 0 || i >= N) continue;
    const double* Pm = side == 0 ? a.crX + (size_t)i * DD : a.crC + (size_t)i * DD;   // X_r(i) / X_l(i)
    cr_load(sP, Pm, (int)DD);
    cr_load(sy, a.cry + (size_t)i * D, D);
    __syncthreads();
    // A_J -= P^T P (lower triangle read later; the full block is kept symmetric)
    for (int c0 = 0; c0 < D; c0 += kCrPC) {
      const int pc = min(kCrPC, D - c0);
      double acc[8][4];
      double old[8][4];   // issued before the products: 32 loads in flight
#pragma unroll
      for (int u = 0; u < 8; ++u)
#pragma unroll
        for (int v = 0; v < 4; ++v) {
          const int ar = ty + 16 * u, c = tx + 16 * v;
          old[u][v] = (ar < D && c < pc) ? __ldcg(AJ + (size_t)ar * D + c0 + c) : 0.0;
        }
      cr_gemm_tn(sP, D, sP + c0, D, D, pc, acc);
#pragma unroll
      for (int u = 0; u < 8; ++u)
#pragma unroll
        for (int v = 0; v < 4; ++v) {
          const int ar = ty + 16 * u, c = tx + 16 * v;
          if (ar < D && c < pc) AJ[(size_t)ar * D + c0 + c] = old[u][v] - acc[u][v];
        }
    }
    // b_J -= P^T y_i
    for (int ar = threadIdx.x; ar < D; ar += kT) {
      double sacc = 0.0;
      for (int m = 0; m < D; ++m) sacc += sP[m * D + ar] * sy[m];
      bJ[ar] = __ldcg(bJ + ar) - sacc;
    }
    if (side == 0) {
      // new left coupling of J (with i - st): -X_r(i)^T X_l(i)
      const double* Xl = a.crC + (size_t)i * DD;
      double* CJ = a.crC + (size_t)J * DD;
      for (int c0 = 0; c0 < D; c0 += kCrPC) {
        const int pc = min(kCrPC, D - c0);
        for (int e0 = threadIdx.x; e0 < D * pc; e0 += 8 * kT) {
          double v[8];
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            const int e = e0 + u * kT, m = e / pc, c = e - m * pc;
            v[u] = e < D * pc ? __ldcg(Xl + (size_t)m * D + c0 + c) : 0.0;
          }
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            const int e = e0 + u * kT, m = e / pc, c = e - m * pc;
            if (e < D * pc) sQ[m * kCrPC + c] = v[u];
          }
        }
        __syncthreads();
        double acc[8][4];
        cr_gemm_tn(sP, D, sQ, kCrPC, D, pc, acc);
#pragma unroll
        for (int u = 0; u < 8; ++u)
#pragma unroll
          for (int v = 0; v < 4; ++v) {
            const int ar = ty + 16 * u, c = tx + 16 * v;
            if (ar < D && c < pc) CJ[(size_t)ar * D + c0 + c] = -acc[u][v];
          }
        __syncthreads();
      }
    }
    __syncthreads();
  }
}

// back substitution of eliminated super-block i at stride st (CTA)
__device__ void cr_backsub(const PgoArgs& a, int i, int st, double* sm) {
  const int D = 7 * a.cr_s, N = a.cr_N, r = i + st, l = i - st;
  const size_t DD = (size_t)D * D;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double* sL = sm;
  double* z = sm + DD;
  double* xl = z + D;
  double* xr = xl + D;
  double* sInv = xr + D;
  cr_load(sL, a.crA + (size_t)i * DD, (int)DD);
  cr_load(xl, a.crx + (size_t)l * D, D);
  if (r < N) cr_load(xr, a.crx + (size_t)r * D, D);
  for (int e = threadIdx.x; e < D; e += kT) sInv[e] = 1.0 / __ldcg(a.crA + (size_t)i * DD + (size_t)e * D + e);
  __syncthreads();
  const double* Xl = a.crC + (size_t)i * DD;
  const double* Xr = a.crX + (size_t)i * DD;
  for (int ar = warp; ar < D; ar += kT / 32) {
    double sacc = 0.0;
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int m = lane + 32 * u;
      if (m < D) {
        sacc += __ldcg(Xl + (size_t)ar * D + m) * xl[m];
        if (r < N) sacc += __ldcg(Xr + (size_t)ar * D + m) * xr[m];
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) sacc += __shfl_xor_sync(0xffffffffu, sacc, o);
    if (lane == 0) z[ar] = __ldcg(a.cry + (size_t)i * D + ar) - sacc;
  }
  __syncthreads();
  cr_ltsolve(sL, sInv, D, z);
  for (int e = threadIdx.x; e < D; e += kT) a.crx[(size_t)i * D + e] = z[e];
}

// the whole solve, every CTA (grid barriers inside); X <- delta (vertex order). Returns
// the CTA-uniform fail flag and |delta|^2 in out2.
__device__ void cr_solve(const PgoArgs& a, double lambda, double* sm, double* X, unsigned int& bt,
                         double (*shR)[4], int nsolve, double* out2) {
  const int D = 7 * a.cr_s, N = a.cr_N, s = a.cr_s;
  const size_t DD = (size_t)D * D;
  double* fail = a.bres + 2 + (nsolve & 1);
#ifdef LC_PGO_TIMING
  // CTA 0 (eliminates super-block st, updates survivor 0 at each level): per-phase cycles
  long long tim[8] = {0, 0, 0, 0, 0, 0, 0, 0}, tlast = clock64();
#define CR_TIC(k) do { if (blockIdx.x == 0 && threadIdx.x == 0) { const long long c_ = clock64(); tim[k] += c_ - tlast; tlast = c_; } } while (0)
#else
#define CR_TIC(k) do { } while (0)
#endif
  cr_assemble(a, lambda);
  CR_TIC(6);
  grid_barrier(a.bar, bt);
  CR_TIC(7);
  // every CTA has read the previous solve's flag (before this solve's first barrier)
  if (blockIdx.x == 0 && threadIdx.x == 0) a.bres[2 + ((nsolve + 1) & 1)] = 0.0;
  int st = 1;
  for (; st < N; st *= 2) {
    for (int i = st + 2 * st * (int)blockIdx.x; i < N; i += 2 * st * (int)gridDim.x)
      if (!cr_eliminate(a, i, st, sm,
#ifdef LC_PGO_TIMING
                        blockIdx.x == 0 ? a.ctim : nullptr
#else
                        nullptr
#endif
                        ) && threadIdx.x == 0)
        *fail = 1.0;
    CR_TIC(0);
    grid_barrier(a.bar, bt);
    CR_TIC(1);
    for (int J = 2 * st * (int)blockIdx.x; J < N; J += 2 * st * (int)gridDim.x) cr_update(a, J, st, sm);
    CR_TIC(2);
    grid_barrier(a.bar, bt);
    CR_TIC(3);
  }
  if (blockIdx.x == 0) {   // the root super-block 0: x_0 = A_0^-1 b_0
    double* sL = sm;
    double* sB = sm + DD;
    double* sInv = sB + (size_t)D * kCrPC;
    double* sBinv = sInv + D;
    double* sRcp = sBinv + 7 * D;
    cr_load(sL, a.crA, (int)DD);
    for (int e = threadIdx.x; e < D; e += kT) sB[e * kCrPC] = __ldcg(a.cry + e);
    __syncthreads();
#if LC_CR_BLOCKED
    if (cr_chol_blocked(sL, D, sInv, sBinv, (int*)sRcp)) {
#else
    if (cr_chol(sL, D, sInv, sBinv, sRcp)) {
#endif
      cr_trsm(sL, sBinv, D, sB, 1);
      double* z = sRcp;
      for (int e = threadIdx.x; e < D; e += kT) z[e] = sB[e * kCrPC];
      __syncthreads();
      cr_ltsolve(sL, sInv, D, z);
      for (int e = threadIdx.x; e < D; e += kT) a.crx[e] = z[e];
    } else if (threadIdx.x == 0) {
      *fail = 1.0;
    }
  }
  CR_TIC(5);
  grid_barrier(a.bar, bt);
  CR_TIC(7);
  for (st >>= 1; st >= 1; st >>= 1) {
    for (int i = st + 2 * st * (int)blockIdx.x; i < N; i += 2 * st * (int)gridDim.x) cr_backsub(a, i, st, sm);
    __syncthreads();
    CR_TIC(4);
    grid_barrier(a.bar, bt);
    CR_TIC(7);
  }
#ifdef LC_PGO_TIMING
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    for (int k = 0; k < 8; ++k) a.counts[k] += (unsigned long long)tim[k];
    for (int k = 0; k < 5; ++k) a.counts[8 + k] += (unsigned long long)a.ctim[k];
  }
#endif
#undef CR_TIC
  // positions -> vertices, |delta|^2 (fixed grid order: deterministic)
  double xx = 0.0;
  for (int e = blockIdx.x * kT + threadIdx.x; e < a.n_v * 7; e += gridDim.x * kT) {
    const int P = e / 7, r = e - 7 * P, I = P / s;
    const double v = __ldcg(a.crx + (size_t)I * D + 7 * (P - I * s) + r);
    X[(size_t)a.ord[P] * kVec + r] = v;
    xx += v * v;
  }
  double tot[4];
  cta_partial(xx, 0.0, 0.0, 0.0, a.part, shR);
  grid_barrier(a.bar, bt);
  grid_total(a.part, tot, shR);
  out2[0] = __ldcg(fail);
  out2[1] = tot[0];
}

__global__ void __launch_bounds__(kT, 1) k_pgo(PgoArgs a) {
  __shared__ double shJ[(kT / 16) * 112];
  __shared__ double shR[kT / 32][4];
  extern __shared__ double dsm[];
  unsigned int bt = 0;
  const int tid = blockIdx.x * kT + threadIdx.x, nth = gridDim.x * kT;
  const int lane8 = threadIdx.x & 7, g8 = tid >> 3, ng8 = nth >> 3;
  const unsigned m8 = 0xffu << (threadIdx.x & 24);
  const int warp = tid >> 5, nwarp = nth >> 5, lane = threadIdx.x & 31;
  double* X = a.vx;
  double* Rr = a.vx + (size_t)a.n_v * kVec;
  double* U = a.vx + 2 * (size_t)a.n_v * kVec;
  double* W = a.vx + 3 * (size_t)a.n_v * kVec;
  double* Pp = a.vx + 4 * (size_t)a.n_v * kVec;
  double* Sv = a.vx + 5 * (size_t)a.n_v * kVec;

  for (int k = tid; k < 13 * a.n_v; k += nth) {
    const double s = a.S_in[k];
    a.S_out[k] = s;
    a.S_tmp[k] = s;
  }
  if (tid < 2) a.bres[2 + tid] = 0.0;   // cyclic-reduction fail flags
  int nsolve = 0;
  grid_barrier(a.bar, bt);
  double* S = a.S_out;
  double* St = a.S_tmp;
  double tot[4];
  cta_partial(chi2_part(a, S), 0.0, 0.0, 0.0, a.part, shR);
  grid_barrier(a.bar, bt);
  grid_total(a.part, tot, shR);
  double chi2 = tot[0];
  const bool lead = blockIdx.x == 0 && threadIdx.x == 0;
  if (lead && a.chi2_out) a.chi2_out[0] = chi2;
  double lambda = a.lambda0;
  int stop = chi2 == 0.0 ? 5 : 0, it = 0, accepted = 0;
  long long cg_total = 0;
  bool relin = true, band_dirty = true;
  while (!stop) {
    if (it >= a.max_iter) { stop = 3; break; }
    if (relin) {
      linearise(a, S, shJ);
      grid_barrier(a.bar, bt);
      // assemble: warp per vertex, lanes over the 56 outputs
      for (int v = warp; v < a.n_v; v += nwarp) {
        const bool fx = a.fixed[v] != 0;
        const int b0 = a.vbeg[v], b1 = a.vbeg[v + 1];
        for (int o = lane; o < kVD; o += 32) {
          double s = 0.0;
          if (fx) {
            s = (o < 49 && (o / 7) == (o % 7)) ? 1.0 : 0.0;
          } else {
            for (int q = b0; q < b1; ++q) {
              const int w = __ldg(&a.vinc2[q].x), e = w >> 1, role = w & 1;
              const int off = o < 49 ? (role ? kOffHjj : kOffHii) + o : (role ? kOffBj : kOffBi) + (o - 49);
              s += __ldcg(a.rec + (size_t)e * kRec + off);
            }
          }
          a.vd[(size_t)v * kVD + o] = s;
        }
      }
      relin = false;
      band_dirty = true;
      grid_barrier(a.bar, bt);
    }
    double xx = 0.0;
    int k = 0;
    bool bad = false;
    double* row = nullptr;
    if (a.bw >= 0) {
      if (band_dirty) {
        band_assemble(a);
        band_dirty = false;
        grid_barrier(a.bar, bt);
      }
      double bfail, bxx;
      if (a.cr_s > 0) {
        double o2[2];
        cr_solve(a, lambda, dsm, X, bt, shR, nsolve++, o2);
        bfail = o2[0];
        bxx = o2[1];
      } else {
        if (blockIdx.x == 0) band_solve(a, lambda, dsm, X);
        grid_barrier(a.bar, bt);
        bfail = __ldcg(a.bres);
        bxx = __ldcg(a.bres + 1);
      }
      ++it;
      row = (lead && a.trace) ? a.trace + 6 * (size_t)(it - 1) : nullptr;
      if (row) { row[0] = chi2; row[1] = lambda; row[2] = -1.0; row[3] = 0.0; row[4] = -1.0; row[5] = 1.0; }
      if (bfail != 0.0) {
        lambda *= 4.0;
        if (lambda > 1e8) stop = 4;
        continue;
      }
      xx = bxx;
      k = 1;
    } else {
    // damped diagonal blocks -> Cholesky factors; x = 0, r = -b, u = P r
    double fail = 0.0, gam = 0.0, dlt = 0.0, rr = 0.0;
    for (int v = g8; v < a.n_v; v += ng8) {
      const double* D = a.vd + (size_t)v * kVD;
      double* L = a.vl + (size_t)v * kVL;
      int okv = 1;
      if (lane8 == 0) {
        double Ld[28];
        for (int i = 0; i < 7 && okv; ++i)
          for (int j = 0; j <= i; ++j) {
            double s = __ldcg(D + 7 * i + j);
            if (i == j) s = s + lambda * s;
            for (int k = 0; k < j; ++k) s -= Ld[i * (i + 1) / 2 + k] * Ld[j * (j + 1) / 2 + k];
            if (i == j) {
              if (!(s > 0.0)) { okv = 0; break; }
              Ld[i * (i + 1) / 2 + i] = sqrt(s);
            } else {
              Ld[i * (i + 1) / 2 + j] = s / Ld[j * (j + 1) / 2 + j];
            }
          }
        if (okv)
          for (int k = 0; k < 28; ++k) L[k] = Ld[k];
      }
      okv = __shfl_sync(m8, okv, threadIdx.x & 24);
      if (!okv) { fail = 1.0; continue; }
      __syncwarp(m8);
      const double bv = lane8 < 7 ? __ldcg(D + 49 + lane8) : 0.0;
      double rv[7];
#pragma unroll
      for (int i = 0; i < 7; ++i) rv[i] = -__shfl_sync(m8, bv, (threadIdx.x & 24) + i);
      const double ul = precond(L, rv, lane8);
      if (lane8 < 7) {
        const size_t o = (size_t)v * kVec + lane8;
        X[o] = 0.0;
        Rr[o] = -bv;
        U[o] = ul;
        gam += (-bv) * ul;
        rr += bv * bv;
      }
    }
    grid_barrier(a.bar, bt);
    for (int v = g8; v < a.n_v; v += ng8) {
      if (lane8 >= 7) continue;
      const double wl = spmv_row(a, v, lane8, U, lambda);
      const size_t o = (size_t)v * kVec + lane8;
      W[o] = wl;
      dlt += wl * U[o];
    }
    cta_partial(gam, dlt, rr, fail, a.part, shR);
    grid_barrier(a.bar, bt);
    grid_total(a.part, tot, shR);
    ++it;
    row = (lead && a.trace) ? a.trace + 6 * (size_t)(it - 1) : nullptr;
    if (row) { row[0] = chi2; row[1] = lambda; row[2] = -1.0; row[3] = 0.0; row[4] = -1.0; row[5] = 0.0; }
    if (tot[3] != 0.0) {
      lambda *= 4.0;
      if (lambda > 1e8) stop = 4;
      continue;
    }
    // preconditioned CG, Chronopoulos-Gear form (one reduction per iteration: two grid
    // barriers -- after the vector update (u visible to the neighbours' SpMV) and after
    // the SpMV + dot products)
    gam = tot[0];
    dlt = tot[1];
    rr = tot[2];
    const double stop2 = (a.cg_tol * a.cg_tol) * rr;
    double alpha = 0.0, gam_old = 0.0, alpha_old = 0.0;
    while (rr > stop2 && k < a.cg_max) {
      double beta = 0.0;
      if (k == 0) {
        if (!(dlt > 0.0)) { bad = true; break; }
        alpha = gam / dlt;
      } else {
        beta = gam / gam_old;
        const double den = dlt - beta * gam / alpha_old;
        if (!(den > 0.0)) { bad = true; break; }
        alpha = gam / den;
      }
      double gn = 0.0, rn = 0.0, xn = 0.0;
      for (int v = g8; v < a.n_v; v += ng8) {
        const size_t o = (size_t)v * kVec + lane8;
        double rl = 0.0;
        if (lane8 < 7) {
          const double pl = k == 0 ? U[o] : U[o] + beta * Pp[o];
          const double sl = k == 0 ? W[o] : W[o] + beta * Sv[o];
          Pp[o] = pl;
          Sv[o] = sl;
          const double xl = X[o] + alpha * pl;
          X[o] = xl;
          rl = Rr[o] - alpha * sl;
          Rr[o] = rl;
          xn += xl * xl;
          rn += rl * rl;
        }
        double rv[7];
#pragma unroll
        for (int i = 0; i < 7; ++i) rv[i] = __shfl_sync(m8, rl, (threadIdx.x & 24) + i);
        const double ul = precond(a.vl + (size_t)v * kVL, rv, lane8);
        if (lane8 < 7) {
          U[o] = ul;
          gn += rl * ul;
        }
      }
      grid_barrier(a.bar, bt);
      double dn2 = 0.0;
      for (int v = g8; v < a.n_v; v += ng8) {
        if (lane8 >= 7) continue;
        const double wl = spmv_row(a, v, lane8, U, lambda);
        const size_t o = (size_t)v * kVec + lane8;
        W[o] = wl;
        dn2 += wl * U[o];
      }
      cta_partial(gn, dn2, rn, xn, a.part, shR);
      grid_barrier(a.bar, bt);
      grid_total(a.part, tot, shR);
      gam_old = gam;
      alpha_old = alpha;
      gam = tot[0];
      dlt = tot[1];
      rr = tot[2];
      xx = tot[3];
      ++k;
    }
    }
    cg_total += k;
    if (row) row[5] = (double)k;
    if (bad) {
      lambda *= 4.0;
      if (lambda > 1e8) stop = 4;
      continue;
    }
    const double dn = sqrt(xx);
    if (row) row[4] = dn;
    if (dn < a.eps_dx) {
      if (row) row[2] = chi2;
      stop = 1;
      break;
    }
    // trial estimate
    for (int v = tid; v < a.n_v; v += nth) {
      if (a.fixed[v]) continue;
      double d[7], E[13], Sv[13], o[13];
#pragma unroll
      for (int r = 0; r < 7; ++r) d[r] = __ldcg(X + (size_t)v * kVec + r);
#pragma unroll
      for (int r = 0; r < 13; ++r) Sv[r] = __ldcg(S + 13 * (size_t)v + r);
      sim3_exp(d, E);
      lc_sim3_compose(E, Sv, o);
#pragma unroll
      for (int r = 0; r < 13; ++r) St[13 * (size_t)v + r] = o[r];
    }
    grid_barrier(a.bar, bt);
    cta_partial(chi2_part(a, St), 0.0, 0.0, 0.0, a.part, shR);
    grid_barrier(a.bar, bt);
    grid_total(a.part, tot, shR);
    const double chi2t = tot[0];
    if (row) row[2] = chi2t;
    if (chi2t < chi2) {
      if (row) row[3] = 1.0;
      ++accepted;
      const double rel = (chi2 - chi2t) / chi2;
      double* sw = S; S = St; St = sw;
      chi2 = chi2t;
      lambda = lambda * 0.5 < 1e-12 ? 1e-12 : lambda * 0.5;
      relin = true;
      if (rel < a.eps_chi2) stop = 2;
      // the rejected buffer must equal the new estimate on free vertices before the next
      // trial overwrites them: trial writes every free vertex, fixed ones are equal in both
    } else {
      lambda *= 4.0;
      if (lambda > 1e8) stop = 4;
    }
  }
  if (S != a.S_out)
    for (int k = tid; k < 13 * a.n_v; k += nth) a.S_out[k] = __ldcg(S + k);
  if (lead) {
    if (a.chi2_out) a.chi2_out[1] = chi2;
    a.counts[LC_COUNT_PGO_ITERS] = (unsigned long long)it;
    a.counts[LC_COUNT_PGO_ACCEPTED] = (unsigned long long)accepted;
    a.counts[LC_COUNT_PGO_SOLVER_ITERS] = (unsigned long long)cg_total;
    a.counts[LC_COUNT_PGO_STOP] = (unsigned long long)stop;
    a.counts[LC_COUNT_PGO_BAND] = (unsigned long long)(a.bw + 1);
    a.counts[LC_COUNT_PGO_CR_LEVELS] = (unsigned long long)a.cr_levels;
  }
}

}  // namespace

static size_t band_smem_bytes(int bw) {
  if (bw < 0) return 0;
  const size_t NB = (size_t)bw + 1;
  return sizeof(double) * (NB * (NB + 1) / 2 * 49 + NB * 8 * 3 + 16 + NB * 49) + 2 * NB * NB;
}
static size_t cr_smem_bytes(int s) {
  const size_t D = 7 * (size_t)s;
  return sizeof(double) * (D * D + D * kCrPC + 9 * D);
}
static size_t pgo_smem_bytes(int bw, int cr_s) { return cr_s > 0 ? cr_smem_bytes(cr_s) : band_smem_bytes(bw); }

int pgo_max_bw() { return kBWMax; }
int pgo_cr_max_s() { return kCrSMax; }
int pgo_cr_s(int bw) { return std::max(bw, 1); }

size_t pgo_scratch_bytes(int n_v, int n_e, int grid, int bw, int cr_s) {
  size_t d = (size_t)n_e * kRec + (size_t)n_v * (kVD + kVL + 6 * kVec + 13) + 4 * (size_t)grid + 8;
  if (bw >= 0) d += 2 * (size_t)n_v * (bw + 1) * 49 + (size_t)n_v * 8;
  if (cr_s > 0) {
    const size_t D = 7 * (size_t)cr_s, N = ((size_t)n_v + cr_s - 1) / cr_s;
    d += 3 * N * D * D + 2 * N * D;
  }
  return sizeof(double) * d + 256;
}

int pgo_grid(lc_ctx* c, int n_v, int n_e, int bw, int cr_s) {
  int dev = 0, sms = 148, per = 1;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const size_t smem = pgo_smem_bytes(bw, cr_s);
  cudaFuncSetAttribute(k_pgo, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_pgo, kT, smem);
  (void)c;
  int64_t work = std::max<int64_t>((int64_t)n_e * 16, (int64_t)n_v * 8);
  if (cr_s > 0) work = std::max<int64_t>(work, (int64_t)((n_v + cr_s - 1) / cr_s) * kT);   // CTA per super-block
  const int need = (int)std::max<int64_t>(1, (work + kT - 1) / kT);
  return std::max(1, std::min(need, sms * std::max(per, 1)));
}

cudaError_t launch_pgo(lc_ctx* c, int n_v, int n_e, const int32_t* d_eij, const double* d_M, const double* d_S_in,
                       const uint8_t* d_fixed, const int32_t* d_vbeg, const int32_t* d_vinc, int bw,
                       const int32_t* d_pos, const int32_t* d_ord, int cr_s, const lc_pgo_params& p,
                       double* d_S_out, void* scratch, int grid, double* d_trace, double* d_chi2,
                       unsigned long long* counts, cudaStream_t s) {
  PgoArgs a;
  a.vinc2 = (const int2*)d_vinc;
  a.n_v = n_v; a.n_e = n_e; a.max_iter = p.max_iter; a.cg_max = p.cg_max_iter;
  a.lambda0 = p.lambda0; a.eps_dx = p.eps_dx; a.eps_chi2 = p.eps_chi2; a.cg_tol = p.cg_tol;
  a.eij = d_eij; a.M = d_M; a.S_in = d_S_in; a.fixed = d_fixed; a.vbeg = d_vbeg;
  a.S_out = d_S_out;
  a.bw = bw; a.pos = d_pos; a.ord = d_ord;
  double* base = (double*)scratch;
  a.rec = base; base += (size_t)n_e * kRec;
  a.vd = base; base += (size_t)n_v * kVD;
  a.vl = base; base += (size_t)n_v * kVL;
  a.vx = base; base += (size_t)n_v * 6 * kVec;
  a.S_tmp = base; base += (size_t)n_v * 13;
  a.part = base; base += 4 * (size_t)grid;
  a.bres = base; base += 8;
  a.band = a.lband = a.yb = nullptr;
  if (bw >= 0) {
    a.band = base; base += (size_t)n_v * (bw + 1) * 49;
    a.lband = base; base += (size_t)n_v * (bw + 1) * 49;
    a.yb = base; base += (size_t)n_v * 8;
  }
  a.cr_s = cr_s; a.cr_N = 0; a.cr_levels = 0;
  a.crA = a.crC = a.crX = a.cry = a.crx = nullptr;
  if (cr_s > 0) {
    const size_t D = 7 * (size_t)cr_s;
    const int N = (n_v + cr_s - 1) / cr_s;
    a.cr_N = N;
    while ((1 << a.cr_levels) < N) ++a.cr_levels;
    a.crA = base; base += (size_t)N * D * D;
    a.crC = base; base += (size_t)N * D * D;
    a.crX = base; base += (size_t)N * D * D;
    a.cry = base; base += (size_t)N * D;
    a.crx = base; base += (size_t)N * D;
  }
  a.ctim = (long long*)((char*)base + 128);   // inside the zeroed 256-byte barrier block
  a.bar = (unsigned int*)base;
  a.trace = d_trace; a.chi2_out = d_chi2; a.counts = counts;
  cudaError_t e = cudaMemsetAsync(a.bar, 0, 256, s);
  if (e != cudaSuccess) return e;
  void* args[] = {&a};
  e = cudaLaunchCooperativeKernel((const void*)k_pgo, dim3(grid), dim3(kT), args, pgo_smem_bytes(bw, cr_s), s);
  c->launches++;
  return e;
}
