// lc_internal.cuh -- device store layout, context and fp64 geometry for liblc.
//
// Layout:
//   kf_pose      double[n_kf][13]       world->camera, mutable by corrections
//   kf_cam       int32[n_kf]
//   kf_fbeg      int32[n_kf+1]          CSR into feature arrays
//   kf_cell      uint16[n_kf][Gs]       per-keyframe cell start offsets, (octave, row, col)-major
//   fc_uv        float2[n_feat]         keypoints, (octave, cell)-major per keyframe
//   fc_meta      uint32[n_feat]         local original index (bits 0-15) | octave << 16
//   fc_desc      uint4[n_feat][2]       descriptors, cell-major
//   feat_mp      int32[n_feat]          associations, ORIGINAL order (mutable)
//   feat_angle   float[n_feat]          original order
//   mp_rec       MpRec[n_mp]            64-B rows: pos, dmax, normal, angle, desc
//   mp_flags     uint8[n_mp]; mp_ref_kf, mp_replaced_by, mp_nobs, mp_corr_ref int32[n_mp]
//   mp_loop_ep   uint32[n_mp]           LoopSet membership stamp (== fuse epoch)
//   kf_S_corr    double[n_kf][13]; kf_in_win int32[n_kf]   loop state (WINDOW -> ALL)
//   kf_win_ep    uint32[n_kf]; kf_win_pos int32[n_kf]      window membership of a fuse call
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <mutex>
#include <string>
#include <unordered_map>
#include <vector>

#include "lc.h"

#define LC_NTHREADS 256

struct __align__(16) MpRec {
  float pos[3];
  float dmax;
  float normal[3];
  float angle;
  uint4 desc[2];
};
static_assert(sizeof(MpRec) == 64, "MpRec must be 64 bytes");

struct DevCam {
  int model;
  int cols, rows;   // octave-0 grid (the per-octave grids are coarsened by the scale factor)
  int pad;
  double fx, fy, cx, cy;
  double k[4];
  double min_x, max_x, min_y, max_y;
  double cell_sx[LC_MAX_LEVELS], cell_sy[LC_MAX_LEVELS];   // octave o: cols_o / (max_x - min_x), ...
};

struct Store {
  int32_t n_kf = 0, n_feat = 0, n_mp = 0, n_cams = 0;
  int32_t n_levels = 0, cols = 0, rows = 0, G = 0;
  // per-octave grids: octave o uses ocols[o] x orows[o] cells (the octave-0
  // grid coarsened by scale_factor^o); the per-keyframe cell table is (octave, row, col)-
  // major, obase[o] = first cell of octave o, G = obase[n_levels] cells in total
  int32_t ocols[LC_MAX_LEVELS] = {}, orows[LC_MAX_LEVELS] = {}, obase[LC_MAX_LEVELS + 1] = {};
  int32_t Gs = 0;        // per-keyframe cell-table stride: round_up(G + 1, 8) (16-B rows for TMA)
  int64_t n_fpad = 0;    // padded feature count of the cell-major arrays
  double scale[LC_MAX_LEVELS];
  int32_t max_F = 0;
  // capacities (entries) of the KF-, feature-, padded-feature- and MP-indexed device arrays:
  // LC_UPLOAD_APPEND grows them geometrically
  int64_t cap_kf = 0, cap_feat = 0, cap_fpad = 0, cap_mp = 0;
  // device arrays
  double* kf_pose = nullptr;
  int32_t* kf_cam = nullptr;
  int32_t* kf_fbeg = nullptr;
  int32_t* kf_fpad = nullptr;   // [n_kf+1] start of each keyframe's cell-major block (multiple of 4)
  uint16_t* kf_cell = nullptr;
  float2* fc_uv = nullptr;
  uint32_t* fc_meta = nullptr;
  uint4* fc_desc = nullptr;
  int32_t* feat_mp = nullptr;
  float* feat_angle = nullptr;
  int32_t* feat_cpos = nullptr;   // [n_feat] cell-major position of each original-order feature
  MpRec* mp_rec = nullptr;
  uint8_t* mp_flags = nullptr;
  int32_t* mp_ref_kf = nullptr;
  int32_t* mp_replaced_by = nullptr;
  int32_t* mp_nobs = nullptr;
  int32_t* mp_corr_ref = nullptr;
  uint32_t* mp_loop_ep = nullptr;
  int32_t* mp_owner = nullptr;
  double* kf_S_corr = nullptr;
  int32_t* kf_in_win = nullptr;
  uint32_t* kf_win_ep = nullptr;
  uint32_t* ep = nullptr;        // [2]: current fuse epoch, k_fuse_prep block-done counter
  int32_t* kf_win_pos = nullptr;
  uint32_t* mp_vbits = nullptr;  // [(n_mp+31)/32] victim bitmap of the current fuse call
  int32_t* kf_dirty = nullptr;   // [1 + n_kf] count + keyframes changed by the apply
  DevCam* cams = nullptr;
  // host copies
  std::vector<int32_t> h_fbeg;
  std::vector<int32_t> h_in_win;  // mirrors kf_in_win (set by WINDOW, cleared by ALL)
};

// Parameters of one matching launch, passed by value.
// compacted survivor of the geometric culls (k_project -> k_match): 16 bytes, the
// projection rounded to fp32 (the exact fp64 (u, v) is recomputed with lc_se3_xyz +
// lc_project -- the same expressions, hence the same bits -- where a window decision
// needs it).
struct __align__(16) Surv {
  int32_t q;
  uint32_t jl;   // (position in the block's query range) | (level << 27)
  float fu, fv;  // (float)u, (float)v
};

struct MatchArgs {
  // store
  const double* kf_pose;  // unused by the kernel (units carry S)
  const int32_t* kf_cam;
  const int32_t* kf_fbeg;
  const int32_t* kf_fpad;
  const uint16_t* kf_cell;
  const float2* fc_uv;
  const uint32_t* fc_meta;
  const uint4* fc_desc;
  const int32_t* feat_mp;
  const MpRec* mp_rec;
  const uint8_t* mp_flags;
  const DevCam* cams;
  int32_t cols, rows, G, n_levels, Gs;
  int32_t ocols[LC_MAX_LEVELS], orows[LC_MAX_LEVELS], obase[LC_MAX_LEVELS + 1];   // per-octave grids
  double scale[LC_MAX_LEVELS];
  // call
  const int32_t* unit_kf;      // [n_units]
  const double* unit_S;        // [n_units][13], or nullptr: kf_S_corr of the unit's keyframe
  const double* kf_S_corr;     // [n_kf][13] S^corr of the last WINDOW correction
  int32_t n_mp;
  const int32_t* unit_param;   // [n_units] (SBP) or nullptr (param 0)
  const int64_t* unit_woff;    // [n_units] offset into the winner table
  const int64_t* unit_toff;    // [n_units] offset into pair_taken (SBP)
  const int64_t* unit_lbeg;    // [n_units] list begin in mp_list
  const int64_t* unit_qoff;    // [n_units] debug query index of list entry 0
  const lc_match_params* params;
  const int32_t* blk_unit;     // [n_blocks]
  const int64_t* blk_q0;       // [n_blocks] list positions [q0, q1)
  const int64_t* blk_q1;
  const int32_t* mp_list;
  const int32_t* taken;        // SBP pair_taken (pair-major) or nullptr
  unsigned long long* winner;  // packed (H<<32)|q, window/pair-major
  unsigned long long* counts;  // [LC_NCOUNT] (fuse) or [n_units][LC_NCOUNT] (SBP)
  int64_t* dbg_best;
  double* dbg_uv;
  int32_t* dbg_ncand;
  int32_t hash_size;           // already-found table slots (>= 1.5 F_max)
  int32_t off_uv, off_meta, off_hash, off_queue;   // dynamic smem carve (bytes)
  int32_t warp_bytes;                              // per-warp ring + candidate slots
  // resolve (orientation + actions / SBP output tables)
  const float* feat_angle;
  const uint32_t* loop_ep;
  const uint32_t* epoch;  // device word: the current fuse call's epoch (set by k_fuse_prep)
  unsigned long long* victim;
  int8_t* action;
  int32_t* out_mp;
  int32_t* out_dist;
  int32_t sole;        // 1: one CTA per unit -> the match CTA initialises and resolves its unit
  Surv* surv;          // survivor buffer (k_project -> k_match), per-block regions
  const int64_t* surv_off;  // [n_blocks] region start (= block query offset)
  int32_t* surv_cnt;        // [n_blocks] survivors written
  int32_t unit_base;   // k_resolve: unit = unit_base + blockIdx.x
  int32_t blk_base;    // k_project / k_match: block = blk_base + blockIdx.x (pipelined chunks)
  uint32_t* loop_ep_w; // non-null: k_project stamps the LoopSet (pipelined host-list mode)
  uint32_t stamp_epoch; // != 0: that epoch (host-known, eager calls), stamped inline in k_project's loop
};

struct lc_graph {
  lc_ctx* ctx = nullptr;
  cudaGraph_t graph = nullptr;
  cudaGraphExec_t exec = nullptr;
  std::vector<void*> dev;     // graph-owned device buffers (argument blocks, scratch)
  int64_t launches = 0;       // library kernels per replay
  int64_t n_fuse = 0;         // fuse calls (epochs) per replay
};

struct lc_ctx {
  int device = 0;
  bool broken = false;
  std::string err;
  Store st;
  bool has_map = false;
  bool has_saved = false;
  uint64_t ep_used = 0;   // fuse epochs consumed since the stamps were last cleared
  // CUDA-graph capture (lc_graph_begin/end): calls on cap_stream are recorded; their
  // argument blocks and scratch live in the graph's own arena
  lc_graph* cap = nullptr;
  cudaStream_t cap_stream = nullptr;
  int64_t cap_launch0 = 0;
  cudaStream_t side = nullptr;   // private stream: capture-time uploads, pipelined list copies
  static constexpr int kPipe = 4;              // chunks of a pipelined host-list fuse
  cudaEvent_t pipe_ev[kPipe + 1] = {};          // [kPipe]: start (side waits on the call stream)
  int64_t launches = 0;
  int sole_mode = -1;   // LC_SOLE env at create: -1 auto, 0 never, 1 whenever lists allow (testing)
  int64_t pipe_min = 1 << 18;   // LC_PIPE_MIN env at create: smallest host list that takes the pipelined upload
  // scratch arena: named growable device buffers
  std::vector<void*> scr_ptr;
  std::vector<size_t> scr_cap;
  // pinned staging ring: argument blocks of the last kPinRing calls may still be in
  // flight, so the host only waits when it laps the ring (not on every call)
  static constexpr int kPinRing = 8;
  void* pin[kPinRing] = {};
  size_t pin_cap[kPinRing] = {};
  size_t pin_cap_max = 0;               // capacity every slot is (re)allocated with
  // lc_set_point_range: the map-point slice [mp_lo, mp_hi) whose positions the correction
  // passes rewrite on this rank (mp_hi < 0: all)
  int32_t mp_lo = 0, mp_hi = -1;
  cudaEvent_t pin_ev[kPinRing] = {};   // recorded after the H2D out of that slot
  bool pin_ev_pending[kPinRing] = {};
  int pin_next = 0;
  std::vector<char> arg_host;   // the host argument block of the current call (reused)
  // staging ring for pageable host inputs (Call::upload): chunks of kStageChunk bytes
  static constexpr int kStageRing = 4;
  static constexpr size_t kStageChunk = size_t(8) << 20;
  static constexpr size_t kStageMin = size_t(1) << 20;   // smaller pageable copies go direct
  void* stg[kStageRing] = {};
  cudaEvent_t stg_ev[kStageRing] = {};
  int stg_next = 0;
  bool stage_on = false;   // LC_STAGE=1: pageable copies through the ring (measured slower than the driver's)
  // saved state (lc_state_save)
  void* sv = nullptr;
  size_t sv_cap = 0;
  std::vector<int32_t> sv_in_win;
  // device-time accounting (lc_profile_*)
  bool prof = false;
  struct ProfRec { int fam; cudaEvent_t a, b; int64_t launches; };
  std::vector<cudaEvent_t> ev_pool;
  std::vector<ProfRec> prof_pending;
  double prof_ms[LC_NPROF] = {};
  int64_t prof_n[LC_NPROF] = {};
  // deferred host copies (outputs to host memory)
  struct HostOut { void* host; const void* dev; size_t bytes; };
  std::vector<HostOut> host_outs;
};

// ---------------------------------------------------------------------------
// fp64 Sim3 arithmetic in the order of DESIGN.md "Sim3 arithmetic" (the build
// uses -fmad=false so nothing below is contracted into an FMA).
// ---------------------------------------------------------------------------
__host__ __device__ __forceinline__ double lc_row3(const double* r, const double* p) {
  return (r[0] * p[0] + r[1] * p[1]) + r[2] * p[2];
}
__host__ __device__ __forceinline__ double lc_col3(const double* R, int i, const double* p) {
  return (R[0 + i] * p[0] + R[3 + i] * p[1]) + R[6 + i] * p[2];
}
__host__ __device__ __forceinline__ void lc_sim3_apply(const double* S, const double* p, double* o) {
  double q0 = lc_row3(S + 0, p), q1 = lc_row3(S + 3, p), q2 = lc_row3(S + 6, p);
  o[0] = S[12] * q0 + S[9];
  o[1] = S[12] * q1 + S[10];
  o[2] = S[12] * q2 + S[11];
}
__host__ __device__ __forceinline__ void lc_sim3_compose(const double* A, const double* B, double* o) {
  double r[13];
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j)
      r[3 * i + j] = (A[3 * i + 0] * B[0 + j] + A[3 * i + 1] * B[3 + j]) + A[3 * i + 2] * B[6 + j];
#pragma unroll
  for (int i = 0; i < 3; ++i) r[9 + i] = A[12] * lc_row3(A + 3 * i, B + 9) + A[9 + i];
  r[12] = A[12] * B[12];
#pragma unroll
  for (int i = 0; i < 13; ++i) o[i] = r[i];
}
__host__ __device__ __forceinline__ void lc_sim3_inverse(const double* S, double* o) {
  double r[13];
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j) r[3 * i + j] = S[3 * j + i];
#pragma unroll
  for (int i = 0; i < 3; ++i) r[9 + i] = -lc_col3(S, i, S + 9) / S[12];
  r[12] = 1.0 / S[12];
#pragma unroll
  for (int i = 0; i < 13; ++i) o[i] = r[i];
}
__host__ __device__ __forceinline__ void lc_sim3_se3(const double* S, double* o) {
  double r[13];
#pragma unroll
  for (int i = 0; i < 9; ++i) r[i] = S[i];
#pragma unroll
  for (int i = 0; i < 3; ++i) r[9 + i] = S[9 + i] / S[12];
  r[12] = 1.0;
#pragma unroll
  for (int i = 0; i < 13; ++i) o[i] = r[i];
}

// Projection (reading A29). Returns u, v in fp64.
// camera coordinates of a map point under the SE3 part T = (R row-major, t) of a
// unit's Sim3 (reading A2), in the order of DESIGN.md "Sim3 arithmetic"
__device__ __forceinline__ void lc_se3_xyz(const double* T, double p0, double p1, double p2,
                                           double& x, double& y, double& z) {
  z = (T[6] * p0 + T[7] * p1) + T[8] * p2 + T[11];
  x = (T[0] * p0 + T[1] * p1) + T[2] * p2 + T[9];
  y = (T[3] * p0 + T[4] * p1) + T[5] * p2 + T[10];
}

__device__ __forceinline__ void lc_project(const DevCam& c, double x, double y, double z,
                                           double& u, double& v) {
  if (c.model == 0) {
    u = ((c.fx * x) / z) + c.cx;
    v = ((c.fy * y) / z) + c.cy;
    return;
  }
  double rho = sqrt((x * x) + (y * y));
  if (rho == 0.0) { u = c.cx; v = c.cy; return; }
  double th = atan2(rho, z);
  double t2 = th * th;
  double a = c.k[3];
  a = c.k[2] + t2 * a;
  a = c.k[1] + t2 * a;
  a = c.k[0] + t2 * a;
  a = 1.0 + t2 * a;
  double r = th * a;
  u = ((c.fx * r) * (x / rho)) + c.cx;
  v = ((c.fy * r) * (y / rho)) + c.cy;
}

// ---------------------------------------------------------------------------
// Programmatic dependent launch (PDL). A kernel launched with launch_pdl may start
// while its stream predecessor is still running; it must (1) touch only data no
// unfinished predecessor writes before pdl_wait(), and (2) execute pdl_wait() before
// it exits (so "predecessor complete" stays transitive along the stream). pdl_trigger()
// lets the next PDL kernel launch once every CTA has triggered or exited.
// ---------------------------------------------------------------------------
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
// Read-only-path load of a predecessor's output after pdl_wait(): a volatile asm statement
// keeps its place after griddepcontrol.wait (an __ldg / const __restrict__ load may be
// treated as invariant and scheduled above the wait).
__device__ __forceinline__ uint32_t ld_nc_after_wait(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.global.nc.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

template <typename... KArgs, typename... Args>
cudaError_t launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                       Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kernel, static_cast<KArgs>(args)...);
}

// Kernel attributes are process-wide: set the dynamic shared-memory limit (and the
// shared-memory carveout) of a kernel once per larger value instead of on every launch
// (a driver call each; the host enqueue of a C5 fuse call was dominated by them).
inline cudaError_t set_smem_attr(const void* fn, int bytes, bool carveout = false) {
  static std::mutex mu;
  static std::unordered_map<const void*, int> done;
  std::lock_guard<std::mutex> lk(mu);
  auto it = done.find(fn);
  if (it != done.end() && it->second >= bytes) return cudaSuccess;
  cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (e == cudaSuccess && carveout)
    e = cudaFuncSetAttribute(fn, cudaFuncAttributePreferredSharedMemoryCarveout, cudaSharedmemCarveoutMaxShared);
  if (e == cudaSuccess) done[fn] = bytes;
  return e;
}

// ---------------------------------------------------------------------------
// kernel launchers (defined in the .cu files)
// ---------------------------------------------------------------------------
cudaError_t launch_upload_pack(lc_ctx* c, int kf0, int f0, int mp0, const float* pos, const float* nrm,
                               const float* dmax, const uint8_t* desc, const float* ang, const float* fuv,
                               const uint8_t* foct, const uint8_t* fdesc, uint32_t* d_errs, cudaStream_t s);
cudaError_t launch_match(lc_ctx* c, int mode, const MatchArgs& a, int n_blocks, int F_max, int part,
                         cudaStream_t s, bool pdl = true);  // part 0: k_project, 1: k_match; blocks [a.blk_base, +n_blocks)
// winner words [0, n_wfeat) are set to NONE except [skip_lo, skip_hi) (sole-mode units)
cudaError_t launch_fuse_prep(lc_ctx* c, int phase, int zero_counts, int64_t skip_lo, int64_t skip_hi, int n_w,
                             const int32_t* d_window, int64_t n_wfeat, const int32_t* mp_list,
                             int64_t n_list_total,
                             unsigned long long* winner, unsigned long long* victim,
                             unsigned long long* counts, cudaStream_t s);   // zeroes counts
cudaError_t launch_forced(lc_ctx* c, int cur_kf, const int32_t* d_forced, unsigned long long* win_cur,
                          unsigned long long* victim, unsigned long long* counts, cudaStream_t s);
cudaError_t launch_resolve(lc_ctx* c, int mode, const MatchArgs& a, int n_units, cudaStream_t s);
cudaError_t launch_fuse_apply(lc_ctx* c, const int64_t* d_woff, const unsigned long long* winner,
                              const unsigned long long* victim, unsigned long long* counts,
                              cudaStream_t s);
cudaError_t launch_correct_window(lc_ctx* c, int cur_pos, int n_w, const int32_t* d_window,
                                  const double* d_Scw, double* d_scr, double* d_outS,
                                  unsigned long long* counts, cudaStream_t s);   // zeroes counts
int correct_window_scratch_stride();
int correct_all_scratch_stride();
cudaError_t launch_csr_units(lc_ctx* c, int n, const int32_t* d_begin, int64_t* d_t, cudaStream_t s);
cudaError_t launch_mp_positions(lc_ctx* c, int op, int lo, int hi, float* xyz, cudaStream_t s);
cudaError_t launch_correct_all(lc_ctx* c, const double* d_Sopt, double* d_scr,
                               unsigned long long* counts, cudaStream_t s);   // zeroes counts
size_t correct_dry_scratch_bytes(int n_batch, int n_slots, int n_mp);
cudaError_t launch_correct_dry(lc_ctx* c, int n_batch, int n_slots, const int32_t* d_wbeg, const int32_t* d_window,
                               const double* d_Scw, void* scratch, double* d_outS, int32_t* d_mp_begin,
                               int64_t capacity, int32_t* d_idx, float* d_pos, unsigned long long* counts,
                               cudaStream_t s);   // WINDOW | DRY_RUN batch (zeroes counts)
cudaError_t launch_adds(lc_ctx* c, int op, int n_w, const int32_t* d_window, const int64_t* d_woff, int64_t n_wfeat,
                        int64_t lo, int64_t hi, unsigned long long* winner, long long* idx, long long* word,
                        unsigned long long* d_n, int64_t n_in, int64_t capacity, cudaStream_t s);
int lists_bitmap_words();       // bitmap path, first pass: id range (32-bit words) a list may span
int lists_bitmap_words_max();   // ... second pass (the wide lists)
cudaError_t launch_kf_idrange(lc_ctx* c, int n_src, const int32_t* d_skf, int2* d_rng, cudaStream_t s);
cudaError_t launch_lists_bitmap(lc_ctx* c, int n, int n_lists, const int32_t* d_sel, int maxw, const int2* d_rng,
                                uint32_t* d_bm, int32_t* d_lo, int32_t* d_counts, const int32_t* d_sbeg,
                                const int32_t* d_skf, cudaStream_t s, bool only_wide = false);
cudaError_t launch_lists_scan(lc_ctx* c, int n, const int32_t* d_counts, int32_t* d_out_begin, cudaStream_t s);
cudaError_t launch_lists_emit_wide(lc_ctx* c, int n, int maxw, const int32_t* d_sbeg, const int32_t* d_skf,
                                   const int32_t* d_lo, const int32_t* d_out_begin, int32_t* d_out, cudaStream_t s);
cudaError_t launch_lists_emit(lc_ctx* c, int n, const uint32_t* d_bm, const int64_t* d_bm_off, const int32_t* d_lo,
                              const int32_t* d_counts, const int32_t* d_out_begin, int32_t* d_out, cudaStream_t s);
int lists_max_unique();     // distinct map points a loop list may hold
int lists_small_unique();   // ... in the first (small hash) pass
cudaError_t launch_lists_dedup(lc_ctx* c, bool large, int n, const int32_t* d_sel, const int32_t* d_sbeg,
                               const int32_t* d_skf, const int64_t* d_reg_off, int32_t* d_reg, int32_t* d_counts,
                               cudaStream_t s);
cudaError_t launch_lists_sort(lc_ctx* c, int n, int max_u, const int64_t* d_reg_off, const int32_t* d_reg,
                              const int32_t* d_out_begin, int32_t* d_out, cudaStream_t s);
cudaError_t launch_fill_u64(lc_ctx* c, unsigned long long* p, int64_t n, unsigned long long v,
                            cudaStream_t s);
cudaError_t launch_state_copy(lc_ctx* c, bool save, cudaStream_t s);
cudaError_t launch_download_pos(lc_ctx* c, float* out, cudaStream_t s);
cudaError_t launch_download_rec(lc_ctx* c, float* normal, float* dmax, uint8_t* desc, cudaStream_t s);
cudaError_t launch_obs_lists(lc_ctx* c, int32_t* d_obeg, int32_t* d_cursor, int32_t* d_bsum,
                             int32_t* d_obs, int32_t* d_obs_kf, cudaStream_t s);   // per-point observation lists
int obs_scan_blocks(int n_mp);
int connections_max_kf();
cudaError_t launch_refine(lc_ctx* c, int n_prob, const int32_t* d_pbeg, const double* P1, const double* P2,
                          const float* uv1, const float* uv2, const float* sig1, const float* sig2,
                          const int32_t* d_cam1, const int32_t* d_cam2, const double* S_in, int max_iter,
                          double th2, double lambda, double* out_S, int32_t* out_inl, uint8_t* out_mask,
                          unsigned long long* counts, cudaStream_t s);
cudaError_t launch_ransac(lc_ctx* c, int n_prob, const int32_t* d_pbeg, const double* P1, const double* P2,
                          const float* uv1, const float* uv2, const float* sig1, const float* sig2,
                          const int32_t* d_cam1, const int32_t* d_cam2, const int32_t* samples, int n_iter,
                          double chi2, int fix_scale, int refit, double* out_S, int32_t* out_inl,
                          uint8_t* out_mask, unsigned long long* counts, cudaStream_t s);
cudaError_t launch_connections(lc_ctx* c, int n_sel, const int32_t* d_idx, int th, int max_edges,
                               const int32_t* d_obeg, const int32_t* d_obs, const int32_t* d_obs_kf,
                               uint8_t* d_first, int32_t* out_n,
                               int32_t* out_kf, int32_t* out_w, unsigned long long* counts,
                               cudaStream_t s);
cudaError_t launch_refresh(lc_ctx* c, int n_sel, const int32_t* d_idx, int what, int32_t* d_obeg,
                           int32_t* d_cursor, int32_t* d_bsum, int32_t* d_obs, int32_t* d_obs_kf,
                           unsigned long long* counts, cudaStream_t s);
int pgo_max_bw();
int pgo_cr_max_s();
int pgo_cr_s(int bw);
size_t pgo_scratch_bytes(int n_v, int n_e, int grid, int bw, int cr_s);
int pgo_grid(lc_ctx* c, int n_v, int n_e, int bw, int cr_s);
cudaError_t launch_pgo(lc_ctx* c, int n_v, int n_e, const int32_t* d_eij, const double* d_M, const double* d_S_in,
                       const uint8_t* d_fixed, const int32_t* d_vbeg, const int32_t* d_vinc, int bw,
                       const int32_t* d_pos, const int32_t* d_ord, int cr_s, const lc_pgo_params& p,
                       double* d_S_out, void* scratch, int grid, double* d_trace, double* d_chi2,
                       unsigned long long* counts, cudaStream_t s);
