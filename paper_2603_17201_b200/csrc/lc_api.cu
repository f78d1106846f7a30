// lc_api.cu -- extern "C" entry points of liblc (include/lc.h): argument
// validation, host/device marshalling through one pinned argument block per
// call, scratch arena management and kernel orchestration.
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <new>
#include <string>
#include <vector>

#include "lc_internal.cuh"

namespace {

thread_local std::string g_create_err = "no error";

struct Fail {
  lc_status st;
};

void set_err(lc_ctx* c, const std::string& m) {
  if (c) c->err = m;
}

#define CK(expr)                                                                         \
  do {                                                                                   \
    cudaError_t e__ = (expr);                                                            \
    if (e__ != cudaSuccess) {                                                            \
      c->broken = true;                                                                  \
      set_err(c, std::string("CUDA error ") + cudaGetErrorString(e__) + " at " #expr);   \
      throw Fail{LC_ECUDA};                                                              \
    }                                                                                    \
  } while (0)

#define REQUIRE(cond, code, msg)      \
  do {                                \
    if (!(cond)) {                    \
      set_err(c, msg);                \
      throw Fail{code};               \
    }                                 \
  } while (0)

bool is_device_ptr(lc_ctx* c, const void* p) {
  if (!p) return false;
  cudaPointerAttributes at;
  if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  if (at.type == cudaMemoryTypeDevice || at.type == cudaMemoryTypeManaged) {
    if (at.type == cudaMemoryTypeDevice && at.device != c->device) {
      set_err(c, "device pointer belongs to another device");
      throw Fail{LC_EINVAL};
    }
    return true;
  }
  return false;
}

size_t round_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

// One API call: scratch slots, a pinned argument block, deferred host outputs.
struct Call {
  lc_ctx* c;
  cudaStream_t s;
  int slot = 0;
  std::vector<char>& args;                // host argument block (the context's, capacity kept)
  std::vector<std::pair<const void**, size_t>> arg_fix;   // (where to store dev ptr, offset)
  std::vector<lc_ctx::HostOut> outs;
  char* d_args = nullptr;

  Call(lc_ctx* ctx, void* stream) : c(ctx), s((cudaStream_t)stream), args(ctx->arg_host) {
    args.clear();
    if (args.capacity() < (size_t(1) << 20)) args.reserve(size_t(1) << 20);
  }

  void* scratch(size_t bytes) {
    bytes = std::max<size_t>(round_up(bytes, 256), 256);
    if (c->cap) return graph_alloc(bytes);
    if ((int)c->scr_ptr.size() <= slot) {
      c->scr_ptr.push_back(nullptr);
      c->scr_cap.push_back(0);
    }
    if (c->scr_cap[slot] < bytes) {
      if (c->scr_ptr[slot]) {
        CK(cudaStreamSynchronize(s));
        CK(cudaFree(c->scr_ptr[slot]));
      }
      c->scr_ptr[slot] = nullptr;
      c->scr_cap[slot] = 0;
      size_t cap = bytes + bytes / 2;
      if (cudaMalloc(&c->scr_ptr[slot], cap) != cudaSuccess) {
        cudaGetLastError();
        set_err(c, "scratch allocation failed");
        throw Fail{LC_ENOMEM};
      }
      c->scr_cap[slot] = cap;
    }
    return c->scr_ptr[slot++];
  }

  // capture: buffers the graph references are its own (freed with it)
  void* graph_alloc(size_t bytes) {
    void* p = nullptr;
    if (cudaMalloc(&p, bytes) != cudaSuccess) {
      cudaGetLastError();
      set_err(c, "graph scratch allocation failed");
      throw Fail{LC_ENOMEM};
    }
    c->cap->dev.push_back(p);
    return p;
  }

  // capture: a [host|dev] host pointer becomes a memcpy node read/written at every
  // replay, so it must stay valid -> page-locked memory only
  void require_pinned(const void* p) {
    cudaPointerAttributes at;
    const bool ok = cudaPointerGetAttributes(&at, p) == cudaSuccess && at.type == cudaMemoryTypeHost;
    cudaGetLastError();
    REQUIRE(ok, LC_EINVAL, "while capturing, host data buffers must be page-locked (pinned)");
  }

  // small [host] control array -> device copy inside the argument block
  template <typename T>
  void arg(const T* host, size_t n, const T** dev_out) {
    size_t off = round_up(args.size(), 16);
    args.resize(off + std::max<size_t>(sizeof(T) * n, 1));
    if (n) memcpy(args.data() + off, host, sizeof(T) * n);
    arg_fix.push_back({(const void**)dev_out, off});
  }

  // stage the argument block: one pinned memcpy + one H2D. While capturing, the block
  // is uploaded once into graph-owned memory (its values are constants of the graph).
  void commit() {
    if (args.empty()) return;
    size_t bytes = round_up(args.size(), 16);
    if (c->cap) {
      d_args = (char*)graph_alloc(bytes);
      CK(cudaMemcpyAsync(d_args, args.data(), args.size(), cudaMemcpyHostToDevice, c->side));
      CK(cudaStreamSynchronize(c->side));
      for (auto& f : arg_fix) *f.first = d_args + f.second;
      return;
    }
    // the whole ring is (re)allocated at once, every slot at the largest block seen so far
    // (x2, >= 1 MB): page-locked allocation synchronises with the device and takes ~1 ms+,
    // so it must not happen slot by slot in the steps that follow the first call (calls of
    // different sizes rotate through the ring)
    if (c->pin_cap_max < bytes) {
      const size_t cap = std::max<size_t>(bytes * 2, (size_t)1 << 20);
      for (int q = 0; q < lc_ctx::kPinRing; ++q) {
        if (c->pin_ev_pending[q]) {
          CK(cudaEventSynchronize(c->pin_ev[q]));
          c->pin_ev_pending[q] = false;
        }
        if (c->pin[q]) CK(cudaFreeHost(c->pin[q]));
        c->pin[q] = nullptr;
        c->pin_cap[q] = 0;
        if (cudaHostAlloc(&c->pin[q], cap, cudaHostAllocDefault) != cudaSuccess) {
          cudaGetLastError();
          c->pin[q] = nullptr;
          c->pin_cap_max = 0;
          set_err(c, "pinned staging allocation failed");
          throw Fail{LC_ENOMEM};
        }
        c->pin_cap[q] = cap;
      }
      c->pin_cap_max = cap;
    }
    const int r = c->pin_next;
    c->pin_next = (r + 1) % lc_ctx::kPinRing;
    if (c->pin_ev_pending[r]) {
      CK(cudaEventSynchronize(c->pin_ev[r]));
      c->pin_ev_pending[r] = false;
    }
    memcpy(c->pin[r], args.data(), args.size());
    d_args = (char*)scratch(bytes);
    CK(cudaMemcpyAsync(d_args, c->pin[r], bytes, cudaMemcpyHostToDevice, s));
    CK(cudaEventRecord(c->pin_ev[r], s));
    c->pin_ev_pending[r] = true;
    for (auto& f : arg_fix) *f.first = d_args + f.second;
  }

  // host -> device copy of `bytes`: page-locked sources (and small or captured copies)
  // directly; pageable sources in chunks through the context's pinned staging ring, so the
  // host memcpy of one chunk overlaps the DMA of the previous ones (lc.h "Ownership")
  void upload(void* dst, const void* src, size_t bytes) {
    if (!bytes) return;
    cudaPointerAttributes at;
    const bool pinned = cudaPointerGetAttributes(&at, src) == cudaSuccess && at.type == cudaMemoryTypeHost;
    cudaGetLastError();
    if (pinned || c->cap || bytes < lc_ctx::kStageMin || !c->stage_on) {
      CK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, s));
      return;
    }
    for (size_t off = 0; off < bytes; off += lc_ctx::kStageChunk) {
      const size_t n = std::min(lc_ctx::kStageChunk, bytes - off);
      const int r = c->stg_next;
      c->stg_next = (r + 1) % lc_ctx::kStageRing;
      if (!c->stg[r]) {
        if (cudaHostAlloc(&c->stg[r], lc_ctx::kStageChunk, cudaHostAllocDefault) != cudaSuccess) {
          cudaGetLastError();
          c->stg[r] = nullptr;
          CK(cudaMemcpyAsync((char*)dst + off, (const char*)src + off, bytes - off, cudaMemcpyHostToDevice, s));
          return;
        }
        CK(cudaEventCreateWithFlags(&c->stg_ev[r], cudaEventDisableTiming));
      } else {
        CK(cudaEventSynchronize(c->stg_ev[r]));   // its previous chunk has left the buffer
      }
      memcpy(c->stg[r], (const char*)src + off, n);
      CK(cudaMemcpyAsync((char*)dst + off, c->stg[r], n, cudaMemcpyHostToDevice, s));
      CK(cudaEventRecord(c->stg_ev[r], s));
    }
  }

  // [host|dev] input: device pointer as-is, host data copied to scratch
  template <typename T>
  const T* in(const T* p, size_t n) {
    if (!p || n == 0) return p;
    if (is_device_ptr(c, p)) return p;
    if (c->cap) require_pinned(p);
    T* d = (T*)scratch(sizeof(T) * n);
    upload(d, p, sizeof(T) * n);
    return d;
  }

  // [host|dev] output (copy_in: also an input, e.g. io tables in APPLY)
  template <typename T>
  T* out(T* p, size_t n, bool copy_in = false) {
    if (!p) return nullptr;
    if (n == 0) return p;
    if (is_device_ptr(c, p)) return p;
    if (c->cap) require_pinned(p);
    T* d = (T*)scratch(sizeof(T) * n);
    if (copy_in) CK(cudaMemcpyAsync(d, p, sizeof(T) * n, cudaMemcpyDefault, s));
    outs.push_back({p, d, sizeof(T) * n});
    return d;
  }

  // counters: accumulated in the caller's buffer when it is device memory (no copy),
  // else in scratch with a copy-out at finish; zeroed by the call's first kernel
  unsigned long long* counts(int64_t* user, size_t n) {
    if (user && is_device_ptr(c, user)) return (unsigned long long*)user;
    unsigned long long* d = (unsigned long long*)scratch(sizeof(uint64_t) * n);
    if (user) {
      if (c->cap) require_pinned(user);
      outs.push_back({user, d, sizeof(uint64_t) * n});
    }
    return d;
  }

  void finish() {
    for (auto& o : outs) CK(cudaMemcpyAsync(o.host, o.dev, o.bytes, cudaMemcpyDefault, s));
    CK(cudaGetLastError());
  }
};

// LC_HOST_PROF=1: host-side time of a call's phases to stderr (enqueue-cost analysis)
struct HostProf {
  bool on;
  const char* name;
  std::chrono::steady_clock::time_point t0, t;
  std::string line;
  HostProf(lc_ctx*, const char* n) : on(getenv("LC_HOST_PROF") != nullptr), name(n) {
    if (on) t0 = t = std::chrono::steady_clock::now();
  }
  void mark(const char* what) {
    if (!on) return;
    auto n = std::chrono::steady_clock::now();
    line += std::string(" ") + what + "=" +
            std::to_string(std::chrono::duration<double, std::micro>(n - t).count()).substr(0, 6);
    t = n;
  }
  ~HostProf() {
    if (!on) return;
    auto n = std::chrono::steady_clock::now();
    fprintf(stderr, "[host] %s us:%s total=%.1f\n", name, line.c_str(),
            std::chrono::duration<double, std::micro>(n - t0).count());
  }
};

// Brackets one launch group with timing events when profiling is on.
struct Prof {
  lc_ctx* c;
  int fam;
  cudaStream_t s;
  cudaEvent_t a = nullptr;
  int64_t l0 = 0;
  static cudaEvent_t get(lc_ctx* c) {
    if (!c->ev_pool.empty()) {
      cudaEvent_t e = c->ev_pool.back();
      c->ev_pool.pop_back();
      return e;
    }
    cudaEvent_t e = nullptr;
    if (cudaEventCreate(&e) != cudaSuccess) { cudaGetLastError(); return nullptr; }
    return e;
  }
  Prof(lc_ctx* ctx, int f, cudaStream_t st) : c(ctx), fam(f), s(st) {
    if (!c->prof || c->cap) return;
    a = get(c);
    if (a) cudaEventRecord(a, s);
    l0 = c->launches;
  }
  ~Prof() {
    if (!a) return;
    cudaEvent_t b = get(c);
    if (!b) return;
    cudaEventRecord(b, s);
    c->prof_pending.push_back({fam, a, b, c->launches - l0});
  }
};

void free_graph(lc_graph* g) {
  if (!g) return;
  if (g->exec) cudaGraphExecDestroy(g->exec);
  if (g->graph) cudaGraphDestroy(g->graph);
  for (void* p : g->dev) cudaFree(p);
  cudaGetLastError();
  delete g;
}

// A failed call inside a capture ends (and discards) the capture.
void abort_capture(lc_ctx* c) {
  if (!c->cap) return;
  cudaGraph_t g = nullptr;
  cudaStreamEndCapture(c->cap_stream, &g);
  if (g) cudaGraphDestroy(g);
  cudaGetLastError();
  cudaStreamSynchronize(c->side);
  free_graph(c->cap);
  c->cap = nullptr;
  c->launches = c->cap_launch0;
}

template <typename F>
lc_status guarded(lc_ctx* c, F&& f) {
  if (!c) return LC_EINVAL;
  if (c->broken) {
    return LC_ECUDA;
  }
  try {
    CK(cudaSetDevice(c->device));
    f();
    return LC_OK;
  } catch (const Fail& e) {
    if (c->cap) {
      const std::string m = c->err;
      abort_capture(c);
      c->err = m + " (capture aborted)";
    }
    return e.st;
  } catch (const std::bad_alloc&) {
    abort_capture(c);
    set_err(c, "host allocation failed");
    return LC_ENOMEM;
  }
}

// Calls that may be recorded into a graph must use the capturing stream; the others
// are refused while a capture is open.
void capture_gate(lc_ctx* c, void* stream, bool allowed) {
  if (!c->cap) return;
  REQUIRE(allowed, LC_ESTATE, "call not allowed while a graph capture is open");
  REQUIRE((cudaStream_t)stream == c->cap_stream, LC_ESTATE,
          "while capturing, calls must use the capturing stream");
}

// Fuse epochs: the device counter restarts (and the stamps are cleared) long before
// it could wrap; n = epochs about to be consumed (1 per fuse call, n_fuse per replay).
void epoch_reserve(lc_ctx* c, int64_t n, cudaStream_t s) {
  Store& st = c->st;
  if (c->ep_used + (uint64_t)n >= 0xFFFFFF00ull) {
    CK(cudaMemsetAsync(st.mp_loop_ep, 0, sizeof(uint32_t) * std::max(st.n_mp, 1), s));
    CK(cudaMemsetAsync(st.kf_win_ep, 0, sizeof(uint32_t) * std::max(st.n_kf, 1), s));
    CK(cudaMemsetAsync(st.ep, 0, sizeof(uint32_t) * 2, s));
    c->ep_used = 0;
  }
  c->ep_used += (uint64_t)n;
}

bool params_ok(const lc_match_params& p) {
  return p.th > 0 && p.max_hamming >= 0 && p.max_hamming <= 256 && p.ratio_den >= 0 &&
         (p.ratio_den == 0 || p.ratio_num >= 0);
}

template <typename T>
void dev_alloc(lc_ctx* c, T** p, size_t n) {
  if (*p) cudaFree(*p);
  *p = nullptr;
  if (cudaMalloc((void**)p, std::max<size_t>(sizeof(T) * n, 16)) != cudaSuccess) {
    cudaGetLastError();
    set_err(c, "device store allocation failed");
    throw Fail{LC_ENOMEM};
  }
}

void free_store(Store& st) {
  void* ptrs[] = {st.kf_pose, st.kf_cam, st.kf_fbeg, st.kf_fpad, st.kf_cell, st.fc_uv, st.fc_meta,
                  st.fc_desc, st.feat_mp, st.feat_angle, st.feat_cpos, st.mp_rec, st.mp_flags, st.mp_ref_kf,
                  st.mp_replaced_by, st.mp_nobs, st.mp_corr_ref, st.mp_loop_ep, st.mp_owner,
                  st.kf_S_corr, st.kf_in_win, st.kf_win_ep, st.kf_win_pos, st.mp_vbits,
                  st.kf_dirty, st.ep, st.cams};
  for (void* p : ptrs)
    if (p) cudaFree(p);
  st = Store();
}

void mark_window(lc_ctx* c, int n_w, const int32_t* window) {
  REQUIRE(n_w >= 1 && window, LC_EINVAL, "window must hold at least one keyframe");
  std::vector<char> seen(c->st.n_kf, 0);
  for (int i = 0; i < n_w; ++i) {
    int k = window[i];
    REQUIRE(k >= 0 && k < c->st.n_kf, LC_ERANGE, "window keyframe index out of range");
    REQUIRE(!seen[k], LC_EINVAL, "duplicate keyframe in window");
    seen[k] = 1;
  }
}

int pick_chunk(int64_t total_q) {
  int64_t ch = (total_q + 148 * 4 - 1) / (148 * 4);
  ch = std::max<int64_t>(64, std::min<int64_t>(4096, ch));
  return (int)round_up((size_t)ch, 32);
}

void fill_match_store(lc_ctx* c, MatchArgs& a) {
  Store& st = c->st;
  a.kf_pose = st.kf_pose;
  a.kf_cam = st.kf_cam;
  a.kf_fbeg = st.kf_fbeg;
  a.kf_fpad = st.kf_fpad;
  a.Gs = st.Gs;
  a.kf_cell = st.kf_cell;
  a.fc_uv = st.fc_uv;
  a.fc_meta = st.fc_meta;
  a.fc_desc = st.fc_desc;
  a.feat_mp = st.feat_mp;
  a.mp_rec = st.mp_rec;
  a.mp_flags = st.mp_flags;
  a.cams = st.cams;
  a.cols = st.cols;
  a.rows = st.rows;
  a.G = st.G;
  for (int i = 0; i < LC_MAX_LEVELS; ++i) { a.ocols[i] = st.ocols[i]; a.orows[i] = st.orows[i]; }
  for (int i = 0; i <= LC_MAX_LEVELS; ++i) a.obase[i] = st.obase[i];
  a.n_levels = st.n_levels;
  for (int i = 0; i < LC_MAX_LEVELS; ++i) a.scale[i] = st.scale[i];
}

// Grow a device array from `used` to at least `need` entries (capacity `cap` -> max(need,
// 1.5 cap)), keeping its first `used` entries (LC_UPLOAD_APPEND).
template <typename T>
void grow(lc_ctx* c, T** p, int64_t used, int64_t need, int64_t cap, int64_t new_cap, cudaStream_t s) {
  if (need <= cap && *p) return;
  T* q = nullptr;
  if (cudaMalloc((void**)&q, std::max<size_t>(sizeof(T) * (size_t)new_cap, 16)) != cudaSuccess) {
    cudaGetLastError();
    set_err(c, "device store allocation failed");
    throw Fail{LC_ENOMEM};
  }
  if (used > 0 && *p) CK(cudaMemcpyAsync(q, *p, sizeof(T) * (size_t)used, cudaMemcpyDeviceToDevice, s));
  CK(cudaStreamSynchronize(s));
  if (*p) cudaFree(*p);
  *p = q;
}

}  // namespace

// ============================================================================
extern "C" {

lc_status lc_create(lc_ctx** out, int32_t device) {
  if (!out) return LC_EINVAL;
  *out = nullptr;
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess || device < 0 || device >= n) {
    cudaGetLastError();
    g_create_err = "no such CUDA device";
    return LC_ECUDA;
  }
  cudaDeviceProp prop;
  if (cudaGetDeviceProperties(&prop, device) != cudaSuccess || prop.major != 10) {
    cudaGetLastError();
    g_create_err = "liblc is built for sm_100a (B200); device is sm_" +
                   std::to_string(prop.major) + std::to_string(prop.minor);
    return LC_ECUDA;
  }
  lc_ctx* c = new (std::nothrow) lc_ctx();
  if (!c) return LC_ENOMEM;
  c->device = device;
  if (const char* e = getenv("LC_SOLE")) c->sole_mode = atoi(e);   // test knob: 0 forbid, 1 force, 2 k_match_sole
  if (const char* e = getenv("LC_STAGE")) c->stage_on = atoi(e) != 0;   // pageable inputs via the staging ring
  if (const char* e = getenv("LC_PIPE_MIN")) c->pipe_min = atoll(e);   // test knob: force / forbid the pipelined list upload
  bool ok = cudaSetDevice(device) == cudaSuccess;
  for (int r = 0; ok && r < lc_ctx::kPinRing; ++r)
    ok = cudaEventCreateWithFlags(&c->pin_ev[r], cudaEventDisableTiming) == cudaSuccess;
  ok = ok && cudaStreamCreateWithFlags(&c->side, cudaStreamNonBlocking) == cudaSuccess;
  for (int r = 0; ok && r <= lc_ctx::kPipe; ++r)
    ok = cudaEventCreateWithFlags(&c->pipe_ev[r], cudaEventDisableTiming) == cudaSuccess;
  if (!ok) {
    for (int r = 0; r < lc_ctx::kPinRing; ++r)
      if (c->pin_ev[r]) cudaEventDestroy(c->pin_ev[r]);
    cudaGetLastError();
    g_create_err = "CUDA context setup failed";
    delete c;
    return LC_ECUDA;
  }
  *out = c;
  return LC_OK;
}

lc_status lc_destroy(lc_ctx* c) {
  if (!c) return LC_EINVAL;
  cudaSetDevice(c->device);
  abort_capture(c);
  cudaDeviceSynchronize();
  free_store(c->st);
  for (void* p : c->scr_ptr)
    if (p) cudaFree(p);
  for (int r = 0; r < lc_ctx::kPinRing; ++r) {
    if (c->pin[r]) cudaFreeHost(c->pin[r]);
    if (c->pin_ev[r]) cudaEventDestroy(c->pin_ev[r]);
  }
  for (int r = 0; r < lc_ctx::kStageRing; ++r) {
    if (c->stg[r]) cudaFreeHost(c->stg[r]);
    if (c->stg_ev[r]) cudaEventDestroy(c->stg_ev[r]);
  }
  if (c->sv) cudaFree(c->sv);
  if (c->side) cudaStreamDestroy(c->side);
  for (int r = 0; r <= lc_ctx::kPipe; ++r)
    if (c->pipe_ev[r]) cudaEventDestroy(c->pipe_ev[r]);
  for (auto& r : c->prof_pending) { cudaEventDestroy(r.a); cudaEventDestroy(r.b); }
  for (cudaEvent_t e : c->ev_pool) cudaEventDestroy(e);
  cudaGetLastError();
  delete c;
  return LC_OK;
}

const char* lc_last_error(const lc_ctx* c) { return c ? c->err.c_str() : g_create_err.c_str(); }

int64_t lc_kernel_launches(const lc_ctx* c) { return c ? c->launches : 0; }

// ----------------------------------------------------------------------------
// CUDA-graph capture of a sequence of calls
lc_status lc_graph_begin(lc_ctx* c, void* stream) {
  return guarded(c, [&] {
    REQUIRE(!c->cap, LC_ESTATE, "a graph capture is already open");
    REQUIRE(c->has_map, LC_ESTATE, "no map uploaded");
    REQUIRE(stream != nullptr, LC_EINVAL, "capture needs a non-default stream");
    lc_graph* g = new lc_graph();
    g->ctx = c;
    cudaError_t e = cudaStreamBeginCapture((cudaStream_t)stream, cudaStreamCaptureModeRelaxed);
    if (e != cudaSuccess) {
      cudaGetLastError();
      delete g;
      set_err(c, std::string("cudaStreamBeginCapture failed: ") + cudaGetErrorString(e));
      throw Fail{LC_ECUDA};
    }
    c->cap = g;
    c->cap_stream = (cudaStream_t)stream;
    c->cap_launch0 = c->launches;
  });
}

lc_status lc_graph_end(lc_ctx* c, void* stream, lc_graph** out) {
  return guarded(c, [&] {
    REQUIRE(out, LC_EINVAL, "null out");
    *out = nullptr;
    REQUIRE(c->cap, LC_ESTATE, "no graph capture open");
    REQUIRE((cudaStream_t)stream == c->cap_stream, LC_ESTATE, "end on a different stream");
    lc_graph* g = c->cap;
    c->cap = nullptr;
    g->launches = c->launches - c->cap_launch0;
    c->launches = c->cap_launch0;   // recorded, not executed
    cudaError_t e = cudaStreamEndCapture(c->cap_stream, &g->graph);
    if (e == cudaSuccess) e = cudaGraphInstantiate(&g->exec, g->graph, 0);
    if (e != cudaSuccess) {
      cudaGetLastError();
      free_graph(g);
      set_err(c, std::string("graph capture failed: ") + cudaGetErrorString(e));
      throw Fail{LC_ECUDA};
    }
    *out = g;
  });
}

lc_status lc_graph_launch(lc_ctx* c, lc_graph* g, void* stream) {
  return guarded(c, [&] {
    REQUIRE(g && g->ctx == c, LC_EINVAL, "graph does not belong to this context");
    capture_gate(c, stream, false);
    if (g->n_fuse) epoch_reserve(c, g->n_fuse, (cudaStream_t)stream);
    CK(cudaGraphLaunch(g->exec, (cudaStream_t)stream));
    c->launches += g->launches;
  });
}

lc_status lc_graph_destroy(lc_ctx* c, lc_graph* g) {
  if (!c || !g || g->ctx != c) return LC_EINVAL;
  cudaSetDevice(c->device);
  cudaDeviceSynchronize();
  free_graph(g);
  return LC_OK;
}

lc_status lc_profile_enable(lc_ctx* c, int32_t on) {
  return guarded(c, [&] {
    capture_gate(c, nullptr, false);
    for (auto& r : c->prof_pending) { c->ev_pool.push_back(r.a); c->ev_pool.push_back(r.b); }
    c->prof_pending.clear();
    if (on) {
      for (int i = 0; i < LC_NPROF; ++i) { c->prof_ms[i] = 0.0; c->prof_n[i] = 0; }
    }
    c->prof = on != 0;
  });
}

lc_status lc_profile_read(lc_ctx* c, double* ms, int64_t* launches) {
  return guarded(c, [&] {
    capture_gate(c, nullptr, false);
    for (auto& r : c->prof_pending) {
      CK(cudaEventSynchronize(r.b));
      float t = 0.f;
      CK(cudaEventElapsedTime(&t, r.a, r.b));
      c->prof_ms[r.fam] += t;
      c->prof_n[r.fam] += r.launches;
      c->ev_pool.push_back(r.a);
      c->ev_pool.push_back(r.b);
    }
    c->prof_pending.clear();
    for (int i = 0; i < LC_NPROF; ++i) {
      if (ms) ms[i] = c->prof_ms[i];
      if (launches) launches[i] = c->prof_n[i];
    }
  });
}

// ----------------------------------------------------------------------------
lc_status lc_upload_map(lc_ctx* c, const lc_map_view* m, const lc_camera* cams, int32_t n_cams,
                        const lc_map_params* prm, int32_t flags, void* stream) {
  return guarded(c, [&] {
    capture_gate(c, stream, false);
    const bool append = (flags & LC_UPLOAD_APPEND) != 0;
    REQUIRE(flags == LC_UPLOAD_REPLACE || flags == LC_UPLOAD_APPEND, LC_EINVAL, "bad flags");
    REQUIRE(m, LC_EINVAL, "null map");
    REQUIRE(!append || c->has_map, LC_ESTATE, "LC_UPLOAD_APPEND before any map upload");
    if (!append) {
      REQUIRE(cams && prm && n_cams >= 1, LC_EINVAL, "null map/camera/params");
      REQUIRE(prm->n_levels >= 1 && prm->n_levels <= LC_MAX_LEVELS, LC_EINVAL, "n_levels out of range");
      REQUIRE(prm->scale_factor > 1.0, LC_EINVAL, "scale_factor must be > 1");
      REQUIRE(prm->grid_cols >= 1 && prm->grid_rows >= 1 && prm->grid_cols <= 1024 &&
                  prm->grid_rows <= 1024 && prm->grid_cols * prm->grid_rows <= 16384,
              LC_EINVAL, "grid size out of range");
      for (int i = 0; i < n_cams; ++i) {
        const lc_camera& k = cams[i];
        REQUIRE(k.model == 0 || k.model == 1, LC_EINVAL, "camera model must be 0 or 1");
        REQUIRE(k.max_x > k.min_x && k.max_y > k.min_y, LC_EINVAL, "empty camera bounds");
      }
    }
    REQUIRE(m->n_kf >= 0 && m->n_feat >= 0 && m->n_mp >= 0, LC_EINVAL, "negative sizes");
    const bool need = m->n_kf > 0;
    REQUIRE(!need || (m->kf_pose && m->kf_cam && m->kf_feat_begin), LC_EINVAL, "null keyframe arrays");
    REQUIRE(m->n_feat == 0 || (m->feat_uv && m->feat_octave && m->feat_angle && m->feat_desc &&
                               m->feat_mp), LC_EINVAL, "null feature arrays");
    REQUIRE(m->n_mp == 0 || (m->mp_pos && m->mp_normal && m->mp_max_dist && m->mp_desc &&
                             m->mp_angle && m->mp_ref_kf && m->mp_flags), LC_EINVAL, "null map-point arrays");
    Call call(c, stream);
    cudaStream_t s = call.s;
    // host copy of the (new) keyframes' CSR (validation + launch configuration)
    std::vector<int32_t> fbeg(m->n_kf + 1, 0);
    if (m->n_kf > 0) {
      if (is_device_ptr(c, m->kf_feat_begin)) {
        CK(cudaMemcpyAsync(fbeg.data(), m->kf_feat_begin, sizeof(int32_t) * (m->n_kf + 1),
                           cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
      } else {
        memcpy(fbeg.data(), m->kf_feat_begin, sizeof(int32_t) * (m->n_kf + 1));
      }
    }
    REQUIRE(fbeg[0] == 0 && fbeg[m->n_kf] == m->n_feat, LC_EINVAL, "kf_feat_begin must span [0, n_feat]");
    int max_F = 0;
    for (int k = 0; k < m->n_kf; ++k) {
      REQUIRE(fbeg[k + 1] >= fbeg[k], LC_EINVAL, "kf_feat_begin not monotone");
      max_F = std::max(max_F, fbeg[k + 1] - fbeg[k]);
    }
    REQUIRE(max_F <= LC_MAX_FEAT_PER_KF, LC_ECAPACITY, "keyframe exceeds LC_MAX_FEAT_PER_KF features");
    CK(cudaStreamSynchronize(s));
    Store& st = c->st;
    // old extents (APPEND) / zero (REPLACE); the new entries go to [kf0, ...), [f0, ...), [mp0, ...)
    int kf0 = 0, f0 = 0, mp0 = 0;
    int64_t fp0 = 0;
    if (append) {
      kf0 = st.n_kf; f0 = st.n_feat; mp0 = st.n_mp; fp0 = st.n_fpad;
      REQUIRE((int64_t)kf0 + m->n_kf < (1LL << 31) && (int64_t)f0 + m->n_feat < (1LL << 31) &&
                  (int64_t)mp0 + m->n_mp < (1LL << 31), LC_ECAPACITY, "store index space exhausted");
    } else {
      free_store(st);
      st.n_cams = n_cams;
      st.n_levels = prm->n_levels; st.cols = prm->grid_cols; st.rows = prm->grid_rows;
      {   // per-octave grids: octave o coarsened by scale_factor^o (its keypoints are that much sparser)
        double f = 1.0;
        st.obase[0] = 0;
        for (int o = 0; o < LC_MAX_LEVELS; ++o) {
          st.ocols[o] = std::max(1, (int)std::ceil(st.cols / f - 1e-9));
          st.orows[o] = std::max(1, (int)std::ceil(st.rows / f - 1e-9));
          st.obase[o + 1] = st.obase[o] + (o < st.n_levels ? st.ocols[o] * st.orows[o] : 0);
          f *= prm->scale_factor;
        }
      }
      st.G = st.obase[st.n_levels];
      REQUIRE(st.G <= 24576, LC_EINVAL, "grid too fine: more than 24576 cells over the octave grids");
      st.Gs = (int32_t)round_up((size_t)st.G + 1, 8);
      st.scale[0] = 1.0;
      for (int n = 1; n < LC_MAX_LEVELS; ++n) st.scale[n] = st.scale[n - 1] * prm->scale_factor;
      st.h_fbeg.assign(1, 0);
      st.h_in_win.clear();
      c->ep_used = 0;
    }
    c->has_map = false;
    c->has_saved = false;
    const int64_t NK = (int64_t)kf0 + m->n_kf, NF = (int64_t)f0 + m->n_feat, NM = (int64_t)mp0 + m->n_mp;
    // padded (multiple-of-4) per-keyframe blocks of the cell-major feature arrays
    std::vector<int32_t> fpad_new(m->n_kf + 1, 0);
    fpad_new[0] = (int32_t)fp0;
    for (int k = 0; k < m->n_kf; ++k)
      fpad_new[k + 1] = fpad_new[k] + (int32_t)round_up((size_t)(fbeg[k + 1] - fbeg[k]), 4);
    const int64_t NPad = fpad_new[m->n_kf];
    const int64_t NP = NPad + 4;
    // capacities: exact for REPLACE, geometric for APPEND
    auto ncap = [&](int64_t need_n, int64_t cap) { return append ? std::max<int64_t>(need_n, cap + cap / 2) : need_n; };
    const int64_t ck = ncap(NK, st.cap_kf), cf = ncap(NF, st.cap_feat), cp = ncap(NP, st.cap_fpad), cm = ncap(NM, st.cap_mp);
    const bool gk = NK > st.cap_kf || !append, gf = NF > st.cap_feat || !append, gp = NP > st.cap_fpad || !append,
               gm = NM > st.cap_mp || !append;
    const int64_t uk = append ? kf0 : 0, uf = append ? f0 : 0, up = append ? fp0 + 4 : 0, um = append ? mp0 : 0;
    if (gk) {
      grow(c, &st.kf_pose, 13 * uk, 13 * NK, 0, 13 * ck, s);
      grow(c, &st.kf_cam, uk, NK, 0, ck, s);
      grow(c, &st.kf_fbeg, uk + 1, NK + 1, 0, ck + 1, s);
      grow(c, &st.kf_fpad, uk + 1, NK + 1, 0, ck + 1, s);
      grow(c, &st.kf_cell, uk * st.Gs, NK * st.Gs, 0, ck * st.Gs, s);
      grow(c, &st.kf_S_corr, 13 * uk, 13 * NK, 0, 13 * ck, s);
      grow(c, &st.kf_in_win, uk, NK, 0, ck, s);
      grow(c, &st.kf_win_ep, uk, NK, 0, ck, s);
      grow(c, &st.kf_win_pos, uk, NK, 0, ck, s);
      grow(c, &st.kf_dirty, uk + 1, NK + 1, 0, ck + 1, s);
      st.cap_kf = ck;
    }
    if (gf) {
      grow(c, &st.feat_mp, uf, NF, 0, cf, s);
      grow(c, &st.feat_angle, uf, NF, 0, cf, s);
      grow(c, &st.feat_cpos, uf, NF, 0, cf, s);
      st.cap_feat = cf;
    }
    if (gp) {
      grow(c, &st.fc_uv, up, NP, 0, cp, s);
      grow(c, &st.fc_meta, up, NP, 0, cp, s);
      grow(c, &st.fc_desc, 2 * up, 2 * NP, 0, 2 * cp, s);
      st.cap_fpad = cp;
    }
    if (gm) {
      grow(c, &st.mp_rec, um, NM, 0, cm, s);
      grow(c, &st.mp_flags, um, NM, 0, cm, s);
      grow(c, &st.mp_ref_kf, um, NM, 0, cm, s);
      grow(c, &st.mp_replaced_by, um, NM, 0, cm, s);
      grow(c, &st.mp_nobs, um, NM, 0, cm, s);
      grow(c, &st.mp_corr_ref, um, NM, 0, cm, s);
      grow(c, &st.mp_loop_ep, um, NM, 0, cm, s);
      grow(c, &st.mp_owner, um, NM, 0, cm, s);
      grow(c, &st.mp_vbits, append ? (um + 31) / 32 : 0, (NM + 31) / 32 + 1, 0, (cm + 31) / 32 + 1, s);
      st.cap_mp = cm;
    }
    if (!append) {
      dev_alloc(c, &st.ep, 2);
      dev_alloc(c, &st.cams, n_cams);
      std::vector<DevCam> dc(n_cams);
      for (int i = 0; i < n_cams; ++i) {
        const lc_camera& k = cams[i];
        DevCam& d = dc[i];
        memset(&d, 0, sizeof(d));
        d.model = k.model; d.cols = st.cols; d.rows = st.rows;
        d.fx = k.fx; d.fy = k.fy; d.cx = k.cx; d.cy = k.cy;
        for (int j = 0; j < 4; ++j) d.k[j] = k.k[j];
        d.min_x = k.min_x; d.max_x = k.max_x; d.min_y = k.min_y; d.max_y = k.max_y;
        for (int o = 0; o < LC_MAX_LEVELS; ++o) {
          d.cell_sx[o] = (double)st.ocols[o] / (k.max_x - k.min_x);
          d.cell_sy[o] = (double)st.orows[o] / (k.max_y - k.min_y);
        }
      }
      CK(cudaMemcpyAsync(st.cams, dc.data(), sizeof(DevCam) * n_cams, cudaMemcpyHostToDevice, s));
      CK(cudaMemsetAsync(st.ep, 0, sizeof(uint32_t) * 2, s));
    }
    st.n_kf = (int32_t)NK; st.n_feat = (int32_t)NF; st.n_mp = (int32_t)NM;
    st.n_fpad = NPad;
    st.max_F = std::max(st.max_F, max_F);
    for (int k = 0; k < m->n_kf; ++k) st.h_fbeg.push_back(f0 + fbeg[k + 1]);
    st.h_in_win.resize(NK, 0);
    // new keyframe / feature / map-point entries
    const size_t nk = m->n_kf, nf = m->n_feat, nm = m->n_mp;
    std::vector<int32_t> fbeg_g(nk + 1), fpad_g(nk + 1);
    for (size_t k = 0; k <= nk; ++k) { fbeg_g[k] = f0 + fbeg[k]; fpad_g[k] = fpad_new[k]; }
    CK(cudaMemsetAsync(st.kf_cell + (size_t)kf0 * st.Gs, 0, sizeof(uint16_t) * nk * st.Gs, s));
    CK(cudaMemsetAsync(st.fc_uv + fp0, 0, sizeof(float2) * (size_t)(NP - fp0), s));
    CK(cudaMemsetAsync(st.fc_meta + fp0, 0, sizeof(uint32_t) * (size_t)(NP - fp0), s));
    if (nk) {
      CK(cudaMemcpyAsync(st.kf_fpad + kf0, fpad_g.data(), sizeof(int32_t) * (nk + 1), cudaMemcpyHostToDevice, s));
      CK(cudaMemcpyAsync(st.kf_fbeg + kf0, fbeg_g.data(), sizeof(int32_t) * (nk + 1), cudaMemcpyHostToDevice, s));
    }
    auto copy_in = [&](void* dst, const void* src, size_t bytes) {
      if (!bytes) return;
      if (is_device_ptr(c, src)) CK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToDevice, s));
      else call.upload(dst, src, bytes);
    };
    copy_in(st.kf_pose + 13 * (size_t)kf0, m->kf_pose, sizeof(double) * 13 * nk);
    copy_in(st.kf_cam + kf0, m->kf_cam, sizeof(int32_t) * nk);
    copy_in(st.feat_mp + f0, m->feat_mp, sizeof(int32_t) * nf);
    copy_in(st.feat_angle + f0, m->feat_angle, sizeof(float) * nf);
    copy_in(st.mp_flags + mp0, m->mp_flags, nm);
    copy_in(st.mp_ref_kf + mp0, m->mp_ref_kf, sizeof(int32_t) * nm);
    if (nk) {
      CK(cudaMemsetAsync(st.kf_S_corr + 13 * (size_t)kf0, 0, sizeof(double) * 13 * nk, s));
      CK(cudaMemsetAsync(st.kf_in_win + kf0, 0, sizeof(int32_t) * nk, s));
      CK(cudaMemsetAsync(st.kf_win_ep + kf0, 0, sizeof(uint32_t) * nk, s));
    }
    // raw SoA inputs the packing kernels read (device pointers used in place)
    const float* pos = call.in(m->mp_pos, 3 * nm);
    const float* nrm = call.in(m->mp_normal, 3 * nm);
    const float* dmx = call.in(m->mp_max_dist, nm);
    const uint8_t* mdesc = call.in(m->mp_desc, 32 * nm);
    const float* ang = call.in(m->mp_angle, nm);
    const float* fuv = call.in(m->feat_uv, 2 * nf);
    const uint8_t* foct = call.in(m->feat_octave, nf);
    const uint8_t* fdesc = call.in(m->feat_desc, 32 * nf);
    uint32_t* d_errs = (uint32_t*)call.scratch(64);
    CK(cudaMemsetAsync(d_errs, 0, 64, s));
    {
      Prof pr(c, LC_PROF_UPLOAD, s);
      CK(launch_upload_pack(c, kf0, f0, mp0, pos, nrm, dmx, mdesc, ang, fuv, foct, fdesc, d_errs, s));
    }
    uint32_t errs[16];
    CK(cudaMemcpyAsync(errs, d_errs, 64, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    REQUIRE(errs[0] == 0, LC_ERANGE, "feature octave >= n_levels");
    REQUIRE(errs[1] == 0, LC_ERANGE, "feat_mp out of range");
    REQUIRE(errs[2] == 0, LC_ERANGE, "mp_ref_kf out of range");
    REQUIRE(errs[3] == 0, LC_ERANGE, "kf_cam out of range");
    c->mp_lo = 0;   // lc_set_point_range: back to all points
    c->mp_hi = -1;
    c->has_map = true;
  });
}

lc_status lc_download_map(lc_ctx* c, const lc_map_state* o, void* stream) {
  return guarded(c, [&] {
    capture_gate(c, stream, false);
    REQUIRE(c->has_map, LC_ESTATE, "no map uploaded");
    REQUIRE(o, LC_EINVAL, "null output struct");
    Call call(c, stream);
    Store& st = c->st;
    auto copy_out = [&](void* dst, const void* src, size_t bytes) {
      if (dst && bytes) CK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDefault, call.s));
    };
    copy_out(o->kf_pose, st.kf_pose, sizeof(double) * 13 * st.n_kf);
    copy_out(o->feat_mp, st.feat_mp, sizeof(int32_t) * st.n_feat);
    copy_out(o->mp_flags, st.mp_flags, st.n_mp);
    copy_out(o->mp_replaced_by, st.mp_replaced_by, sizeof(int32_t) * st.n_mp);
    copy_out(o->mp_nobs, st.mp_nobs, sizeof(int32_t) * st.n_mp);
    if (o->mp_pos && st.n_mp) {
      float* d = call.out(o->mp_pos, 3 * (size_t)st.n_mp);
      CK(launch_download_pos(c, d, call.s));
    }
    if ((o->mp_normal || o->mp_max_dist || o->mp_desc) && st.n_mp) {
      float* dn = call.out(o->mp_normal, 3 * (size_t)st.n_mp);
      float* dd = call.out(o->mp_max_dist, (size_t)st.n_mp);
      uint8_t* de = call.out(o->mp_desc, 32 * (size_t)st.n_mp);
      CK(launch_download_rec(c, dn, dd, de, call.s));
    }
    call.finish();
  });
}

lc_status lc_refresh_mappoints(lc_ctx* c, int32_t n, const int32_t* mp_idx, int32_t what,
                               int64_t* out_counts, void* stream) {
  return guarded(c, [&] {
    capture_gate(c, stream, true);
    REQUIRE(c->has_map, LC_ESTATE, "no map uploaded");
    REQUIRE(what >= 1 && what <= (LC_REFRESH_DESC | LC_REFRESH_NORMAL), LC_EINVAL, "bad what");
    REQUIRE(mp_idx == nullptr || n >= 0, LC_EINVAL, "n < 0");
    Store& st = c->st;
    Call call(c, stream);
    const int n_sel = mp_idx ? n : st.n_mp;
    const int32_t* d_idx = mp_idx ? call.in(mp_idx, (size_t)n_sel) : nullptr;
    const int nb = (st.n_mp + LC_NTHREADS * 8 - 1) / (LC_NTHREADS * 8);
    int32_t* d_obeg = (int32_t*)call.scratch(sizeof(int32_t) * ((size_t)st.n_mp + 1));
    int32_t* d_cursor = (int32_t*)call.scratch(sizeof(int32_t) * std::max<size_t>(st.n_mp, 1));
    int32_t* d_bsum = (int32_t*)call.scratch(sizeof(int32_t) * std::max(nb, 1));
    int32_t* d_obs = (int32_t*)call.scratch(sizeof(int32_t) * std::max<size_t>(st.n_feat, 1));
    int32_t* d_obs_kf = (int32_t*)call.scratch(sizeof(int32_t) * std::max<size_t>(st.n_feat, 1));
    unsigned long long* cnt = (unsigned long long*)call.scratch(sizeof(uint64_t) * LC_NCOUNT);
    CK(cudaMemsetAsync(cnt, 0, sizeof(uint64_t) * LC_NCOUNT, call.s));
    {
      Prof pr(c, LC_PROF_REFRESH, call.s);
      CK(launch_refresh(c, n_sel, d_idx, what, d_obeg, d_cursor, d_bsum, d_obs, d_obs_kf, cnt, call.s));
    }
    if (out_counts) {
      int64_t* d = call.out(out_counts, LC_NCOUNT);
      CK(cudaMemcpyAsync(d, cnt, sizeof(uint64_t) * LC_NCOUNT, cudaMemcpyDeviceToDevice, call.s));
    }
    call.finish();
  });
}

lc_status lc_update_connections(lc_ctx* c, int32_t n, const int32_t* kf_idx, int32_t th,
                                int32_t max_edges, int32_t* out_n, int32_t* out_kf, int32_t* out_w,
                                int64_t* out_counts, void* stream) {
  return guarded(c, [&] {
    capture_gate(c, stream, true);
    REQUIRE(c->has_map, LC_ESTATE, "no map uploaded");
    REQUIRE(kf_idx == nullptr || n >= 0, LC_EINVAL, "n < 0");
    REQUIRE(max_edges >= 0 && th >= 1, LC_EINVAL, "bad max_edges / th");
    REQUIRE(c->st.n_kf <= connections_max_kf(), LC_EINVAL, "too many keyframes for the shared weight array");
    REQUIRE(out_n, LC_EINVAL, "null out_n");
    REQUIRE(max_edges == 0 || (out_kf && out_w), LC_EINVAL, "null out_kf / out_w");
    Store& st = c->st;
    Call call(c, stream);
    const int n_sel = kf_idx ? n : st.n_kf;
    const int32_t* d_idx = kf_idx ? call.in(kf_idx, (size_t)n_sel) : nullptr;
    int32_t* d_n = call.out(out_n, (size_t)n_sel);
    int32_t* d_kf = max_edges ? call.out(out_kf, (size_t)n_sel * max_edges, true) : nullptr;
    int32_t* d_w = max_edges ? call.out(out_w, (size_t)n_sel * max_edges, true) : nullptr;
    int32_t* d_obeg = (int32_t*)call.scratch(sizeof(int32_t) * ((size_t)st.n_mp + 1));
    int32_t* d_cursor = (int32_t*)call.scratch(sizeof(int32_t) * std::max<size_t>(st.n_mp, 1));
    int32_t* d_bsum = (int32_t*)call.scratch(sizeof(int32_t) * std::max(obs_scan_blocks(st.n_mp), 1));
    int32_t* d_obs = (int32_t*)call.scratch(sizeof(int32_t) * std::max<size_t>(st.n_feat, 1));
    int32_t* d_obs_kf = (int32_t*)call.scratch(sizeof(int32_t) * std::max<size_t>(st.n_feat, 1));
    uint8_t* d_first = (uint8_t*)call.scratch(std::max<size_t>(st.n_feat, 1));
    unsigned long long* cnt = call.counts(out_counts, LC_NCOUNT);
    CK(cudaMemsetAsync(cnt, 0, sizeof(uint64_t) * LC_NCOUNT, call.s));
    {
      Prof pr(c, LC_PROF_CONN, call.s);
      CK(launch_obs_lists(c, d_obeg, d_cursor, d_bsum, d_obs, d_obs_kf, call.s));
      CK(launch_connections(c, n_sel, d_idx, th, max_edges, d_obeg, d_obs, d_obs_kf, d_first, d_n, d_kf,
                            d_w, cnt, call.s));
    }
    call.finish();
  });
}

lc_status lc_sim3_ransac(lc_ctx* c, int32_t n_prob, const int32_t* prob_begin, const double* P1,
                         const double* P2, const float* uv1, const float* uv2, const float* sigma2_1,
                         const float* sigma2_2, const int32_t* cam1, const int32_t* cam2,
                         const int32_t* samples, int32_t n_iter, double chi2, int32_t fix_scale,
                         int32_t refit, lc_sim3* out_S12, int32_t* out_inliers, uint8_t* out_mask,
                         int64_t* out_counts, void* stream) {
  return guarded(c, [&] {
    capture_gate(c, stream, true);
    REQUIRE(c->has_map, LC_ESTATE, "no map uploaded (cameras)");
    REQUIRE(n_prob >= 0 && n_iter >= 0, LC_EINVAL, "bad sizes");
    REQUIRE(n_prob == 0 || (prob_begin && cam1 && cam2 && out_S12 && out_inliers), LC_EINVAL, "null argument");
    Call call(c, stream);
    int64_t n_corr = 0;
    if (n_prob > 0) {
      REQUIRE(prob_begin[0] == 0, LC_EINVAL, "prob_begin[0] must be 0");
      for (int b = 0; b < n_prob; ++b) {
        REQUIRE(prob_begin[b + 1] >= prob_begin[b], LC_EINVAL, "prob_begin not monotone");
        REQUIRE(cam1[b] >= 0 && cam1[b] < c->st.n_cams && cam2[b] >= 0 && cam2[b] < c->st.n_cams, LC_EINVAL,
                "camera index out of range");
      }
      n_corr = prob_begin[n_prob];
      REQUIRE(n_corr == 0 || (P1 && P2 && uv1 && uv2 && sigma2_1 && sigma2_2 && out_mask), LC_EINVAL,
              "null correspondence array");
      REQUIRE(n_iter == 0 || samples, LC_EINVAL, "null samples");
    }
    const int32_t *d_pb = nullptr, *d_c1 = nullptr, *d_c2 = nullptr;
    if (n_prob > 0) {
      call.arg(prob_begin, (size_t)n_prob + 1, &d_pb);
      call.arg(cam1, (size_t)n_prob, &d_c1);
      call.arg(cam2, (size_t)n_prob, &d_c2);
      call.commit();
    }
    const double* dP1 = call.in(P1, 3 * (size_t)n_corr);
    const double* dP2 = call.in(P2, 3 * (size_t)n_corr);
    const float* du1 = call.in(uv1, 2 * (size_t)n_corr);
    const float* du2 = call.in(uv2, 2 * (size_t)n_corr);
    const float* ds1 = call.in(sigma2_1, (size_t)n_corr);
    const float* ds2 = call.in(sigma2_2, (size_t)n_corr);
    const int32_t* dsm = call.in(samples, 3 * (size_t)n_prob * n_iter);
    double* dS = (double*)call.out((double*)out_S12, 13 * (size_t)n_prob);
    int32_t* dI = call.out(out_inliers, (size_t)n_prob);
    uint8_t* dM = call.out(out_mask, (size_t)n_corr);
    unsigned long long* cnt = call.counts(out_counts, LC_NCOUNT);
    CK(cudaMemsetAsync(cnt, 0, sizeof(uint64_t) * LC_NCOUNT, call.s));
    {
      Prof pr(c, LC_PROF_RANSAC, call.s);
      CK(launch_ransac(c, n_prob, d_pb, dP1, dP2, du1, du2, ds1, ds2, d_c1, d_c2, dsm, n_iter, chi2, fix_scale,
                       refit, dS, dI, dM, cnt, call.s));
    }
    call.finish();
  });
}

lc_status lc_sim3_refine(lc_ctx* c, int32_t n_prob, const int32_t* prob_begin, const double* P1,
                         const double* P2, const float* uv1, const float* uv2, const float* sigma2_1,
                         const float* sigma2_2, const int32_t* cam1, const int32_t* cam2,
                         const lc_sim3* S_init, int32_t max_iter, double th2, double lambda,
                         lc_sim3* out_S, int32_t* out_inliers, uint8_t* out_mask, int64_t* out_counts,
                         void* stream) {
  return guarded(c, [&] {
    capture_gate(c, stream, true);
    REQUIRE(c->has_map, LC_ESTATE, "no map uploaded (cameras)");
    REQUIRE(n_prob >= 0 && max_iter >= 0 && th2 > 0.0 && lambda >= 0.0, LC_EINVAL, "bad sizes / parameters");
    REQUIRE(n_prob == 0 || (prob_begin && cam1 && cam2 && S_init && out_S && out_inliers), LC_EINVAL,
            "null argument");
    Call call(c, stream);
    int64_t n_corr = 0;
    if (n_prob > 0) {
      REQUIRE(prob_begin[0] == 0, LC_EINVAL, "prob_begin[0] must be 0");
      for (int b = 0; b < n_prob; ++b) {
        REQUIRE(prob_begin[b + 1] >= prob_begin[b], LC_EINVAL, "prob_begin not monotone");
        REQUIRE(cam1[b] >= 0 && cam1[b] < c->st.n_cams && cam2[b] >= 0 && cam2[b] < c->st.n_cams, LC_EINVAL,
                "camera index out of range");
      }
      n_corr = prob_begin[n_prob];
      REQUIRE(n_corr == 0 || (P1 && P2 && uv1 && uv2 && sigma2_1 && sigma2_2 && out_mask), LC_EINVAL,
              "null correspondence array");
    }
    const int32_t *d_pb = nullptr, *d_c1 = nullptr, *d_c2 = nullptr;
    if (n_prob > 0) {
      call.arg(prob_begin, (size_t)n_prob + 1, &d_pb);
      call.arg(cam1, (size_t)n_prob, &d_c1);
      call.arg(cam2, (size_t)n_prob, &d_c2);
      call.commit();
    }
    const double* dP1 = call.in(P1, 3 * (size_t)n_corr);
    const double* dP2 = call.in(P2, 3 * (size_t)n_corr);
    const float* du1 = call.in(uv1, 2 * (size_t)n_corr);
    const float* du2 = call.in(uv2, 2 * (size_t)n_corr);
    const float* ds1 = call.in(sigma2_1, (size_t)n_corr);
    const float* ds2 = call.in(sigma2_2, (size_t)n_corr);
    const double* dS0 = call.in((const double*)S_init, 13 * (size_t)n_prob);
    double* dS = (double*)call.out((double*)out_S, 13 * (size_t)n_prob);
    int32_t* dI = call.out(out_inliers, (size_t)n_prob);
    uint8_t* dM = call.out(out_mask, (size_t)n_corr);
    unsigned long long* cnt = call.counts(out_counts, LC_NCOUNT);
    CK(cudaMemsetAsync(cnt, 0, sizeof(uint64_t) * LC_NCOUNT, call.s));
    {
      Prof pr(c, LC_PROF_REFINE, call.s);
      CK(launch_refine(c, n_prob, d_pb, dP1, dP2, du1, du2, ds1, ds2, d_c1, d_c2, dS0, max_iter, th2, lambda,
                       dS, dI, dM, cnt, call.s));
    }
    call.finish();
  });
}

// Reverse Cuthill-McKee ordering of the free vertices (the symbolic phase of the banded
// direct solve, A54): BFS from a pseudo-peripheral vertex of each component, neighbours
// in ascending (degree, index); fixed vertices (no couplings) are placed last. Returns
// the block bandwidth max |pos(i) - pos(j)| over free-free edges.
static int pgo_rcm(int32_t n_v, const uint8_t* fixed, int32_t n_e, const int32_t* eij, std::vector<int32_t>& pos,
                   std::vector<int32_t>& ord) {
  std::vector<int32_t> deg(n_v, 0), beg((size_t)n_v + 1, 0), adj;
  for (int32_t e = 0; e < n_e; ++e) {
    const int32_t i = eij[2 * e], j = eij[2 * e + 1];
    if (fixed[i] || fixed[j]) continue;
    deg[i]++;
    deg[j]++;
  }
  for (int32_t v = 0; v < n_v; ++v) beg[v + 1] = beg[v] + deg[v];
  adj.resize(beg[n_v]);
  {
    std::vector<int32_t> cur(beg.begin(), beg.end() - 1);
    for (int32_t e = 0; e < n_e; ++e) {
      const int32_t i = eij[2 * e], j = eij[2 * e + 1];
      if (fixed[i] || fixed[j]) continue;
      adj[cur[i]++] = j;
      adj[cur[j]++] = i;
    }
  }
  for (int32_t v = 0; v < n_v; ++v)
    std::sort(adj.begin() + beg[v], adj.begin() + beg[v + 1], [&](int32_t x, int32_t y) {
      return deg[x] != deg[y] ? deg[x] < deg[y] : x < y;
    });
  std::vector<int32_t> seen(n_v, 0), level(n_v, -1), order, comp, clev;
  order.reserve(n_v);
  auto bfs = [&](int32_t s) {   // level structure of s's component (unseen vertices)
    comp.clear();
    clev.clear();
    comp.push_back(s);
    clev.push_back(0);
    level[s] = 0;
    for (size_t h = 0; h < comp.size(); ++h) {
      const int32_t u = comp[h];
      for (int32_t q = beg[u]; q < beg[u + 1]; ++q) {
        const int32_t w = adj[q];
        if (!seen[w] && level[w] < 0) {
          level[w] = level[u] + 1;
          comp.push_back(w);
          clev.push_back(level[w]);
        }
      }
    }
    for (int32_t u : comp) level[u] = -1;
  };
  for (int32_t s0 = 0; s0 < n_v; ++s0) {
    if (fixed[s0] || seen[s0]) continue;
    int32_t s = s0;
    for (int sweep = 0; sweep < 2; ++sweep) {   // pseudo-peripheral start: min degree in the last level
      bfs(s);
      const int32_t lmax = clev.back();
      int32_t best = -1;
      for (size_t h = 0; h < comp.size(); ++h)
        if (clev[h] == lmax && (best < 0 || deg[comp[h]] < deg[best] ||
                                (deg[comp[h]] == deg[best] && comp[h] < best)))
          best = comp[h];
      s = best;
    }
    bfs(s);
    for (int32_t u : comp) {
      seen[u] = 1;
      order.push_back(u);
    }
  }
  std::reverse(order.begin(), order.end());
  for (int32_t v = 0; v < n_v; ++v)
    if (fixed[v]) order.push_back(v);
  pos.assign(n_v, 0);
  ord = order;
  for (int32_t p = 0; p < n_v; ++p) pos[order[p]] = p;
  int bw = 0;
  for (int32_t e = 0; e < n_e; ++e) {
    const int32_t i = eij[2 * e], j = eij[2 * e + 1];
    if (fixed[i] || fixed[j]) continue;
    bw = std::max(bw, std::abs(pos[i] - pos[j]));
  }
  return bw;
}

lc_status lc_pgo_sim3(lc_ctx* c, int32_t n_v, const lc_sim3* S_init, const uint8_t* fixed, int32_t n_e,
                      const int32_t* edge_ij, const lc_sim3* M, const lc_pgo_params* params, lc_sim3* out_S,
                      double* out_trace, double* out_chi2, int64_t* out_counts, void* stream) {
  return guarded(c, [&] {
    capture_gate(c, stream, true);
    REQUIRE(params, LC_EINVAL, "null params");
    const lc_pgo_params p = *params;
    REQUIRE(n_v >= 0 && n_e >= 0 && n_e < (1 << 30) && p.max_iter >= 0 && p.cg_max_iter >= 1 && p.lambda0 > 0.0 &&
                p.eps_dx >= 0.0 && p.eps_chi2 >= 0.0 && p.cg_tol >= 0.0 && p.solver >= 0 && p.solver <= 3,
            LC_EINVAL, "bad sizes / parameters");
    REQUIRE(n_v == 0 || (S_init && fixed && out_S), LC_EINVAL, "null vertex array");
    REQUIRE(n_e == 0 || (edge_ij && M), LC_EINVAL, "null edge array");
    // incidence lists (symbolic structure of the block-sparse system): per vertex, its
    // edges in ascending edge order as ((edge << 1) | role (0: i, 1: j), other vertex)
    std::vector<int32_t> vbeg((size_t)n_v + 1, 0), vinc((size_t)4 * n_e);
    for (int32_t e = 0; e < n_e; ++e) {
      const int32_t i = edge_ij[2 * e], j = edge_ij[2 * e + 1];
      REQUIRE(i >= 0 && i < n_v && j >= 0 && j < n_v, LC_ERANGE, "edge vertex out of range");
      REQUIRE(i != j, LC_EINVAL, "edge with i == j");
      vbeg[i + 1]++;
      vbeg[j + 1]++;
    }
    for (int32_t v = 0; v < n_v; ++v) vbeg[v + 1] += vbeg[v];
    {
      std::vector<int32_t> cur(vbeg.begin(), vbeg.end() - 1);
      for (int32_t e = 0; e < n_e; ++e) {
        const int32_t i = edge_ij[2 * e], j = edge_ij[2 * e + 1];
        const int32_t qi = cur[i]++, qj = cur[j]++;
        vinc[2 * qi] = (e << 1);
        vinc[2 * qi + 1] = j;
        vinc[2 * qj] = (e << 1) | 1;
        vinc[2 * qj + 1] = i;
      }
    }
    Call call(c, stream);
    unsigned long long* cnt = call.counts(out_counts, LC_NCOUNT);
    CK(cudaMemsetAsync(cnt, 0, sizeof(uint64_t) * LC_NCOUNT, call.s));
    if (n_v == 0) {
      if (out_chi2) {
        double* dc = call.out(out_chi2, 2);
        CK(cudaMemsetAsync(dc, 0, 2 * sizeof(double), call.s));
      }
      call.finish();
      return;
    }
    const int32_t *d_eij = nullptr, *d_vbeg = nullptr, *d_vinc = nullptr;
    const uint8_t* d_fixed = nullptr;
    call.arg(fixed, (size_t)n_v, &d_fixed);
    call.arg(vbeg.data(), vbeg.size(), &d_vbeg);
    if (n_e > 0) {
      call.arg(edge_ij, (size_t)2 * n_e, &d_eij);
      call.arg(vinc.data(), vinc.size(), &d_vinc);
    }
    const double* dM = call.in((const double*)M, 13 * (size_t)n_e);
    const double* dS0 = call.in((const double*)S_init, 13 * (size_t)n_v);
    double* dS = (double*)call.out((double*)out_S, 13 * (size_t)n_v);
    double* dT = out_trace ? call.out(out_trace, 6 * (size_t)std::max(p.max_iter, 1)) : nullptr;
    double* dC = out_chi2 ? call.out(out_chi2, 2) : nullptr;
    if (dT) CK(cudaMemsetAsync(dT, 0, 6 * sizeof(double) * std::max(p.max_iter, 1), call.s));
    // solver (A54/A54b): in a reverse Cuthill-McKee order, block cyclic reduction over
    // super-blocks of bw positions when they fit one CTA's shared memory and there are at
    // least 4 of them, else the banded Cholesky when the bandwidth fits its window, else
    // block-Jacobi CG
    std::vector<int32_t> pos, ord;
    int bw = pgo_rcm(n_v, fixed, n_e, edge_ij, pos, ord);
    REQUIRE(!(p.solver == LC_PGO_SOLVER_BAND && bw > pgo_max_bw()), LC_EINVAL,
            "LC_PGO_SOLVER_BAND: block bandwidth exceeds the banded solver's window");
    REQUIRE(!(p.solver == LC_PGO_SOLVER_CR && pgo_cr_s(bw) > pgo_cr_max_s()), LC_EINVAL,
            "LC_PGO_SOLVER_CR: block bandwidth exceeds the cyclic-reduction super-block");
    int cr_s = 0;
    if (p.solver == LC_PGO_SOLVER_CR ||
        (p.solver == LC_PGO_SOLVER_AUTO && pgo_cr_s(bw) <= pgo_cr_max_s() && n_v >= 4 * pgo_cr_s(bw)))
      cr_s = pgo_cr_s(bw);
    if (p.solver == LC_PGO_SOLVER_CG || (cr_s == 0 && bw > pgo_max_bw())) bw = -1;
    const int32_t *d_pos = nullptr, *d_ord = nullptr;
    if (bw >= 0) {
      call.arg(pos.data(), pos.size(), &d_pos);
      call.arg(ord.data(), ord.size(), &d_ord);
    }
    call.commit();
    const int grid = pgo_grid(c, n_v, n_e, bw, cr_s);
    void* scr = call.scratch(pgo_scratch_bytes(n_v, n_e, grid, bw, cr_s));
    {
      Prof pr(c, LC_PROF_PGO, call.s);
      CK(launch_pgo(c, n_v, n_e, d_eij, dM, dS0, d_fixed, d_vbeg, d_vinc, bw, d_pos, d_ord, cr_s, p, dS, scr, grid,
                    dT, dC, cnt, call.s));
    }
    call.finish();
  });
}

lc_status lc_state_save(lc_ctx* c, void* stream) {
  return guarded(c, [&] {
    capture_gate(c, stream, false);
    REQUIRE(c->has_map, LC_ESTATE, "no map uploaded");
    Prof pr(c, LC_PROF_STATE, (cudaStream_t)stream);
    CK(launch_state_copy(c, true, (cudaStream_t)stream));
    c->sv_in_win = c->st.h_in_win;
    c->has_saved = true;
  });
}

lc_status lc_state_restore(lc_ctx* c, void* stream) {
  return guarded(c, [&] {
    capture_gate(c, stream, false);
    REQUIRE(c->has_map && c->has_saved, LC_ESTATE, "no saved state");
    Prof pr(c, LC_PROF_STATE, (cudaStream_t)stream);
    CK(launch_state_copy(c, false, (cudaStream_t)stream));
    c->st.h_in_win = c->sv_in_win;
  });
}

// ----------------------------------------------------------------------------
lc_status lc_correct_sim3(lc_ctx* c, int32_t mode, int32_t n_batch, const int32_t* cur_kf,
                          const lc_sim3* S_cw_corr, const int32_t* window_begin, const int32_t* window_kf,
                          const lc_sim3* S_opt, lc_sim3* out_S_corr, int32_t* out_mp_begin,
                          int32_t* out_mp_idx, float* out_mp_pos, int64_t out_capacity, int64_t* out_counts,
                          void* stream) {
  return guarded(c, [&] {
    const bool dry = mode == (LC_CORRECT_WINDOW | LC_DRY_RUN);
    HostProf hp(c, "lc_correct_sim3");
    capture_gate(c, stream, !dry);
    REQUIRE(c->has_map, LC_ESTATE, "no map uploaded");
    REQUIRE(mode == LC_CORRECT_WINDOW || mode == LC_CORRECT_ALL || dry, LC_EINVAL, "bad mode");
    Store& st = c->st;
    Call call(c, stream);
    unsigned long long* cnt = call.counts(out_counts, LC_NCOUNT);   // zeroed by the first kernel
    hp.mark("counts");
    if (mode & LC_CORRECT_WINDOW) {
      REQUIRE(cur_kf && S_cw_corr && window_begin && window_kf, LC_EINVAL, "null WINDOW argument");
      REQUIRE(dry ? n_batch >= 1 : n_batch == 1, LC_EINVAL, "n_batch must be 1 (>= 1 with LC_DRY_RUN)");
      REQUIRE(window_begin[0] == 0, LC_EINVAL, "window_begin[0] must be 0");
      for (int b = 0; b < n_batch; ++b) {
        REQUIRE(cur_kf[b] >= 0 && cur_kf[b] < st.n_kf, LC_ERANGE, "cur_kf out of range");
        REQUIRE(window_begin[b + 1] > window_begin[b], LC_EINVAL, "empty window");
        mark_window(c, window_begin[b + 1] - window_begin[b], window_kf + window_begin[b]);
        REQUIRE(window_kf[window_begin[b]] == cur_kf[b], LC_EINVAL, "a window must start with its cur_kf");
      }
      const int n_slots = window_begin[n_batch];
      const int32_t* d_win = nullptr;
      const double* d_S = nullptr;
      const int32_t* d_wb = nullptr;
      call.arg(window_kf, n_slots, &d_win);
      call.arg((const double*)S_cw_corr, 13 * (size_t)n_batch, &d_S);
      call.arg(window_begin, (size_t)n_batch + 1, &d_wb);
      hp.mark("validate");
      call.commit();
      hp.mark("commit");
      if (dry) {
        REQUIRE(out_S_corr && out_mp_begin && out_capacity >= 0 && (out_capacity == 0 || (out_mp_idx && out_mp_pos)),
                LC_EINVAL, "null DRY_RUN output");
        void* scr = call.scratch(correct_dry_scratch_bytes(n_batch, n_slots, st.n_mp));
        double* dS = (double*)call.out((double*)out_S_corr, 13 * (size_t)n_slots);
        int32_t* dB = call.out(out_mp_begin, (size_t)n_batch + 1);
        int32_t* dI = out_capacity ? call.out(out_mp_idx, (size_t)out_capacity) : nullptr;
        float* dP = out_capacity ? call.out(out_mp_pos, 3 * (size_t)out_capacity) : nullptr;
        {
          Prof pr(c, LC_PROF_CORRECT_WINDOW, call.s);
          CK(launch_correct_dry(c, n_batch, n_slots, d_wb, d_win, d_S, scr, dS, dB, out_capacity, dI, dP, cnt,
                                call.s));
        }
        int32_t total = 0;
        CK(cudaMemcpyAsync(&total, dB + n_batch, sizeof(int32_t), cudaMemcpyDeviceToHost, call.s));
        call.finish();
        CK(cudaStreamSynchronize(call.s));
        REQUIRE((int64_t)total <= out_capacity, LC_ECAPACITY,
                "DRY_RUN: " + std::to_string(total) + " corrected points exceed out_capacity");
        return;
      }
      const int n_window = n_slots;
      double* scr = (double*)call.scratch(sizeof(double) * correct_window_scratch_stride() * (size_t)n_window);
      double* d_outS = (out_S_corr && is_device_ptr(c, out_S_corr)) ? (double*)out_S_corr : nullptr;
      hp.mark("scratch");
      {
        Prof pr(c, LC_PROF_CORRECT_WINDOW, call.s);
        CK(launch_correct_window(c, 0, n_window, d_win, d_S, scr, d_outS, cnt, call.s));
      }
      hp.mark("launch");
      if (out_S_corr && !d_outS) {
        CK(cudaMemcpy2DAsync(out_S_corr, sizeof(lc_sim3), scr + 28, sizeof(double) * correct_window_scratch_stride(),
                             sizeof(lc_sim3), n_window, cudaMemcpyDefault, call.s));
      }
      std::fill(st.h_in_win.begin(), st.h_in_win.end(), 0);
      for (int i = 0; i < n_window; ++i) st.h_in_win[window_kf[i]] = 1;
    } else {
      REQUIRE(S_opt, LC_EINVAL, "null S_opt");
      const double* d_opt = call.in((const double*)S_opt, 13 * (size_t)st.n_kf);
      double* scr = (double*)call.scratch(sizeof(double) * correct_all_scratch_stride() * (size_t)std::max(st.n_kf, 1));
      {
        Prof pr(c, LC_PROF_CORRECT_ALL, call.s);
        CK(launch_correct_all(c, d_opt, scr, cnt, call.s));
      }
      std::fill(st.h_in_win.begin(), st.h_in_win.end(), 0);
    }
    call.finish();
  });
}

// ----------------------------------------------------------------------------
lc_status lc_fuse(lc_ctx* c, int32_t phase, int32_t w_lo, int32_t w_hi, int32_t n_window,
                  const int32_t* window_kf, const lc_sim3* window_S, const int32_t* win_list_begin,
                  const int32_t* mp_list, int64_t n_list, const lc_match_params* params,
                  int32_t cur_kf, const int32_t* forced_mp,
                  int64_t* io_winner, int64_t* io_victim, int8_t* out_action,
                  const lc_query_debug* dbg, int64_t* out_counts, void* stream) {
  return guarded(c, [&] {
    HostProf hp(c, "lc_fuse");
    capture_gate(c, stream, true);
    REQUIRE(c->has_map, LC_ESTATE, "no map uploaded");
    REQUIRE(phase == LC_FUSE_PLAN || phase == LC_FUSE_APPLY || phase == LC_FUSE_ALL, LC_EINVAL, "bad phase");
    REQUIRE(params && params_ok(*params), LC_EINVAL, "bad match params");
    REQUIRE(n_list >= 0 && (n_list == 0 || mp_list), LC_EINVAL, "bad mp_list");
    Store& st = c->st;
    mark_window(c, n_window, window_kf);
    hp.mark("mark");
    if (phase != LC_FUSE_PLAN) { w_lo = 0; w_hi = n_window; }
    if (phase == LC_FUSE_APPLY) { w_lo = w_hi = 0; }
    REQUIRE(0 <= w_lo && w_lo <= w_hi && w_hi <= n_window, LC_EINVAL, "bad shard range");
    // device-resident list offsets (e.g. lc_loop_lists with a device out_begin): nothing is
    // read back; n_list is then the list buffer's capacity (>= the offsets' total)
    const bool dev_csr = win_list_begin && is_device_ptr(c, win_list_begin);
    if (win_list_begin && !dev_csr) {
      REQUIRE(win_list_begin[0] == 0 && win_list_begin[n_window] == n_list, LC_EINVAL,
              "win_list_begin must span [0, n_list]");
      for (int i = 0; i < n_window; ++i)
        REQUIRE(win_list_begin[i + 1] >= win_list_begin[i], LC_EINVAL, "win_list_begin not monotone");
    }
    if (dev_csr && (phase & LC_FUSE_PLAN)) {
      REQUIRE(w_lo == 0 && w_hi == n_window, LC_EINVAL, "device win_list_begin: full-window PLAN only");
      REQUIRE(!dbg, LC_EINVAL, "device win_list_begin: no per-query debug outputs");
      REQUIRE(!forced_mp, LC_EINVAL, "device win_list_begin: no forced matches");
      REQUIRE(n_list == 0 || is_device_ptr(c, mp_list), LC_EINVAL, "device win_list_begin needs a device mp_list");
    }
    int cur_pos = -1;   // forced loop matches (O9.4): cur_kf must be a window keyframe
    if (forced_mp && (phase & LC_FUSE_PLAN)) {
      for (int i = 0; i < n_window; ++i)
        if (window_kf[i] == cur_kf) cur_pos = i;
      REQUIRE(cur_pos >= 0, LC_EINVAL, "forced_mp given but cur_kf is not a window keyframe");
    }
    if (!window_S && (phase & LC_FUSE_PLAN))
      for (int i = 0; i < n_window; ++i)
        REQUIRE(st.h_in_win[window_kf[i]], LC_ESTATE,
                "window_S NULL but a window keyframe has no stored WINDOW correction");
    Call call(c, stream);
    // ---- unit tables (one unit per window position) ----
    std::vector<int64_t> woff(n_window + 1, 0), lbeg(n_window), qoff(n_window);
    for (int i = 0; i < n_window; ++i) {
      int k = window_kf[i];
      woff[i + 1] = woff[i] + (st.h_fbeg[k + 1] - st.h_fbeg[k]);
      lbeg[i] = dev_csr ? 0 : win_list_begin ? win_list_begin[i] : 0;
      qoff[i] = dev_csr ? 0 : win_list_begin ? win_list_begin[i] : (int64_t)i * n_list;
    }
    const int64_t n_wfeat = woff[n_window];
    int64_t total_q = 0;
    int F_max = 0;
    for (int i = w_lo; i < w_hi; ++i) {
      int64_t len = dev_csr ? 0 : win_list_begin ? (int64_t)win_list_begin[i + 1] - win_list_begin[i] : n_list;
      total_q += len;
      F_max = std::max<int>(F_max, (int)(woff[i + 1] - woff[i]));
    }
    if (dev_csr) total_q = n_list;
    // sole mode: one CTA per window keyframe, which initialises and resolves its own
    // winner words (no winner-table init pass, no separate resolve launch). Used when
    // the shard already has enough keyframes to fill the GPU and no list is huge.
    int64_t max_len = 0;
    for (int i = w_lo; i < w_hi && !dev_csr; ++i)
      max_len = std::max<int64_t>(max_len, win_list_begin ? (int64_t)win_list_begin[i + 1] - win_list_begin[i] : n_list);
    // pipelined host list: a full-range PLAN whose per-keyframe lists are in host
    // memory uploads them in kPipe chunks on a side stream; k_project / k_match run
    // on each chunk's blocks as it lands (k_project stamps the LoopSet), the resolve
    // after all of them
    const bool pipe = (phase & LC_FUSE_PLAN) && win_list_begin && !dev_csr && n_list >= c->pipe_min && !dbg &&
                      !c->cap && w_lo == 0 && w_hi == n_window && !is_device_ptr(c, mp_list) &&
                      cur_pos < 0;   // the forced step needs the LoopSet stamped up front
    // sole mode: one k_match CTA per window keyframe, which initialises and resolves its
    // own unit (no winner-table init pass, no resolve launch) -- used when the shard fills
    // the GPU; LC_SOLE=0 forbids it, 1 forces it, 2 forces the queued-item k_match_sole
    // kernel (measured slower at C5)
    const bool sole = !pipe && max_len <= 16384 && w_hi > w_lo &&
                      (dev_csr || (c->sole_mode < 0 ? (w_hi - w_lo) >= 2 * 148 : c->sole_mode >= 1));
    // a full-range PLAN without forced matches stamps the LoopSet in k_project (after its
    // PDL wait, from its own list entries) instead of a separate pass over the lists in
    // k_fuse_prep; a shard's PLAN needs the whole window's LoopSet, so prep stamps it there
    const bool stamp_proj = (phase & LC_FUSE_PLAN) && win_list_begin && w_lo == 0 && w_hi == n_window &&
                            cur_pos < 0;
    const int64_t ch = sole ? std::max<int64_t>(max_len, 1) : pick_chunk(total_q);
    std::vector<int32_t> bunit;
    std::vector<int64_t> bq0, bq1;
    bunit.reserve(w_hi - w_lo + 64);
    bq0.reserve(w_hi - w_lo + 64);
    bq1.reserve(w_hi - w_lo + 64);
    for (int i = w_lo; i < w_hi; ++i) {
      int64_t b = lbeg[i];
      int64_t e = dev_csr ? 0 : b + (win_list_begin ? (int64_t)win_list_begin[i + 1] - win_list_begin[i] : n_list);
      if (sole) {
        bunit.push_back(i);
        bq0.push_back(b);
        bq1.push_back(e);
        continue;
      }
      for (int64_t q = b; q < e; q += ch) {
        bunit.push_back(i);
        bq0.push_back(q);
        bq1.push_back(std::min<int64_t>(q + ch, e));
      }
    }
    std::vector<int64_t> boff(bunit.size() + 1, 0);
    for (size_t b = 0; b < bunit.size(); ++b) boff[b + 1] = boff[b] + (bq1[b] - bq0[b]);
    hp.mark("blocks");
    MatchArgs a;
    memset(&a, 0, sizeof(a));
    fill_match_store(c, a);
    const int64_t* d_boff = nullptr;
    const int32_t* d_win = nullptr;
    const int64_t *d_woff = nullptr, *d_lbeg = nullptr, *d_qoff = nullptr, *d_bq0 = nullptr, *d_bq1 = nullptr;
    const int32_t* d_bunit = nullptr;
    const double* d_S = nullptr;
    const lc_match_params* d_prm = nullptr;
    call.arg(window_kf, n_window, &d_win);
    call.arg(woff.data(), n_window + 1, &d_woff);
    call.arg(params, 1, &d_prm);
    call.arg(bunit.data(), bunit.size(), &d_bunit);
    if (!dev_csr) {
      call.arg(lbeg.data(), n_window, &d_lbeg);
      call.arg(qoff.data(), n_window, &d_qoff);
      call.arg(bq0.data(), bq0.size(), &d_bq0);
      call.arg(bq1.data(), bq1.size(), &d_bq1);
      call.arg(boff.data(), boff.size(), &d_boff);
    }
    if (window_S) {   // device-resident transforms are used in place, host ones ride in the block
      if (is_device_ptr(c, window_S)) d_S = (const double*)window_S;
      else call.arg((const double*)window_S, 13 * (size_t)n_window, &d_S);
    }
    hp.mark("tables");
    call.commit();
    hp.mark("commit");
    if (dev_csr) {   // the unit / block tables from the device offsets (one block per unit)
      int64_t* t = (int64_t*)call.scratch(sizeof(int64_t) * (5 * (size_t)n_window + 1));
      d_lbeg = t; d_qoff = t + n_window; d_bq0 = t + 2 * (size_t)n_window; d_bq1 = t + 3 * (size_t)n_window;
      d_boff = t + 4 * (size_t)n_window;
      CK(launch_csr_units(c, n_window, win_list_begin, t, call.s));
    }
    Surv* d_surv = (Surv*)call.scratch(sizeof(Surv) * std::max<int64_t>(dev_csr ? n_list : boff.back(), 1));
    int32_t* d_scnt = (int32_t*)call.scratch(sizeof(int32_t) * std::max<size_t>(bunit.size(), 1));
    const int32_t* d_list = nullptr;
    int pipe_b[lc_ctx::kPipe + 1] = {};   // block boundaries of the chunks
    if (pipe) {
      int32_t* dl = (int32_t*)call.scratch(sizeof(int32_t) * (size_t)n_list);
      const int nb = (int)bunit.size();
      const int64_t tot = boff[nb];
      pipe_b[0] = 0;
      for (int k = 1; k < lc_ctx::kPipe; ++k) {
        int b = pipe_b[k - 1];
        while (b < nb && boff[b] < tot * k / lc_ctx::kPipe) ++b;
        pipe_b[k] = b;
      }
      pipe_b[lc_ctx::kPipe] = nb;
      // the side stream first waits for the work already on the call stream (the list
      // buffer may still be read by an earlier call)
      CK(cudaEventRecord(c->pipe_ev[lc_ctx::kPipe], call.s));
      CK(cudaStreamWaitEvent(c->side, c->pipe_ev[lc_ctx::kPipe], 0));
      for (int k = 0; k < lc_ctx::kPipe; ++k) {
        const int b0 = pipe_b[k], b1 = pipe_b[k + 1];
        if (b1 > b0) {
          const int64_t l0 = bq0[b0], l1 = bq1[b1 - 1];
          CK(cudaMemcpyAsync(dl + l0, mp_list + l0, sizeof(int32_t) * (size_t)(l1 - l0),
                             cudaMemcpyHostToDevice, c->side));
        }
        CK(cudaEventRecord(c->pipe_ev[k], c->side));
      }
      d_list = dl;
    } else {
      d_list = call.in(mp_list, (size_t)n_list);
    }
    unsigned long long* win = (unsigned long long*)call.out(io_winner, (size_t)n_wfeat, phase == LC_FUSE_APPLY);
    if (!win) win = (unsigned long long*)call.scratch(sizeof(uint64_t) * std::max<int64_t>(n_wfeat, 1));
    unsigned long long* vic = (unsigned long long*)call.out(io_victim, (size_t)st.n_mp, phase == LC_FUSE_APPLY);
    if (!vic) vic = (unsigned long long*)call.scratch(sizeof(uint64_t) * std::max(st.n_mp, 1));
    int8_t* act = call.out(out_action, (size_t)n_wfeat);
    if (act && (phase & LC_FUSE_PLAN)) CK(cudaMemsetAsync(act, 0, (size_t)n_wfeat, call.s));
    unsigned long long* cnt = call.counts(out_counts, LC_NCOUNT);   // zeroed by k_fuse_prep
    const int64_t n_q_all = win_list_begin ? n_list : (int64_t)n_window * n_list;
    int64_t* dbg_best = nullptr;
    double* dbg_uv = nullptr;
    int32_t* dbg_nc = nullptr;
    if (dbg && (phase & LC_FUSE_PLAN)) {
      dbg_best = call.out(dbg->best, (size_t)n_q_all, true);
      dbg_uv = call.out(dbg->uv, 2 * (size_t)n_q_all, true);
      dbg_nc = call.out(dbg->ncand, (size_t)n_q_all, true);
    }
    // ---- epoch (LoopSet stamp / window membership) ----
    const int n_ep = cur_pos >= 0 ? 2 : 1;
    if (c->cap) c->cap->n_fuse += n_ep;
    else epoch_reserve(c, n_ep, call.s);
    if (cur_pos >= 0) {   // O9.4: the forced matches, applied before the search
      const int32_t* d_forced = call.in(forced_mp, (size_t)(st.h_fbeg[cur_kf + 1] - st.h_fbeg[cur_kf]));
      Prof pr(c, LC_PROF_APPLY, call.s);
      CK(launch_fuse_prep(c, LC_FUSE_PLAN, 1, 0, 0, n_window, d_win, n_wfeat, d_list, n_list, win, vic, cnt,
                          call.s));
      CK(launch_forced(c, cur_kf, d_forced, win + woff[cur_pos], vic, cnt, call.s));
      CK(launch_fuse_apply(c, d_woff, win, vic, cnt, call.s));
    }
    {
      Prof pr(c, LC_PROF_FUSE_PREP, call.s);
      // sole-mode CTAs initialise their own units' words; every other word of the
      // table (the other shards' units included) is set to NONE here (lc.h contract)
      const int64_t skip_lo = sole ? woff[w_lo] : 0, skip_hi = sole ? woff[w_hi] : 0;
      CK(launch_fuse_prep(c, phase, cur_pos < 0 ? 1 : 0, skip_lo, skip_hi, n_window, d_win, n_wfeat, d_list,
                          (pipe || stamp_proj) ? 0 : n_list, win, vic, cnt, call.s));
    }
    if (phase & LC_FUSE_PLAN) {
      a.unit_kf = d_win;
      a.unit_S = d_S;
      a.kf_S_corr = st.kf_S_corr;
      a.unit_param = nullptr;
      a.unit_woff = d_woff;
      a.unit_toff = d_woff;
      a.unit_lbeg = d_lbeg;
      a.unit_qoff = d_qoff;
      a.params = d_prm;
      a.blk_unit = d_bunit;
      a.blk_q0 = d_bq0;
      a.blk_q1 = d_bq1;
      a.mp_list = d_list;
      a.taken = nullptr;
      a.winner = win;
      a.counts = cnt;
      a.n_mp = st.n_mp;
      a.dbg_best = dbg_best;
      a.dbg_uv = dbg_uv;
      a.dbg_ncand = dbg_nc;
      a.feat_angle = st.feat_angle;
      a.loop_ep = st.mp_loop_ep;
      a.epoch = st.ep;
      a.victim = vic;
      a.action = act;
      a.unit_base = w_lo;
      a.surv = d_surv;
      a.surv_off = d_boff;
      a.surv_cnt = d_scnt;
      a.sole = sole ? (c->sole_mode == 2 ? 2 : 1) : 0;
      a.loop_ep_w = (pipe || stamp_proj) ? st.mp_loop_ep : nullptr;   // k_project stamps the LoopSet
      // eager calls know the epoch on the host: k_fuse_prep's epoch = ep[0] + 1 and every
      // fuse epoch is reserved through ep_used (epoch_reserve), so ep_used is this call's
      // (main) epoch; a captured call's replays take theirs from the device counter
      a.stamp_epoch = (a.loop_ep_w && !c->cap) ? (uint32_t)c->ep_used : 0u;
      if (pipe) {
        for (int k = 0; k < lc_ctx::kPipe; ++k) {
          const int b0 = pipe_b[k], nbk = pipe_b[k + 1] - pipe_b[k];
          CK(cudaStreamWaitEvent(call.s, c->pipe_ev[k], 0));
          if (nbk == 0) continue;
          a.blk_base = b0;
          {
            Prof pr(c, LC_PROF_PROJECT, call.s);
            CK(launch_match(c, 0, a, nbk, F_max, 0, call.s, false));
          }
          Prof pr(c, LC_PROF_MATCH, call.s);
          CK(launch_match(c, 0, a, nbk, F_max, 1, call.s));
        }
        a.blk_base = 0;
      } else {
        {
          Prof pr(c, LC_PROF_PROJECT, call.s);
          CK(launch_match(c, 0, a, (int)bunit.size(), F_max, 0, call.s));
        }
        Prof pr(c, LC_PROF_MATCH, call.s);
        CK(launch_match(c, 0, a, (int)bunit.size(), F_max, 1, call.s));
      }
      if (!sole) {
        Prof pr(c, LC_PROF_RESOLVE, call.s);
        CK(launch_resolve(c, 0, a, w_hi - w_lo, call.s));
      }
    }
    if (phase & LC_FUSE_APPLY) {
      Prof pr(c, LC_PROF_APPLY, call.s);
      CK(launch_fuse_apply(c, d_woff, win, vic, cnt, call.s));
    }
    hp.mark("launches");
    call.finish();
  });
}

// ----------------------------------------------------------------------------
lc_status lc_loop_lists(lc_ctx* c, int32_t n, const int32_t* src_begin, const int32_t* src_kf, int32_t* out_begin,
                        int32_t* out_list, int64_t capacity, void* stream) {
  return guarded(c, [&] {
    capture_gate(c, stream, false);
    REQUIRE(c->has_map, LC_ESTATE, "no map uploaded");
    REQUIRE(n >= 0 && src_begin && out_begin && capacity >= 0 && (capacity == 0 || out_list), LC_EINVAL,
            "null argument / negative size");
    REQUIRE(src_begin[0] == 0, LC_EINVAL, "src_begin[0] must be 0");
    Store& st = c->st;
    std::vector<int64_t> reg_off((size_t)n + 1, 0);
    const int umax = lists_max_unique();
    int64_t ub_sum = 0, ub_max = 0;   // upper bounds of the lists' lengths (their sources' features)
    for (int l = 0; l < n; ++l) {
      REQUIRE(src_begin[l + 1] >= src_begin[l], LC_EINVAL, "src_begin not monotone");
      int64_t ub = 0;
      for (int j = src_begin[l]; j < src_begin[l + 1]; ++j) {
        const int k = src_kf[j];
        REQUIRE(k >= 0 && k < st.n_kf, LC_ERANGE, "source keyframe out of range");
        ub += st.h_fbeg[k + 1] - st.h_fbeg[k];
      }
      reg_off[l + 1] = reg_off[l] + std::min<int64_t>(ub, umax);
      ub_sum += ub;
      ub_max = std::max(ub_max, ub);
    }
    const bool dev_mode = is_device_ptr(c, out_begin);
    if (dev_mode) {
      REQUIRE(capacity == 0 || is_device_ptr(c, out_list), LC_EINVAL, "a device out_begin needs a device out_list");
      REQUIRE((int64_t)st.n_mp <= 32 * (int64_t)lists_bitmap_words_max(), LC_ECAPACITY,
              "device out_begin: maps of more than " + std::to_string(32 * lists_bitmap_words_max()) +
              " map points need the host-offset path");
      REQUIRE(ub_sum <= capacity, LC_ECAPACITY,
              "device out_begin: capacity must hold the lists' upper bound " + std::to_string(ub_sum));
      REQUIRE(ub_max <= 261888, LC_ECAPACITY, "device out_begin: a list may exceed 261888 entries");
      if (n == 0) {
        CK(cudaMemsetAsync(out_begin, 0, sizeof(int32_t), (cudaStream_t)stream));
        return;
      }
    } else {
      out_begin[0] = 0;
    }
    if (n == 0) return;
    Call call(c, stream);
    const int32_t *d_sb = nullptr, *d_sk = nullptr;
    const int64_t* d_ro = nullptr;
    call.arg(src_begin, (size_t)n + 1, &d_sb);
    call.arg(src_kf, (size_t)std::max(src_begin[n], 1), &d_sk);
    call.arg(reg_off.data(), reg_off.size(), &d_ro);
    std::vector<int64_t> bmo0;
    const int64_t* d_bmo0 = nullptr;
    if (dev_mode) {   // bitmap offsets of the first pass (l * w1), in the argument block
      bmo0.resize(n);
      for (int l = 0; l < n; ++l) bmo0[l] = (int64_t)l * lists_bitmap_words();
      call.arg(bmo0.data(), bmo0.size(), &d_bmo0);
    }
    call.commit();
    if (dev_mode) {
      // device-resident offsets, no host synchronisation (lc.h): first pass (small bitmaps,
      // global), the wide lists counted in a second pass (large shared-memory bitmap), a scan
      // of the counts into out_begin, then both emissions (the wide lists' bitmaps rebuilt)
      const int w1 = lists_bitmap_words(), w2 = lists_bitmap_words_max();
      uint32_t* d_bm = (uint32_t*)call.scratch(sizeof(uint32_t) * (size_t)n * w1);
      int32_t* d_lo = (int32_t*)call.scratch(sizeof(int32_t) * 2 * (size_t)n);
      int32_t* d_cnt = (int32_t*)call.scratch(sizeof(int32_t) * (size_t)n);
      int2* d_rng = (int2*)call.scratch(sizeof(int2) * (size_t)std::max(src_begin[n], 1));
      CK(launch_kf_idrange(c, src_begin[n], d_sk, d_rng, call.s));
      CK(launch_lists_bitmap(c, n, n, nullptr, w1, d_rng, d_bm, d_lo, d_cnt, d_sb, d_sk, call.s));
      CK(launch_lists_bitmap(c, n, n, nullptr, w2, d_rng, nullptr, d_lo, d_cnt, d_sb, d_sk, call.s, true));
      CK(launch_lists_scan(c, n, d_cnt, out_begin, call.s));
      CK(launch_lists_emit(c, n, d_bm, d_bmo0, d_lo, d_cnt, out_begin, out_list, call.s));
      CK(launch_lists_emit_wide(c, n, w2, d_sb, d_sk, d_lo, out_begin, out_list, call.s));
      return;
    }
    // bitmap path (ascending unique by construction): a small bitmap per list first; the
    // lists whose id range is wider (-1 counts) again with the large one; beyond that the
    // general hash + sort path
    const int w1 = lists_bitmap_words(), w2 = lists_bitmap_words_max();
    uint32_t* d_bm = (uint32_t*)call.scratch(sizeof(uint32_t) * (size_t)n * w1);
    int32_t* d_lo = (int32_t*)call.scratch(sizeof(int32_t) * 2 * (size_t)n);   // first id, words
    int32_t* d_cnt = (int32_t*)call.scratch(sizeof(int32_t) * (size_t)n);
    int2* d_rng = (int2*)call.scratch(sizeof(int2) * (size_t)std::max(src_begin[n], 1));
    CK(launch_kf_idrange(c, src_begin[n], d_sk, d_rng, call.s));
    CK(launch_lists_bitmap(c, n, n, nullptr, w1, d_rng, d_bm, d_lo, d_cnt, d_sb, d_sk, call.s));
    std::vector<int32_t> cnt(n);
    CK(cudaMemcpyAsync(cnt.data(), d_cnt, sizeof(int32_t) * n, cudaMemcpyDeviceToHost, call.s));
    CK(cudaStreamSynchronize(call.s));
    std::vector<int64_t> bm_off(n);
    for (int l = 0; l < n; ++l) bm_off[l] = (int64_t)l * w1;
    std::vector<int32_t> wide;
    for (int l = 0; l < n; ++l)
      if (cnt[l] < 0) wide.push_back(l);
    uint32_t* d_bm2 = nullptr;
    if (!wide.empty()) {
      d_bm2 = (uint32_t*)call.scratch(sizeof(uint32_t) * wide.size() * (size_t)w2);
      const int32_t* d_wide = call.in(wide.data(), wide.size());
      CK(launch_lists_bitmap(c, (int)wide.size(), n, d_wide, w2, d_rng, d_bm2, d_lo, d_cnt, d_sb, d_sk, call.s));
      CK(cudaMemcpyAsync(cnt.data(), d_cnt, sizeof(int32_t) * n, cudaMemcpyDeviceToHost, call.s));
      CK(cudaStreamSynchronize(call.s));
      for (size_t i = 0; i < wide.size(); ++i) bm_off[wide[i]] = (int64_t)(d_bm2 - d_bm) + (int64_t)i * w2;
    }
    std::vector<int32_t> hashed;   // still too wide (maps of more than 1.8M points): hash + sort
    for (int l = 0; l < n; ++l)
      if (cnt[l] < 0) hashed.push_back(l);
    int32_t* d_reg = nullptr;
    if (!hashed.empty()) {
      d_reg = (int32_t*)call.scratch(sizeof(int32_t) * (size_t)std::max<int64_t>(reg_off[n], 1));
      const int32_t* d_h = call.in(hashed.data(), hashed.size());
      int32_t* d_hcnt = (int32_t*)call.scratch(sizeof(int32_t) * (size_t)n);
      std::vector<int32_t> hcnt(n);
      CK(launch_lists_dedup(c, false, (int)hashed.size(), d_h, d_sb, d_sk, d_ro, d_reg, d_hcnt, call.s));
      CK(cudaMemcpyAsync(hcnt.data(), d_hcnt, sizeof(int32_t) * n, cudaMemcpyDeviceToHost, call.s));
      CK(cudaStreamSynchronize(call.s));
      std::vector<int32_t> big;
      for (int l : hashed)
        if (hcnt[l] < 0) big.push_back(l);
      if (!big.empty()) {
        const int32_t* d_big = call.in(big.data(), big.size());
        CK(launch_lists_dedup(c, true, (int)big.size(), d_big, d_sb, d_sk, d_ro, d_reg, d_hcnt, call.s));
        CK(cudaMemcpyAsync(hcnt.data(), d_hcnt, sizeof(int32_t) * n, cudaMemcpyDeviceToHost, call.s));
        CK(cudaStreamSynchronize(call.s));
      }
      for (int l : hashed) {
        REQUIRE(hcnt[l] >= 0, LC_ECAPACITY, "a loop list holds more than " + std::to_string(umax) + " map points");
        cnt[l] = hcnt[l];
      }
    }
    for (int l = 0; l < n; ++l) out_begin[l + 1] = out_begin[l] + cnt[l];
    REQUIRE((int64_t)out_begin[n] <= capacity, LC_ECAPACITY,
            "loop lists: " + std::to_string(out_begin[n]) + " entries exceed capacity");
    const int32_t* d_ob = call.in(out_begin, (size_t)n + 1);
    const int64_t* d_bmo = call.in(bm_off.data(), bm_off.size());
    int32_t* d_out = call.out(out_list, (size_t)out_begin[n]);
    // the hashed lists keep -1 in the bitmap counts: k_lists_emit skips them
    CK(launch_lists_emit(c, n, d_bm, d_bmo, d_lo, d_cnt, d_ob, d_out, call.s));
    for (int l : hashed) {   // bitonic sort into place (one launch each; only maps over 1.8M points)
      const int64_t* d_one_ro = call.in(&reg_off[l], 2);
      const int32_t ob2[2] = {0, cnt[l]};
      const int32_t* d_ob2 = call.in(ob2, 2);   // (pageable -> staged before the call returns)
      CK(launch_lists_sort(c, 1, cnt[l], d_one_ro, d_reg, d_ob2, d_out + out_begin[l], call.s));
    }
    call.finish();
  });
}

// ----------------------------------------------------------------------------
lc_status lc_set_point_range(lc_ctx* c, int32_t mp_lo, int32_t mp_hi) {
  return guarded(c, [&] {
    capture_gate(c, (void*)c->cap_stream, true);
    REQUIRE(c->has_map, LC_ESTATE, "no map uploaded");
    if (mp_hi < 0) { c->mp_lo = 0; c->mp_hi = -1; return; }
    REQUIRE(mp_lo >= 0 && mp_lo <= mp_hi && mp_hi <= c->st.n_mp, LC_EINVAL, "bad map-point range");
    c->mp_lo = mp_lo;
    c->mp_hi = mp_hi;
  });
}

lc_status lc_mp_positions(lc_ctx* c, int32_t op, int32_t mp_lo, int32_t mp_hi, float* xyz, void* stream) {
  return guarded(c, [&] {
    capture_gate(c, stream, true);
    REQUIRE(c->has_map, LC_ESTATE, "no map uploaded");
    REQUIRE(op == LC_POS_GET || op == LC_POS_SET, LC_EINVAL, "bad op");
    REQUIRE(mp_lo >= 0 && mp_lo <= mp_hi && mp_hi <= c->st.n_mp, LC_EINVAL, "bad map-point range");
    const size_t n = 3 * (size_t)(mp_hi - mp_lo);
    REQUIRE(n == 0 || xyz, LC_EINVAL, "null xyz");
    if (n == 0) return;
    Call call(c, stream);
    float* d = op == LC_POS_GET ? call.out(xyz, n) : const_cast<float*>(call.in((const float*)xyz, n));
    CK(launch_mp_positions(c, op, mp_lo, mp_hi, d, call.s));
    call.finish();
  });
}

// ----------------------------------------------------------------------------
lc_status lc_fuse_adds(lc_ctx* c, int32_t op, int32_t n_window, const int32_t* window_kf, int32_t w_lo,
                       int32_t w_hi, int64_t* io_winner, int64_t* io_idx, int64_t* io_word, int64_t* io_n,
                       int64_t capacity, void* stream) {
  return guarded(c, [&] {
    capture_gate(c, stream, op == LC_ADDS_UNPACK);
    REQUIRE(c->has_map, LC_ESTATE, "no map uploaded");
    REQUIRE(op == LC_ADDS_PACK || op == LC_ADDS_UNPACK, LC_EINVAL, "bad op");
    REQUIRE(io_winner && io_n && capacity >= 0 && (capacity == 0 || (io_idx && io_word)), LC_EINVAL, "null argument");
    mark_window(c, n_window, window_kf);
    REQUIRE(0 <= w_lo && w_lo <= w_hi && w_hi <= n_window, LC_EINVAL, "bad shard range");
    Store& st = c->st;
    std::vector<int64_t> woff(n_window + 1, 0);
    for (int i = 0; i < n_window; ++i) woff[i + 1] = woff[i] + (st.h_fbeg[window_kf[i] + 1] - st.h_fbeg[window_kf[i]]);
    Call call(c, stream);
    const int32_t* d_win = nullptr;
    const int64_t* d_woff = nullptr;
    call.arg(window_kf, n_window, &d_win);
    call.arg(woff.data(), woff.size(), &d_woff);
    call.commit();
    const int64_t n_wfeat = woff[n_window];
    if (op == LC_ADDS_PACK) {
      const int64_t* d_w = call.in(io_winner, (size_t)n_wfeat);
      int64_t* d_i = capacity ? call.out(io_idx, (size_t)capacity) : nullptr;
      int64_t* d_o = capacity ? call.out(io_word, (size_t)capacity) : nullptr;
      unsigned long long* d_n = (unsigned long long*)call.scratch(sizeof(unsigned long long));
      CK(launch_adds(c, op, n_window, d_win, d_woff, n_wfeat, woff[w_lo], woff[w_hi], (unsigned long long*)d_w,
                     (long long*)d_i, (long long*)d_o, d_n, 0, capacity, call.s));
      unsigned long long n = 0;
      CK(cudaMemcpyAsync(&n, d_n, sizeof(n), cudaMemcpyDeviceToHost, call.s));
      call.finish();
      CK(cudaStreamSynchronize(call.s));
      *io_n = (int64_t)n;
      REQUIRE((int64_t)n <= capacity, LC_ECAPACITY, "lc_fuse_adds: more ADDs than capacity");
      return;
    }
    REQUIRE(*io_n >= 0 && *io_n <= capacity, LC_EINVAL, "io_n outside [0, capacity]");
    int64_t* d_w = call.out(io_winner, (size_t)n_wfeat);
    const int64_t* d_i = call.in(io_idx, (size_t)*io_n);
    const int64_t* d_o = call.in(io_word, (size_t)*io_n);
    CK(launch_adds(c, op, n_window, d_win, d_woff, n_wfeat, 0, 0, (unsigned long long*)d_w, (long long*)d_i,
                   (long long*)d_o, nullptr, *io_n, capacity, call.s));
    call.finish();
  });
}

// ----------------------------------------------------------------------------
lc_status lc_search_by_projection(lc_ctx* c, int32_t n_pairs, const int32_t* pair_kf,
                                  const lc_sim3* pair_S, const int32_t* pair_param,
                                  const lc_match_params* params, int32_t n_params,
                                  const int32_t* pair_list_begin, const int32_t* mp_list,
                                  const int32_t* pair_taken, int32_t* out_feat_mp,
                                  int32_t* out_feat_dist, const lc_query_debug* dbg,
                                  int64_t* out_counts, void* stream) {
  return guarded(c, [&] {
    capture_gate(c, stream, true);
    REQUIRE(c->has_map, LC_ESTATE, "no map uploaded");
    REQUIRE(n_pairs >= 0, LC_EINVAL, "n_pairs < 0");
    if (n_pairs == 0) return;
    REQUIRE(pair_kf && pair_S && pair_param && pair_list_begin && params && n_params >= 1,
            LC_EINVAL, "null pair arrays or params");
    REQUIRE(out_feat_mp && out_feat_dist, LC_EINVAL, "null outputs");
    for (int i = 0; i < n_params; ++i) REQUIRE(params_ok(params[i]), LC_EINVAL, "bad match params");
    Store& st = c->st;
    REQUIRE(pair_list_begin[0] == 0, LC_EINVAL, "pair_list_begin[0] must be 0");
    const int64_t n_list = pair_list_begin[n_pairs];
    REQUIRE(n_list == 0 || mp_list, LC_EINVAL, "null mp_list");
    std::vector<int64_t> off(n_pairs + 1, 0), lbeg(n_pairs);
    int F_max = 0;
    int64_t total_q = 0;
    for (int p = 0; p < n_pairs; ++p) {
      int k = pair_kf[p];
      REQUIRE(k >= 0 && k < st.n_kf, LC_ERANGE, "pair keyframe out of range");
      REQUIRE(pair_param[p] >= 0 && pair_param[p] < n_params, LC_EINVAL, "pair_param out of range");
      REQUIRE(pair_list_begin[p + 1] >= pair_list_begin[p], LC_EINVAL, "pair_list_begin not monotone");
      int F = st.h_fbeg[k + 1] - st.h_fbeg[k];
      off[p + 1] = off[p] + F;
      lbeg[p] = pair_list_begin[p];
      F_max = std::max(F_max, F);
      total_q += pair_list_begin[p + 1] - pair_list_begin[p];
    }
    const int64_t n_tot = off[n_pairs];
    const int ch = pick_chunk(total_q);
    std::vector<int32_t> bunit;
    std::vector<int64_t> bq0, bq1;
    for (int p = 0; p < n_pairs; ++p)
      for (int64_t q = pair_list_begin[p]; q < pair_list_begin[p + 1]; q += ch) {
        bunit.push_back(p);
        bq0.push_back(q);
        bq1.push_back(std::min<int64_t>(q + ch, pair_list_begin[p + 1]));
      }
    std::vector<int64_t> boff(bunit.size() + 1, 0);
    for (size_t b = 0; b < bunit.size(); ++b) boff[b + 1] = boff[b] + (bq1[b] - bq0[b]);
    const int64_t* d_boff = nullptr;
    Call call(c, stream);
    const int32_t *d_kf = nullptr, *d_param = nullptr, *d_bunit = nullptr;
    const int64_t *d_off = nullptr, *d_lbeg = nullptr, *d_bq0 = nullptr, *d_bq1 = nullptr;
    const double* d_S = nullptr;
    const lc_match_params* d_prm = nullptr;
    call.arg(pair_kf, n_pairs, &d_kf);
    call.arg(pair_param, n_pairs, &d_param);
    call.arg(off.data(), n_pairs + 1, &d_off);
    call.arg(lbeg.data(), n_pairs, &d_lbeg);
    call.arg(bunit.data(), bunit.size(), &d_bunit);
    call.arg(bq0.data(), bq0.size(), &d_bq0);
    call.arg(bq1.data(), bq1.size(), &d_bq1);
    call.arg((const double*)pair_S, 13 * (size_t)n_pairs, &d_S);
    call.arg(params, n_params, &d_prm);
    call.arg(boff.data(), boff.size(), &d_boff);
    call.commit();
    Surv* d_surv = (Surv*)call.scratch(sizeof(Surv) * std::max<int64_t>(boff.back(), 1));
    int32_t* d_scnt = (int32_t*)call.scratch(sizeof(int32_t) * std::max<size_t>(bunit.size(), 1));
    const int32_t* d_list = call.in(mp_list, (size_t)n_list);
    const int32_t* d_taken = call.in(pair_taken, (size_t)n_tot);
    int32_t* o_mp = call.out(out_feat_mp, (size_t)n_tot);
    int32_t* o_dist = call.out(out_feat_dist, (size_t)n_tot);
    unsigned long long* win = (unsigned long long*)call.scratch(sizeof(uint64_t) * std::max<int64_t>(n_tot, 1));
    unsigned long long* cnt = (unsigned long long*)call.scratch(sizeof(uint64_t) * LC_NCOUNT * n_pairs);
    CK(cudaMemsetAsync(cnt, 0, sizeof(uint64_t) * LC_NCOUNT * n_pairs, call.s));
    CK(launch_fill_u64(c, win, n_tot, 0x7FFFFFFFFFFFFFFFull, call.s));
    MatchArgs a;
    memset(&a, 0, sizeof(a));
    fill_match_store(c, a);
    a.unit_kf = d_kf;
    a.unit_S = d_S;
    a.kf_S_corr = st.kf_S_corr;
    a.unit_param = d_param;
    a.unit_woff = d_off;
    a.unit_toff = d_off;
    a.unit_lbeg = d_lbeg;
    a.unit_qoff = d_lbeg;
    a.params = d_prm;
    a.blk_unit = d_bunit;
    a.blk_q0 = d_bq0;
    a.blk_q1 = d_bq1;
    a.mp_list = d_list;
    a.taken = d_taken;
    a.feat_angle = st.feat_angle;
    a.out_mp = o_mp;
    a.out_dist = o_dist;
    a.sole = 0;
    a.unit_base = 0;
    a.surv = d_surv;
    a.surv_off = d_boff;
    a.surv_cnt = d_scnt;
    a.winner = win;
    a.counts = cnt;
    a.n_mp = st.n_mp;
    if (dbg) {
      a.dbg_best = call.out(dbg->best, (size_t)n_list, true);
      a.dbg_uv = call.out(dbg->uv, 2 * (size_t)n_list, true);
      a.dbg_ncand = call.out(dbg->ncand, (size_t)n_list, true);
    }
    {
      Prof pr(c, LC_PROF_SBP_MATCH, call.s);
      CK(launch_match(c, 1, a, (int)bunit.size(), F_max, 0, call.s));
      CK(launch_match(c, 1, a, (int)bunit.size(), F_max, 1, call.s));
    }
    Prof pr(c, LC_PROF_SBP_RESOLVE, call.s);
    CK(launch_resolve(c, 1, a, n_pairs, call.s));
    if (out_counts) {
      int64_t* d = call.out(out_counts, (size_t)LC_NCOUNT * n_pairs);
      CK(cudaMemcpyAsync(d, cnt, sizeof(uint64_t) * LC_NCOUNT * n_pairs, cudaMemcpyDeviceToDevice, call.s));
    }
    call.finish();
  });
}

}  // extern "C"
