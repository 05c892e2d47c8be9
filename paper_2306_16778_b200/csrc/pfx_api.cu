// C ABI entry points (include/pfx.h): argument checks, host<->device staging,
// device arena, pole-table upload, dispatch to the kernels.
#include <cuda_runtime.h>

#include <chrono>
#include <cmath>
#include <algorithm>
#include <cstdio>
#include <cstring>
#include <atomic>
#include <mutex>
#include <string>
#include <vector>

#include "pfx_common.cuh"

namespace pfx {

// kernels (defined in the other translation units)
int dense_batched_supported(int64_t d);
int dense_batched_slots(int d, int64_t nsys);
int dense_batched_run(const double* A, int a_complex, int d, int batch, const double* V, int v_complex, int ncols,
                      int full, int real_path, int solve_only, double shift_c, const double2* theta_d, const double2* coef_d,
                      int npairs, double* out, cudaStream_t stream, float* launch_ms, int pivot);
int dense_large_run(const double* A, int a_complex, int d, const double* V, int v_complex, int ncols, int full,
                    int real_path, double shift_c, const double2* theta_d, const double2* coef_d, int npairs,
                    double* out, cudaStream_t stream, float* per_pair_ms, int pivot, const double* A_host = nullptr,
                    const double* V_host = nullptr, double* out_host = nullptr);
int dense_large_cols_run(const double* A, int a_complex, int d, double shift_c, const double2* theta_d,
                         const double2* coef_d, int npairs, const int64_t* ranges, double* out, int accumulate,
                         cudaStream_t stream, int pivot);
int tridiag_run(const double* diag, const double* off, int64_t N, const double* V, int64_t nrhs, double shift_c,
                const double2* theta_d, const double2* coef_d, int npairs, double* out, cudaStream_t stream,
                float* launch_ms, const double* V_host = nullptr, double* out_host = nullptr,
                const TriShard* sh = nullptr);
int banded_run(const double* band, int64_t N, int64_t kb, const double* V, int64_t nrhs, double shift_c,
               const double2* theta_d, const double2* coef_d, int npairs, double* out, cudaStream_t stream,
               float* per_pair_ms, const double* band_host = nullptr, const double* V_host = nullptr);
int pole_table_host(int n, double* theta2, double* coef2);
int dense_blocked_eligible(int64_t d, int64_t batch, int npairs, int full, int64_t ncols);
int dense_blocked_run(const double* A, int a_complex, int d, int batch, const double* V, int v_complex, int nr,
                      int real_path, double shift_c, const double2* theta_d, const double2* coef_d, int npairs,
                      double* out, cudaStream_t stream, float* launch_ms, int pivot);

// d <= 512: many systems with few right-hand sides go to the batched blocked path (block
// toolkit, dense_blocked.cu), the rest to the one-CTA-per-system kernel (dense_batched.cu)
static int dense_small_run(const double* A, int a_complex, int d, int batch, const double* V, int v_complex,
                           int ncols, int full, int real_path, double shift_c, const double2* th, const double2* co,
                           int npairs, double* out, cudaStream_t stream, float* ms, int pivot) {
  if (pivot != 1 && dense_blocked_eligible(d, batch, npairs, full, ncols))
    return dense_blocked_run(A, a_complex, d, batch, V, v_complex, ncols, real_path, shift_c, th, co, npairs, out,
                             stream, ms, pivot);
  return dense_batched_run(A, a_complex, d, batch, V, v_complex, ncols, full, real_path, 0, shift_c, th, co, npairs,
                           out, stream, ms, pivot);
}
int shifted_solve_large(const double* A, int a_complex, int d, const double2* theta_d, const double* V, int nrhs,
                        double2* Y, cudaStream_t stream);

static thread_local std::string g_err;

void set_error(const std::string& msg) { g_err = msg; }

int fail(int status, const std::string& msg) {
  g_err = msg;
  return status;
}

// ---- kernel timing -------------------------------------------------------------
namespace {
struct ProfRec {
  std::string name;
  cudaEvent_t e0, e1;
  double flops;
  cudaStream_t stream;
};
std::mutex g_prof_mu;
std::vector<ProfRec> g_prof;
bool g_prof_on = false;
}  // namespace

bool prof_on() { return g_prof_on; }

static thread_local const char* g_prof_tag = nullptr;
void prof_set_tag(const char* tag) { g_prof_tag = tag; }
const char* prof_get_tag() { return g_prof_tag; }

void prof_mark(const char* name_, cudaStream_t stream, bool begin, double flops) {
  const std::string name = g_prof_tag ? std::string(name_) + "@" + g_prof_tag : std::string(name_);
  std::lock_guard<std::mutex> lk(g_prof_mu);
  if (begin) {
    ProfRec r;
    r.name = name;
    r.flops = flops;
    r.stream = stream;
    cudaEventCreate(&r.e0);
    cudaEventCreate(&r.e1);
    cudaEventRecord(r.e0, stream);
    g_prof.push_back(r);
  } else {
    for (auto it = g_prof.rbegin(); it != g_prof.rend(); ++it)
      if (it->name == name) {
        cudaEventRecord(it->e1, stream);
        break;
      }
  }
}

// ---- arena ------------------------------------------------------------------
namespace {
constexpr int kMaxDev = 16;
constexpr int kSlots = 8;
struct Arena {
  void* ptr[kSlots] = {};
  size_t cap[kSlots] = {};
};
Arena g_arena[kMaxDev];
std::mutex g_arena_mu;
}  // namespace

int* pinned_word() {
  thread_local int* p = nullptr;
  if (!p && cudaMallocHost(reinterpret_cast<void**>(&p), 64) != cudaSuccess) {
    cudaGetLastError();
    p = nullptr;
  }
  return p;
}

int sync_stream(cudaStream_t stream) {
  const auto t0 = std::chrono::steady_clock::now();
  for (;;) {
    const cudaError_t q = cudaStreamQuery(stream);
    if (q == cudaSuccess) return PFX_OK;
    if (q != cudaErrorNotReady) return fail(PFX_CUDA, std::string("cudaStreamQuery: ") + cudaGetErrorString(q));
    if (std::chrono::steady_clock::now() - t0 > std::chrono::microseconds(200)) break;
  }
  PFX_CUDA_TRY(cudaStreamSynchronize(stream));
  return PFX_OK;
}

int current_device() {
  int dev = -1;
  if (cudaGetDevice(&dev) != cudaSuccess) {
    cudaGetLastError();
    return -1;
  }
  return dev;
}

int device_sms() {
  static int sms_of[kMaxDevices] = {};
  const int dev = current_device();
  if (dev < 0 || dev >= kMaxDevices) return 148;
  if (!sms_of[dev] && cudaDeviceGetAttribute(&sms_of[dev], cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) {
    cudaGetLastError();
    return 148;
  }
  return sms_of[dev];
}

int raise_smem_limit(const void* kernel, size_t bytes) {
  struct Entry {
    const void* kernel;
    int dev;
    size_t bytes;
  };
  static std::mutex mu;
  static std::vector<Entry> set;
  const int dev = current_device();
  std::lock_guard<std::mutex> lk(mu);
  for (auto& e : set)
    if (e.kernel == kernel && e.dev == dev) {
      if (e.bytes >= bytes) return PFX_OK;
      PFX_CUDA_TRY(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
      e.bytes = bytes;
      return PFX_OK;
    }
  PFX_CUDA_TRY(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
  set.push_back(Entry{kernel, dev, bytes});
  return PFX_OK;
}

// ---- per-device call lock and pivoting policy -------------------------------------
namespace {
std::recursive_mutex g_dev_mu[kMaxDevices];
std::atomic<int> g_pivot_mode{PFX_PIVOT_CHECKED};
std::atomic<long long> g_pivot_fallbacks{0};
}  // namespace

// Device-memory calls may return before their kernels finish (stream-ordered on the caller's
// stream), so the host lock alone does not keep two calls on different streams out of the
// shared workspace: every call also makes its stream wait for the previous call's
// "workspace free" event and records that event on its own stream when it returns.
cudaEvent_t g_ws_free[kMaxDevices] = {};

struct DeviceLock {
  std::unique_lock<std::recursive_mutex> lk;
  bool ok = false;
  int dev = -1;
  cudaStream_t stream = nullptr;
  explicit DeviceLock(cudaStream_t s) : stream(s) {
    dev = current_device();
    if (dev < 0 || dev >= kMaxDevices) return;
    lk = std::unique_lock<std::recursive_mutex>(g_dev_mu[dev]);
    if (!g_ws_free[dev] && cudaEventCreateWithFlags(&g_ws_free[dev], cudaEventDisableTiming) != cudaSuccess) {
      cudaGetLastError();
      return;
    }
    if (cudaStreamWaitEvent(stream, g_ws_free[dev], 0) != cudaSuccess) {
      cudaGetLastError();
      return;
    }
    ok = true;
  }
  ~DeviceLock() {
    if (ok && cudaEventRecord(g_ws_free[dev], stream) != cudaSuccess) cudaGetLastError();
  }
};
#define PFX_DEVICE_LOCK(stream)                                                    \
  ::pfx::DeviceLock _pfx_dev_lock(stream);                                         \
  if (!_pfx_dev_lock.ok) return ::pfx::fail(PFX_CUDA, "no usable CUDA device (or device index >= 16)")

int pivot_mode() { return g_pivot_mode.load(); }
void note_pivot_fallback() { g_pivot_fallbacks.fetch_add(1); }

void* scratch(int slot, size_t bytes) {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev >= kMaxDev || slot >= kSlots) return nullptr;
  std::lock_guard<std::mutex> lk(g_arena_mu);
  Arena& a = g_arena[dev];
  if (bytes == 0) bytes = 16;
  if (a.cap[slot] < bytes) {
    if (a.ptr[slot]) {
      cudaDeviceSynchronize();
      cudaFree(a.ptr[slot]);
      a.ptr[slot] = nullptr;
      a.cap[slot] = 0;
    }
    size_t want = bytes + bytes / 8;
    if (cudaMalloc(&a.ptr[slot], want) != cudaSuccess) {
      cudaGetLastError();
      return nullptr;
    }
    a.cap[slot] = want;
  }
  return a.ptr[slot];
}

void release_scratch() {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev >= kMaxDev) return;
  std::lock_guard<std::mutex> lk(g_arena_mu);
  cudaDeviceSynchronize();
  for (int s = 0; s < kSlots; ++s) {
    if (g_arena[dev].ptr[s]) cudaFree(g_arena[dev].ptr[s]);
    g_arena[dev].ptr[s] = nullptr;
    g_arena[dev].cap[s] = 0;
  }
}

// Upload poles (host, interleaved) into a device table.  Tables are cached per device by
// value and never overwritten (a kernel still reading one on another stream stays valid),
// so repeated calls with the same order neither copy nor synchronise.
namespace {
struct PoleEntry {
  std::vector<double> host;
  double2* dev = nullptr;
};
std::vector<PoleEntry> g_pole_cache[kMaxDevices];
std::mutex g_pole_mu;
// Bounded: a caller sweeping many shifts (shifted_solve in a loop) would otherwise grow the
// cache without limit.  Evicting is safe because every call returns synchronised under its
// device lock, so no kernel can still be reading an evicted table.
constexpr size_t kPoleCacheMax = 32;
}  // namespace

static void release_poles(int devid) {
  std::lock_guard<std::mutex> lk(g_pole_mu);
  for (PoleEntry& e : g_pole_cache[devid])
    if (e.dev) cudaFree(e.dev);
  g_pole_cache[devid].clear();
}

static int upload_poles(const double* theta2, const double* coef2, int npairs, cudaStream_t stream,
                        const double2** th, const double2** co) {
  const int devid = current_device();
  if (devid < 0 || devid >= kMaxDevices) return fail(PFX_CUDA, "device index out of range");
  std::vector<double> tmp(4 * (size_t)npairs);
  std::memcpy(tmp.data(), theta2, 2 * npairs * sizeof(double));
  std::memcpy(tmp.data() + 2 * npairs, coef2, 2 * npairs * sizeof(double));
  std::lock_guard<std::mutex> lk(g_pole_mu);
  for (const PoleEntry& e : g_pole_cache[devid])
    if (e.host == tmp) {
      *th = e.dev;
      *co = e.dev + npairs;
      return PFX_OK;
    }
  if (g_pole_cache[devid].size() >= kPoleCacheMax) {
    cudaFree(g_pole_cache[devid].front().dev);
    g_pole_cache[devid].erase(g_pole_cache[devid].begin());
  }
  PoleEntry e;
  e.host = tmp;
  PFX_CUDA_TRY(cudaMalloc(&e.dev, tmp.size() * sizeof(double)));
  PFX_CUDA_TRY(cudaMemcpyAsync(e.dev, tmp.data(), tmp.size() * sizeof(double), cudaMemcpyHostToDevice, stream));
  if (int rc_ = sync_stream(stream)) return rc_;
  g_pole_cache[devid].push_back(e);
  *th = e.dev;
  *co = e.dev + npairs;
  return PFX_OK;
}

static int check_poles(const double* theta2, const double* coef2, int npairs) {
  if (!theta2 || !coef2) return fail(PFX_BADARG, "theta2/coef2 must be non-null host arrays");
  if (npairs < 1 || npairs > 32) return fail(PFX_BADARG, "npairs must be in [1, 32]");
  for (int k = 0; k < npairs; ++k) {
    if (!std::isfinite(theta2[2 * k]) || !std::isfinite(theta2[2 * k + 1]) || !std::isfinite(coef2[2 * k]) ||
        !std::isfinite(coef2[2 * k + 1]))
      return fail(PFX_BADARG, "non-finite pole or residue");
    if (!(theta2[2 * k + 1] > 0.0)) return fail(PFX_BADARG, "pole representatives must have Im(theta) > 0");
  }
  return PFX_OK;
}

// Pivoting argument of the dense kernels (pfx_set_pivot_mode; PFX_DENSE_PIVOT=1 in the
// environment forces ALWAYS, for A/B checks): 0 = interchange-free, unchecked; 1 = partial
// pivoting (getrf interchanges); 2 = checked: the interchange-free factorisation verifies that
// partial pivoting would have chosen every diagonal pivot, else the call refactors with
// interchanges.
static int dense_pivot_arg() {
  static const bool force_piv = getenv("PFX_DENSE_PIVOT") != nullptr;
  if (force_piv) return 1;
  switch (pivot_mode()) {
    case PFX_PIVOT_ALWAYS: return 1;
    case PFX_PIVOT_NONE: return 0;
    default: return 2;
  }
}

// Host staging: copy host inputs into arena slots 3..5, output into slot 6.
struct Staged {
  const double* in[3] = {nullptr, nullptr, nullptr};
  double* out = nullptr;
};

static int stage_in(int mem, int slot, const double* src, size_t bytes, cudaStream_t stream, const double** dst) {
  if (mem == PFX_MEM_DEVICE || src == nullptr || bytes == 0) {
    *dst = src;
    return PFX_OK;
  }
  void* p = scratch(slot, bytes);
  if (!p) return fail(PFX_CUDA, "staging allocation failed");
  PFX_CUDA_TRY(cudaMemcpyAsync(p, src, bytes, cudaMemcpyHostToDevice, stream));
  *dst = static_cast<const double*>(p);
  return PFX_OK;
}

}  // namespace pfx

using namespace pfx;

extern "C" {

int pfx_version(void) { return 100; }

int pfx_prof_enable(int on) {
  g_prof_on = on != 0;
  return PFX_OK;
}

int pfx_prof_read(char* buf, int buflen) {
  std::lock_guard<std::mutex> lk(g_prof_mu);
  std::vector<std::string> names;
  std::vector<int> counts;
  std::vector<double> totals;
  std::vector<double> fl;
  // PFX_PROF_TIMELINE=<file>: every launch's (name, stream, start, end) in ms from the first
  // launch appended to <file> (critical-path analysis of the multi-stream band steps)
  static const char* tl_path = getenv("PFX_PROF_TIMELINE");
  FILE* tl = (tl_path && !g_prof.empty()) ? fopen(tl_path, "a") : nullptr;
  if (tl) {
    cudaEventSynchronize(g_prof.back().e1);
    fprintf(tl, "# timeline %zu launches\n", g_prof.size());
  }
  // the timeline pass runs before any event is destroyed (every record is timed against the
  // first launch's start event)
  if (tl) {
    for (auto& r : g_prof) {
      cudaEventSynchronize(r.e1);
      float a = 0.0f, b = 0.0f;
      cudaEventElapsedTime(&a, g_prof.front().e0, r.e0);
      cudaEventElapsedTime(&b, g_prof.front().e0, r.e1);
      fprintf(tl, "%s %p %.4f %.4f\n", r.name.c_str(), (void*)r.stream, a * 1e3, b * 1e3);
    }
  }
  for (auto& r : g_prof) {
    cudaEventSynchronize(r.e1);
    float ms = 0.0f;
    cudaEventElapsedTime(&ms, r.e0, r.e1);
    cudaEventDestroy(r.e0);
    cudaEventDestroy(r.e1);
    size_t i = 0;
    for (; i < names.size(); ++i)
      if (names[i] == r.name) break;
    if (i == names.size()) {
      names.push_back(r.name);
      counts.push_back(0);
      totals.push_back(0.0);
      fl.push_back(0.0);
    }
    counts[i] += 1;
    totals[i] += ms;
    fl[i] += r.flops;
  }
  if (tl) fclose(tl);
  g_prof.clear();
  std::string out;
  char line[256];
  for (size_t i = 0; i < names.size(); ++i) {
    snprintf(line, sizeof(line), "%s %d %.6f %.6e\n", names[i].c_str(), counts[i], totals[i], fl[i]);
    out += line;
  }
  if (buf && buflen > 0) {
    size_t n = std::min<size_t>(out.size(), (size_t)buflen - 1);
    memcpy(buf, out.data(), n);
    buf[n] = 0;
  }
  return (int)out.size() + 1;
}

const char* pfx_last_error(void) { return g_err.c_str(); }

int pfx_release(void) {
  PFX_DEVICE_LOCK(nullptr);
  release_scratch();
  release_poles(current_device());
  return PFX_OK;
}

int pfx_set_pivot_mode(int mode) {
  if (mode != PFX_PIVOT_CHECKED && mode != PFX_PIVOT_ALWAYS && mode != PFX_PIVOT_NONE)
    return fail(PFX_BADARG, "pivot mode must be PFX_PIVOT_CHECKED, PFX_PIVOT_ALWAYS or PFX_PIVOT_NONE");
  g_pivot_mode.store(mode);
  return PFX_OK;
}

int pfx_get_pivot_mode(void) { return g_pivot_mode.load(); }

long long pfx_pivot_fallbacks(void) { return g_pivot_fallbacks.load(); }

int pfx_pole_table(int n, double* theta2, double* coef2) {
  if (!theta2 || !coef2) return fail(PFX_BADARG, "null output array");
  if (n < 2 || n > 64 || (n & 1)) return fail(PFX_BADARG, "order must be even and in [2, 64]");
  return pole_table_host(n, theta2, coef2);
}

int pfx_expm_dense(int mem, const double* A, int a_complex, int64_t d, int64_t batch, const double* V,
                   int v_complex, int64_t nrhs, double shift_c, const double* theta2, const double* coef2,
                   int npairs, double* out, int out_complex, float* per_pair_ms, void* stream_) {
  g_err.clear();
  cudaStream_t stream = static_cast<cudaStream_t>(stream_);
  if (mem != PFX_MEM_DEVICE && mem != PFX_MEM_HOST) return fail(PFX_BADARG, "mem must be PFX_MEM_DEVICE or PFX_MEM_HOST");
  if (!A || !out) return fail(PFX_BADARG, "A and out must be non-null");
  if (d < 1 || batch < 1 || nrhs < 0) return fail(PFX_BADARG, "need d >= 1, batch >= 1, nrhs >= 0");
  if (nrhs > 0 && !V) return fail(PFX_BADARG, "action mode needs V");
  if (!std::isfinite(shift_c)) return fail(PFX_BADARG, "shift must be finite");
  int rc = check_poles(theta2, coef2, npairs);
  if (rc) return rc;
  const int full = nrhs == 0;
  const int real_path = (!a_complex) && (full || !v_complex);
  if (out_complex != !real_path)
    return fail(PFX_BADARG, "out_complex must be 1 exactly when A is complex or V is complex (engine.py:185)");
  const int ncols = full ? (int)d : (int)nrhs;
  if (!dense_batched_supported(d) && batch != 1)
    return fail(PFX_BADARG, "batched dense path supports d <= 512; larger matrices must be passed one at a time");
  const size_t abytes = (size_t)batch * d * d * sizeof(double) * (a_complex ? 2 : 1);
  const size_t vbytes = full ? 0 : (size_t)batch * d * nrhs * sizeof(double) * (v_complex ? 2 : 1);
  const size_t obytes = (size_t)batch * d * ncols * sizeof(double) * (out_complex ? 2 : 1);
  PFX_DEVICE_LOCK(stream);  // argument checks above need no device
  const double2 *th = nullptr, *co = nullptr;
  rc = upload_poles(theta2, coef2, npairs, stream, &th, &co);
  if (rc) return rc;
  if (mem == PFX_MEM_HOST && dense_batched_supported(d) && batch > 1) {
    // Host batches: the matrices go in by chunks on a copy stream and each chunk is factored
    // as soon as it has landed, so the copy-in hides behind the factorisations.  Chunks hold
    // five rounds of the resident CTAs' systems (whole rounds: no extra tail); the remainder
    // goes first, where its short copy starts the pipeline.
    const int64_t slots = dense_batched_slots((int)d, batch * npairs);
    const int64_t per = std::max<int64_t>(1, slots * 5 / npairs);
    if (batch >= 2 * per) {
      static cudaStream_t cins[kMaxDevices] = {};
      static std::vector<cudaEvent_t> evss[kMaxDevices];
      const int dev = current_device();
      cudaStream_t& cin = cins[dev];
      std::vector<cudaEvent_t>& evs = evss[dev];
      if (!cin) PFX_CUDA_TRY(cudaStreamCreateWithFlags(&cin, cudaStreamNonBlocking));
      const int64_t first = batch % per ? batch % per : per;
      const int64_t nch = 1 + (batch - first + per - 1) / per;
      while ((int64_t)evs.size() < nch + 1) {
        cudaEvent_t e;
        PFX_CUDA_TRY(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        evs.push_back(e);
      }
      const size_t am = abytes / batch, vm = vbytes / batch, om = obytes / batch;  // bytes per matrix
      char* Ad = static_cast<char*>(scratch(3, abytes));
      char* Vd = vbytes ? static_cast<char*>(scratch(4, vbytes)) : nullptr;
      char* Od = static_cast<char*>(scratch(6, obytes));
      if (!Ad || (vbytes && !Vd) || !Od) return fail(PFX_CUDA, "staging allocation failed");
      // the staging buffers are idle on entry (host-mode calls end synchronised)
      PFX_CUDA_TRY(cudaEventRecord(evs[nch], stream));  // poles uploaded
      PFX_CUDA_TRY(cudaStreamWaitEvent(cin, evs[nch], 0));
      auto chunk = [&](int64_t i, int64_t& b0, int64_t& nb) {
        b0 = i == 0 ? 0 : first + (i - 1) * per;
        nb = i == 0 ? first : std::min(per, batch - b0);
      };
      for (int64_t i = 0; i < nch; ++i) {
        int64_t b0, nb;
        chunk(i, b0, nb);
        PFX_CUDA_TRY(cudaMemcpyAsync(Ad + b0 * am, reinterpret_cast<const char*>(A) + b0 * am, nb * am,
                                     cudaMemcpyHostToDevice, cin));
        if (vbytes)
          PFX_CUDA_TRY(cudaMemcpyAsync(Vd + b0 * vm, reinterpret_cast<const char*>(V) + b0 * vm, nb * vm,
                                       cudaMemcpyHostToDevice, cin));
        PFX_CUDA_TRY(cudaEventRecord(evs[i], cin));
      }
      const int pivot = dense_pivot_arg();
      float tot = 0.0f;
      for (int64_t i = 0; i < nch; ++i) {
        int64_t b0, nb;
        chunk(i, b0, nb);
        PFX_CUDA_TRY(cudaStreamWaitEvent(stream, evs[i], 0));
        float ms = 0.0f;
        // returns synchronised (status word); the next chunk's copy is already in flight
        rc = dense_small_run(reinterpret_cast<const double*>(Ad + b0 * am), a_complex, (int)d, (int)nb,
                             vbytes ? reinterpret_cast<const double*>(Vd + b0 * vm) : nullptr, v_complex, ncols, full,
                             real_path, shift_c, th, co, npairs, reinterpret_cast<double*>(Od + b0 * om), stream,
                             per_pair_ms ? &ms : nullptr, pivot);
        if (rc) return rc;
        tot += ms;
        PFX_CUDA_TRY(cudaMemcpyAsync(reinterpret_cast<char*>(out) + b0 * om, Od + b0 * om, nb * om,
                                     cudaMemcpyDeviceToHost, stream));
      }
      if (per_pair_ms)
        for (int k = 0; k < npairs; ++k) per_pair_ms[k] = tot;
      return sync_stream(stream);
    }
  }
  if (mem == PFX_MEM_HOST && !dense_batched_supported(d)) {
    // large matrices: dense_large_run pipelines the copies (row chunks in, row chunks out)
    double* Ad = static_cast<double*>(scratch(3, abytes));
    double* Vd = vbytes ? static_cast<double*>(scratch(4, vbytes)) : nullptr;
    double* Od = static_cast<double*>(scratch(6, obytes));
    if (!Ad || (vbytes && !Vd) || !Od) return fail(PFX_CUDA, "staging allocation failed");
    rc = dense_large_run(Ad, a_complex, (int)d, Vd, v_complex, ncols, full, real_path, shift_c, th, co, npairs, Od,
                         stream, per_pair_ms, dense_pivot_arg(), A, V, out);
    return rc;
  }
  const double *Ad = nullptr, *Vd = nullptr;
  if ((rc = stage_in(mem, 3, A, abytes, stream, &Ad))) return rc;
  if ((rc = stage_in(mem, 4, V, vbytes, stream, &Vd))) return rc;
  double* Od = out;
  if (mem == PFX_MEM_HOST) {
    Od = static_cast<double*>(scratch(6, obytes));
    if (!Od) return fail(PFX_CUDA, "staging allocation failed");
  }
  float ms = 0.0f;
  if (dense_batched_supported(d)) {
    const int pivot = dense_pivot_arg();
    rc = dense_small_run(Ad, a_complex, (int)d, (int)batch, Vd, v_complex, ncols, full, real_path, shift_c, th, co,
                         npairs, Od, stream, per_pair_ms ? &ms : nullptr, pivot);
    if (per_pair_ms)
      for (int k = 0; k < npairs; ++k) per_pair_ms[k] = ms;
  } else {
    rc = dense_large_run(Ad, a_complex, (int)d, Vd, v_complex, ncols, full, real_path, shift_c, th, co, npairs, Od,
                         stream, per_pair_ms, dense_pivot_arg());
  }
  if (rc) return rc;
  if (mem == PFX_MEM_HOST) {
    PFX_CUDA_TRY(cudaMemcpyAsync(out, Od, obytes, cudaMemcpyDeviceToHost, stream));
    if (int rc_ = sync_stream(stream)) return rc_;
  }
  return PFX_OK;
}

int pfx_expm_dense_cols(int mem, const double* A, int a_complex, int64_t d, double shift_c, const double* theta2,
                        const double* coef2, int npairs, const int64_t* col_ranges, double* out, int out_complex,
                        int accumulate, void* stream_) {
  g_err.clear();
  cudaStream_t stream = static_cast<cudaStream_t>(stream_);
  if (mem != PFX_MEM_DEVICE && mem != PFX_MEM_HOST) return fail(PFX_BADARG, "mem must be PFX_MEM_DEVICE or PFX_MEM_HOST");
  if (!A || !out || !col_ranges) return fail(PFX_BADARG, "A, out and col_ranges must be non-null");
  if (dense_batched_supported(d) || d > (1 << 20))
    return fail(PFX_BADARG, "the column split applies to the blocked large path (d > 512)");
  if (!std::isfinite(shift_c)) return fail(PFX_BADARG, "shift must be finite");
  int rc = check_poles(theta2, coef2, npairs);
  if (rc) return rc;
  if (out_complex != (a_complex ? 1 : 0))
    return fail(PFX_BADARG, "out_complex must be 1 exactly when A is complex (engine.py:185)");
  for (int k = 0; k < npairs; ++k) {
    const int64_t c0 = col_ranges[2 * k], c1 = col_ranges[2 * k + 1];
    if (c0 < 0 || c1 <= c0 || c1 > d || c0 % 64 != 0)
      return fail(PFX_BADARG, "column ranges need 0 <= c0 < c1 <= d with c0 a multiple of 64");
  }
  const size_t abytes = (size_t)d * d * sizeof(double) * (a_complex ? 2 : 1);
  const size_t obytes = (size_t)d * d * sizeof(double) * (out_complex ? 2 : 1);
  PFX_DEVICE_LOCK(stream);
  const double2 *th = nullptr, *co = nullptr;
  if ((rc = upload_poles(theta2, coef2, npairs, stream, &th, &co))) return rc;
  const double* Ad = nullptr;
  if ((rc = stage_in(mem, 3, A, abytes, stream, &Ad))) return rc;
  double* Od = out;
  if (mem == PFX_MEM_HOST) {
    Od = static_cast<double*>(scratch(6, obytes));
    if (!Od) return fail(PFX_CUDA, "staging allocation failed");
    if (accumulate) PFX_CUDA_TRY(cudaMemcpyAsync(Od, out, obytes, cudaMemcpyHostToDevice, stream));
  }
  rc = dense_large_cols_run(Ad, a_complex, (int)d, shift_c, th, co, npairs, col_ranges, Od, accumulate, stream,
                            dense_pivot_arg());
  if (rc) return rc;
  if (mem == PFX_MEM_HOST) {
    PFX_CUDA_TRY(cudaMemcpyAsync(out, Od, obytes, cudaMemcpyDeviceToHost, stream));
    if (int rc_ = sync_stream(stream)) return rc_;
  }
  return PFX_OK;
}

int pfx_expm_tridiag(int mem, const double* diag, const double* off, int64_t N, const double* V, int64_t nrhs,
                     double shift_c, const double* theta2, const double* coef2, int npairs, double* out,
                     float* per_pair_ms, void* stream_) {
  g_err.clear();
  cudaStream_t stream = static_cast<cudaStream_t>(stream_);
  if (mem != PFX_MEM_DEVICE && mem != PFX_MEM_HOST) return fail(PFX_BADARG, "bad mem kind");
  if (N < 1 || nrhs < 1) return fail(PFX_BADARG, "need N >= 1 and nrhs >= 1");
  if (!diag || !V || !out || (N > 1 && !off)) return fail(PFX_BADARG, "null array");
  if (!std::isfinite(shift_c)) return fail(PFX_BADARG, "shift must be finite");
  int rc = check_poles(theta2, coef2, npairs);
  if (rc) return rc;
  PFX_DEVICE_LOCK(stream);  // argument checks above need no device
  const double2 *th = nullptr, *co = nullptr;
  if ((rc = upload_poles(theta2, coef2, npairs, stream, &th, &co))) return rc;
  const double *Dd = nullptr, *Od_ = nullptr, *Vd = nullptr;
  const size_t vbytes = (size_t)N * nrhs * sizeof(double);
  // host mode on the on-chip path (npairs <= 16): V and out move in row groups overlapped
  // with the sweeps / fixes (tridiag_run); otherwise staged whole
  const bool pipe = mem == PFX_MEM_HOST && npairs <= 16;
  if ((rc = stage_in(mem, 3, diag, N * sizeof(double), stream, &Dd))) return rc;
  if ((rc = stage_in(mem, 4, off, (N - 1) * sizeof(double), stream, &Od_))) return rc;
  if (pipe) {
    Vd = static_cast<const double*>(scratch(5, vbytes));
    if (!Vd) return fail(PFX_CUDA, "staging allocation failed");
  } else if ((rc = stage_in(mem, 5, V, vbytes, stream, &Vd))) {
    return rc;
  }
  double* Out = out;
  const size_t obytes = vbytes;
  if (mem == PFX_MEM_HOST) {
    Out = static_cast<double*>(scratch(6, obytes));
    if (!Out) return fail(PFX_CUDA, "staging allocation failed");
  }
  float ms = 0.0f;
  rc = tridiag_run(Dd, Od_, N, Vd, nrhs, shift_c, th, co, npairs, Out, stream, per_pair_ms ? &ms : nullptr,
                   pipe ? V : nullptr, pipe ? out : nullptr);
  if (rc) return rc;
  if (per_pair_ms)
    for (int k = 0; k < npairs; ++k) per_pair_ms[k] = ms;
  if (mem == PFX_MEM_HOST) {
    if (!pipe) PFX_CUDA_TRY(cudaMemcpyAsync(out, Out, obytes, cudaMemcpyDeviceToHost, stream));
    if (int rc_ = sync_stream(stream)) return rc_;
  }
  return PFX_OK;
}

int pfx_tridiag_shard_rows(int64_t N, int64_t nrhs, int rank, int nranks, int64_t* r0, int64_t* r1) {
  g_err.clear();
  if (N < 1 || nrhs < 1 || nranks < 1 || rank < 0 || rank >= nranks || !r0 || !r1)
    return fail(PFX_BADARG, "bad shard arguments");
  int L = 0, P = 0;
  int64_t c0 = 0, c1 = 0;
  if (int rc = tri_partition(N, nrhs, rank, nranks, &L, &P, &c0, &c1)) return rc;
  *r0 = std::min<int64_t>(c0 * L, N);
  *r1 = std::min<int64_t>(c1 * L, N);
  return PFX_OK;
}

int pfx_expm_tridiag_shard(const double* diag, const double* off, int64_t N, const double* V, int64_t nrhs,
                           double shift_c, const double* theta2, const double* coef2, int npairs, double* out,
                           int rank, int nranks, pfx_allgather_fn allgather, void* ctx, void* stream_) {
  g_err.clear();
  cudaStream_t stream = static_cast<cudaStream_t>(stream_);
  if (N < 1 || nrhs < 1) return fail(PFX_BADARG, "need N >= 1 and nrhs >= 1");
  if (!diag || !V || !out || (N > 1 && !off)) return fail(PFX_BADARG, "null array");
  if (nranks < 1 || rank < 0 || rank >= nranks || (nranks > 1 && !allgather)) return fail(PFX_BADARG, "bad shard arguments");
  if (!std::isfinite(shift_c)) return fail(PFX_BADARG, "shift must be finite");
  int rc = check_poles(theta2, coef2, npairs);
  if (rc) return rc;
  if (npairs > 16) return fail(PFX_BADARG, "row sharding needs npairs <= 16 (n <= 32)");
  PFX_DEVICE_LOCK(stream);  // argument checks above need no device
  const double2 *th = nullptr, *co = nullptr;
  if ((rc = upload_poles(theta2, coef2, npairs, stream, &th, &co))) return rc;
  TriShard sh{rank, nranks, allgather, ctx};
  return tridiag_run(diag, off, N, V, nrhs, shift_c, th, co, npairs, out, stream, nullptr, nullptr, nullptr, &sh);
}

int pfx_expm_banded(int mem, const double* band, int64_t N, int64_t kb, const double* V, int64_t nrhs,
                    double shift_c, const double* theta2, const double* coef2, int npairs, double* out,
                    float* per_pair_ms, void* stream_) {
  g_err.clear();
  cudaStream_t stream = static_cast<cudaStream_t>(stream_);
  if (mem != PFX_MEM_DEVICE && mem != PFX_MEM_HOST) return fail(PFX_BADARG, "bad mem kind");
  if (N < 1 || nrhs < 1 || kb < 0) return fail(PFX_BADARG, "need N >= 1, nrhs >= 1, kb >= 0");
  if (!band || !V || !out) return fail(PFX_BADARG, "null array");
  if (!std::isfinite(shift_c)) return fail(PFX_BADARG, "shift must be finite");
  int rc = check_poles(theta2, coef2, npairs);
  if (rc) return rc;
  PFX_DEVICE_LOCK(stream);  // argument checks above need no device
  const double2 *th = nullptr, *co = nullptr;
  if ((rc = upload_poles(theta2, coef2, npairs, stream, &th, &co))) return rc;
  const double *Bd = nullptr, *Vd = nullptr;
  if (mem == PFX_MEM_HOST) {  // copied in by row chunks inside banded_run, overlapping the build
    Bd = static_cast<const double*>(scratch(3, (size_t)(kb + 1) * N * sizeof(double)));
    Vd = static_cast<const double*>(scratch(5, (size_t)N * nrhs * sizeof(double)));
    if (!Bd || !Vd) return fail(PFX_CUDA, "staging allocation failed");
  } else {
    Bd = band;
    Vd = V;
  }
  double* Out = out;
  const size_t obytes = (size_t)N * nrhs * sizeof(double);
  if (mem == PFX_MEM_HOST) {
    Out = static_cast<double*>(scratch(6, obytes));
    if (!Out) return fail(PFX_CUDA, "staging allocation failed");
  }
  rc = banded_run(Bd, N, kb, Vd, nrhs, shift_c, th, co, npairs, Out, stream, per_pair_ms,
                  mem == PFX_MEM_HOST ? band : nullptr, mem == PFX_MEM_HOST ? V : nullptr);
  if (rc) return rc;
  if (mem == PFX_MEM_HOST) {
    PFX_CUDA_TRY(cudaMemcpyAsync(out, Out, obytes, cudaMemcpyDeviceToHost, stream));
    if (int rc_ = sync_stream(stream)) return rc_;
  }
  return PFX_OK;
}

int pfx_shifted_solve(int mem, const double* A, int a_complex, int64_t d, double theta_re, double theta_im,
                      const double* V, int64_t nrhs, double* Y, void* stream_) {
  g_err.clear();
  cudaStream_t stream = static_cast<cudaStream_t>(stream_);
  if (mem != PFX_MEM_DEVICE && mem != PFX_MEM_HOST) return fail(PFX_BADARG, "bad mem kind");
  if (!A || !V || !Y || d < 1 || nrhs < 1) return fail(PFX_BADARG, "need A, V, Y non-null, d >= 1, nrhs >= 1");
  if (!std::isfinite(theta_re) || !std::isfinite(theta_im)) return fail(PFX_BADARG, "non-finite shift");
  // one system, residue 1: stage = Y = (A + theta I)^{-1} V (complex V, complex Y)
  double th2[2] = {theta_re, theta_im}, co2[2] = {1.0, 0.0};
  PFX_DEVICE_LOCK(stream);  // argument checks above need no device
  const double2 *th = nullptr, *co = nullptr;
  int rc = upload_poles(th2, co2, 1, stream, &th, &co);
  if (rc) return rc;
  const size_t abytes = (size_t)d * d * sizeof(double) * (a_complex ? 2 : 1);
  const size_t vbytes = (size_t)d * nrhs * 2 * sizeof(double);
  const double *Ad = nullptr, *Vd = nullptr;
  if ((rc = stage_in(mem, 3, A, abytes, stream, &Ad))) return rc;
  if ((rc = stage_in(mem, 4, V, vbytes, stream, &Vd))) return rc;
  double* Yd = Y;
  if (mem == PFX_MEM_HOST) {
    Yd = static_cast<double*>(scratch(6, vbytes));
    if (!Yd) return fail(PFX_CUDA, "staging allocation failed");
  }
  if (dense_batched_supported(d))
    rc = dense_batched_run(Ad, a_complex, (int)d, 1, Vd, 1, (int)nrhs, 0, 0, 1, 0.0, th, co, 1, Yd, stream, nullptr,
                           1);  // general shift: partial pivoting
  else
    rc = shifted_solve_large(Ad, a_complex, (int)d, th, Vd, (int)nrhs, reinterpret_cast<double2*>(Yd), stream);
  if (rc) return rc;
  if (mem == PFX_MEM_HOST) {
    PFX_CUDA_TRY(cudaMemcpyAsync(Y, Yd, vbytes, cudaMemcpyDeviceToHost, stream));
    if (int rc_ = sync_stream(stream)) return rc_;
  }
  return PFX_OK;
}

}  // extern "C"
