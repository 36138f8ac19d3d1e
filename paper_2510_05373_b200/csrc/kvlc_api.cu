// Library-level entry points: version, error text, device probe.
#include "kvlc_common.cuh"

#include <mutex>
#include <unordered_set>

namespace kvlc {

static thread_local char g_err[512] = "";

void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

int fail(int code, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
  return code;
}

int check_launch(const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(KVLC_ECUDA, "%s launch failed: %s", what, cudaGetErrorString(e));
  return KVLC_OK;
}

bool device_ok() {
  static int cached = -1;
  static std::mutex mu;
  std::lock_guard<std::mutex> lock(mu);
  if (cached < 0) {
    int dev = 0, major = 0, n = 0;
    cached = 0;
    if (cudaGetDeviceCount(&n) == cudaSuccess && n > 0 && cudaGetDevice(&dev) == cudaSuccess &&
        cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev) == cudaSuccess)
      cached = major == 10 ? 1 : 0;
    cudaGetLastError();
  }
  return cached == 1;
}

// The decode launch overlaps the previous kernel on its stream (programmatic dependent
// launch) and issues its first chunks' code copies before griddepcontrol.wait.  Entry
// points that write codes or chunk counts mark the CACHE (keyed by its code buffer, so
// the mark is independent of host thread and stream); the next decode of a marked cache
// launches without the overlap and clears the mark.  Writers outside the library call
// kvlc_note_cache_write().
namespace {
std::mutex g_dirty_mu;
std::unordered_set<const void*> g_dirty;
}  // namespace

void note_cache_write(const kvlc_cache* c) {
  if (!c) return;
  std::lock_guard<std::mutex> lock(g_dirty_mu);
  g_dirty.insert(c->kcodes);
}

bool take_cache_write(const kvlc_cache* c) {
  std::lock_guard<std::mutex> lock(g_dirty_mu);
  return g_dirty.erase(c->kcodes) > 0;
}

}  // namespace kvlc

extern "C" {

int kvlc_version(void) { return 10000; /* 1.0.0 */ }

const char* kvlc_last_error(void) { return kvlc::g_err; }

int kvlc_device_ok(void) { return kvlc::device_ok() ? 1 : 0; }

void kvlc_note_cache_write(const kvlc_cache* c) { kvlc::note_cache_write(c); }

}  // extern "C"
