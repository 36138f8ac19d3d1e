// Library-level entry points: version, error text, device probe.
#include "kvlc_common.cuh"

#include <mutex>

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
// launch) and issues cache reads (code stream, chunk counts, residual window) before
// griddepcontrol.wait.  Entry points that write cache state mark their stream; the next
// decode on a marked stream launches without the overlap.  Per host thread, last 8 streams.
namespace {
thread_local void* tl_dirty[8];
thread_local int tl_ndirty = 0;
}  // namespace

void note_cache_write(void* stream) {
  for (int i = 0; i < tl_ndirty; ++i)
    if (tl_dirty[i] == stream) return;
  if (tl_ndirty < 8) {
    tl_dirty[tl_ndirty++] = stream;
  } else {
    for (int i = 1; i < 8; ++i) tl_dirty[i - 1] = tl_dirty[i];
    tl_dirty[7] = stream;
  }
}

bool take_cache_write(void* stream) {
  for (int i = 0; i < tl_ndirty; ++i)
    if (tl_dirty[i] == stream) {
      tl_dirty[i] = tl_dirty[--tl_ndirty];
      return true;
    }
  return false;
}

}  // namespace kvlc

extern "C" {

int kvlc_version(void) { return 10000; /* 1.0.0 */ }

const char* kvlc_last_error(void) { return kvlc::g_err; }

int kvlc_device_ok(void) { return kvlc::device_ok() ? 1 : 0; }

}  // extern "C"
