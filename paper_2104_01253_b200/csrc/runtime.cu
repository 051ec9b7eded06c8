// Error reporting and device queries behind the C-ABI.
#include "common.cuh"

#include <cstdlib>

#include <cstdarg>
#include <cstdio>
#include <mutex>

namespace kls {

static thread_local char g_err[512] = "";

int fail(int code, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
  return code;
}

int check_launch(const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(KLS_ECUDA, "%s: %s", what, cudaGetErrorString(e));
  return KLS_OK;
}

int sm_count() {
  static int cache[64] = {0};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return 148;
  if (cache[dev] == 0) {
    int n = 0;
    if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n <= 0)
      n = 148;
    cache[dev] = n;
  }
  return cache[dev];
}

}  // namespace kls

KLS_API int kls_version(void) { return 1; }

KLS_API const char* kls_last_error(void) { return kls::g_err; }

KLS_API int kls_device_sm_count(void) { return kls::sm_count(); }

// Block the host until all work queued on `stream` has finished.
KLS_API int kls_stream_sync(void* stream) {
  cudaError_t e = cudaStreamSynchronize(static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return kls::fail(KLS_ECUDA, "stream sync: %s", cudaGetErrorString(e));
  return KLS_OK;
}

// Device-side address of page-locked host memory (for kernels that write
// their few reduced scalars straight to the host).
KLS_API int kls_host_device_ptr(void* host, void** dev) {
  if (host == nullptr || dev == nullptr) return kls::fail(KLS_EINVAL, "host_device_ptr: null");
  cudaError_t e = cudaHostGetDevicePointer(dev, host, 0);
  if (e != cudaSuccess) return kls::fail(KLS_ECUDA, "host_device_ptr: %s", cudaGetErrorString(e));
  return KLS_OK;
}

namespace kls {
bool pdl_enabled() {
  static const bool on = [] {
    const char* e = getenv("KLS_PDL");
    return !(e != nullptr && e[0] == '0');
  }();
  return on;
}
}  // namespace kls
