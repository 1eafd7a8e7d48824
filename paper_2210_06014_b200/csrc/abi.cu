// Error plumbing and device queries of the C ABI (include/ft_b200.h).
#include <stdarg.h>
#include <string.h>

#include "ft_common.cuh"

namespace ft {

static thread_local char g_err[1024] = "";

void set_error(const char *fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

int fail(ft_status st, const char *fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
  return (int)st;
}

int check_launch(const char *what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(FT_ERR_CUDA, "%s launch: %s", what, cudaGetErrorString(e));
  return FT_OK;
}

// The builder / generator / evaluator take their scratch stream-ordered from the device's
// default memory pool.  Keep freed blocks in the pool (release threshold = max) so repeated
// builds do not map and unmap gigabytes each time.
void keep_pool() {
  static int done = 0;
  if (done) return;
  int dev = 0;
  cudaMemPool_t pool;
  if (cudaGetDevice(&dev) == cudaSuccess && cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
    uint64_t thr = ~0ull;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
  }
  done = 1;
}

int sm_count() {
  static int cached = 0;
  if (!cached) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&cached, cudaDevAttrMultiProcessorCount, dev);
    if (cached <= 0) cached = 148;
  }
  return cached;
}

}  // namespace ft

extern "C" const char *ft_last_error(void) { return ft::g_err; }

extern "C" int ft_abi_version(void) { return 2; }

extern "C" int ft_sm_count(int32_t *out) {
  if (!out) return ft::fail(FT_ERR_ARG, "ft_sm_count: null out");
  int dev = 0;
  FT_CUDA(cudaGetDevice(&dev));
  int n = 0;
  FT_CUDA(cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev));
  *out = n;
  return FT_OK;
}
