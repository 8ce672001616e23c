// Library-level C ABI: version, thread-local last-error string.
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include "common.cuh"

namespace nirc {

static thread_local char g_last_error[512] = {0};

void set_last_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_last_error, sizeof(g_last_error), fmt, ap);
  va_end(ap);
}

int check_cuda(cudaError_t e, const char* what) {
  set_last_error("%s: %s", what, cudaGetErrorString(e));
  return NIRC_E_CUDA;
}

}  // namespace nirc

extern "C" const char* nirc_version(void) { return "nirc_b200 0.1.0 sm_100a"; }

extern "C" int nirc_last_error(char* buf, int buflen) {
  if (!buf || buflen <= 0) return (int)strlen(nirc::g_last_error);
  snprintf(buf, (size_t)buflen, "%s", nirc::g_last_error);
  return (int)strlen(buf);
}
