// Status plumbing of the C ABI (include/tokencarve_b200.h).
#include "common.cuh"

namespace tcb {

static thread_local char g_err[1024] = "";

int set_error(int code, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
  return code;
}

int check_launch(const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return set_error(TCB_ECUDA, "%s: %s", what, cudaGetErrorString(e));
  return TCB_OK;
}

}  // namespace tcb

extern "C" const char* tcb_last_error(void) { return tcb::g_err; }

extern "C" int tcb_abi_version(void) { return 2; }  // 2: packed-bit masks, no kv_idx
