// C-ABI housekeeping: version, thread-local error text, device sync helper.
#include <cstdlib>
#include <cstdarg>
#include <cstdio>

#include "common.cuh"

namespace gfm {
static thread_local char g_err[512] = "";
static int g_gemm_mode = GFM_GEMM_TC3;

int gemm_mode() { return g_gemm_mode; }
// launches of the CTA-pair GEMM kernel since load (tests assert the path ran)
long long g_pair_launches = 0;
// CTA-pair GEMM kernels (default on; GFM_TC_PAIR=0 at first use or
// gfm_set_tc_pairs(0) selects the single-CTA kernels)
static int g_tc_pairs = -1;
bool tc_pairs() {
  if (g_tc_pairs < 0) g_tc_pairs = getenv("GFM_TC_PAIR") ? atoi(getenv("GFM_TC_PAIR")) : 1;
  return g_tc_pairs != 0;
}
bool pdl_enabled() {
  static const bool v = [] {
    const char* e = getenv("GFM_NO_PDL");
    return !(e && e[0] == '1');
  }();
  return v;
}

void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}
}  // namespace gfm

extern "C" {

int gfm_abi_version(void) { return GFM_ABI_VERSION; }

const char* gfm_last_error(void) { return gfm::g_err; }

int gfm_device_sm_count(void) { return gfm::num_sms(); }

int gfm_set_gemm_mode(int mode) {
  if (mode != GFM_GEMM_SIMT && mode != GFM_GEMM_TC3 && mode != GFM_GEMM_TC1 &&
      mode != GFM_GEMM_MIXED) {
    gfm::set_error("gfm_set_gemm_mode: unknown mode %d", mode);
    return GFM_EINVAL;
  }
  gfm::g_gemm_mode = mode;
  return 0;
}

int gfm_get_gemm_mode(void) { return gfm::g_gemm_mode; }

long long gfm_tc_pair_launches(void) { return gfm::g_pair_launches; }

int gfm_set_tc_pairs(int on) {
  const int prev = gfm::tc_pairs() ? 1 : 0;
  gfm::g_tc_pairs = on ? 1 : 0;
  return prev;
}

int gfm_stream_sync(void* stream) {
  cudaError_t e = cudaStreamSynchronize((cudaStream_t)stream);
  if (e != cudaSuccess) gfm::set_error("gfm_stream_sync: %s", cudaGetErrorString(e));
  return (int)e;
}

}  // extern "C"
