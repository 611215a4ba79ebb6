// Error reporting and version of the C ABI (include/fpvs.h).
#include <stdlib.h>

#include "common.cuh"

namespace fpvs {

static thread_local char g_err[512] = "";

int set_error(int code, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
  return code;
}

bool pdl_enabled() {
  static const bool on = [] {
    const char* e = getenv("FPVS_PDL");
    return !(e && e[0] == '0');
  }();
  return on;
}

}  // namespace fpvs

extern "C" const char* fpvs_last_error(void) { return fpvs::g_err; }
extern "C" int fpvs_abi_version(void) { return 4; }  // 2: f64 interleave, double tau, exchange, k^3 maps; 3: row-bits head; 4: brick conv
