// Error plumbing and small ABI utilities (no global mutable state besides
// thread-local error text / launch counters and a lazily cached SM count).
#include <atomic>
#include <mutex>
#include "ctp_common.cuh"

namespace ctp {

static thread_local char g_err[512] = "";
static thread_local int64_t g_launches = 0;

void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

int64_t& launch_counter() { return g_launches; }

int num_sms() {
  // per-device lazy query under a mutex (SURVEY s8(b) threading rules)
  static std::mutex mu;
  static int cached[64] = {0};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return kNumSMs;
  std::lock_guard<std::mutex> lk(mu);
  if (cached[dev] == 0) {
    int n = 0;
    if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n <= 0) n = kNumSMs;
    cached[dev] = n;
  }
  return cached[dev];
}

int check_level_desc(const ctp_level_out& lo, int64_t lnx, int64_t lny, int64_t lnz_global, int level) {
  if (lo.out == nullptr) return CTP_OK;
  if (lo.layout == CTP_LAYOUT_XYZ) return CTP_OK;
  CTP_REQUIRE(lo.layout == CTP_LAYOUT_ATLAS, CTP_E_UNSUPPORTED, "level %d: unknown layout %d", level, lo.layout);
  CTP_REQUIRE(lo.s >= 1 && lo.grid >= 1, CTP_E_INVALID, "level %d: bad scheme s=%d grid=%d", level, lo.s, lo.grid);
  // slicemap.py:52-61
  CTP_REQUIRE((int64_t)lo.grid * lo.s == lo.atlas_dim, CTP_E_UNSUPPORTED,
              "level %d: grid %d x slice %d != atlas %d", level, lo.grid, lo.s, lo.atlas_dim);
  int64_t per = (int64_t)lo.grid * lo.grid;
  CTP_REQUIRE(lo.map_count == (lo.s + per - 1) / per, CTP_E_UNSUPPORTED,
              "level %d: %d maps cannot hold %d slices at %lld/map", level, lo.map_count, lo.s, (long long)per);
  // pipeline.py:226-237 pads, never crops
  CTP_REQUIRE(lnx <= lo.s && lny <= lo.s && lnz_global <= lo.s, CTP_E_INVALID,
              "level %d: dims (%lld,%lld,%lld) exceed scheme edge %d", level, (long long)lnx, (long long)lny,
              (long long)lnz_global, lo.s);
  return CTP_OK;
}

}  // namespace ctp

extern "C" {

const char* ctp_last_error(void) { return ctp::g_err; }

int ctp_abi_version(void) { return CTP_ABI_VERSION; }

int64_t ctp_launch_count(int32_t reset) {
  int64_t n = ctp::g_launches;
  if (reset) ctp::g_launches = 0;
  return n;
}

}  // extern "C"
