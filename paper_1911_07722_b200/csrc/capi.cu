// C-ABI glue: error reporting, ABI version, host RNG entry points.
#include <stdarg.h>
#include <stdio.h>

#include "common.cuh"
#include "rng.cuh"

namespace syscd {
static thread_local char g_err[512] = "";
void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}
}  // namespace syscd

using namespace syscd;

extern "C" int syscd_abi_version(void) { return SYSCD_ABI_VERSION; }

extern "C" const char* syscd_last_error(void) { return g_err; }

extern "C" int syscd_rng_permutation(uint64_t seed, const uint64_t* key, int32_t key_len,
                                     int64_t n, int64_t* out) {
  if (n < 0 || key_len < 0 || key_len > 8 || (key_len > 0 && !key) || (n > 0 && !out)) {
    set_error("syscd_rng_permutation: invalid arguments");
    return SYSCD_EINVAL;
  }
  Pcg64 g;
  pcg_seed_keyed(&g, seed, key, key_len);
  for (int64_t i = 0; i < n; ++i) out[i] = i;
  pcg_shuffle(&g, out, n);
  return SYSCD_OK;
}

extern "C" int syscd_rng_integers(uint64_t seed, const uint64_t* key, int32_t key_len, int64_t lo,
                                  int64_t hi, int64_t count, int64_t* out) {
  if (hi <= lo || count < 0 || key_len < 0 || key_len > 8 || (key_len > 0 && !key) ||
      (count > 0 && !out)) {
    set_error("syscd_rng_integers: invalid arguments");
    return SYSCD_EINVAL;
  }
  Pcg64 g;
  pcg_seed_keyed(&g, seed, key, key_len);
  for (int64_t i = 0; i < count; ++i) out[i] = pcg_integers(&g, lo, hi);
  return SYSCD_OK;
}
