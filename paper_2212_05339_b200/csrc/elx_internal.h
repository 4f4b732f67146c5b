// Internal helpers shared by the host (.cpp) and device (.cu) translation units.
#pragma once

#include <atomic>
#include <cstdarg>
#include <cstdint>
#include <cstdio>
#include <string>

#include "elixir_b200.h"

namespace elx {

// Thread-local error message behind elx_last_error().
void set_error(const char* fmt, ...);
void clear_error();

// Global launch counter behind elx_launch_count().
extern std::atomic<int64_t> g_launches;
inline void count_launch(int64_t k = 1) { g_launches.fetch_add(k, std::memory_order_relaxed); }

inline int fail(int code, const char* fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  set_error("%s", buf);
  return code;
}

inline int dtype_size(int32_t dt) {
  switch (dt) {
    case ELX_F32: return 4;
    case ELX_BF16: return 2;
    case ELX_F16: return 2;
    default: return 0;
  }
}

}  // namespace elx
