// ABI plumbing: version, thread-local error text, launch counter.
#include "elx_internal.h"

namespace elx {

static thread_local std::string t_error;
std::atomic<int64_t> g_launches{0};

void set_error(const char* fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  t_error = buf;
}

void clear_error() { t_error.clear(); }

}  // namespace elx

extern "C" {

int32_t elx_abi_version(void) { return ELX_ABI_VERSION; }

const char* elx_last_error(void) { return elx::t_error.c_str(); }

int64_t elx_launch_count(void) { return elx::g_launches.load(std::memory_order_relaxed); }

int64_t elx_sizeof(int32_t which) {
  switch (which) {
    case 0: return (int64_t)sizeof(elx_event);
    case 1: return (int64_t)sizeof(elx_sim_counters);
    case 2: return (int64_t)sizeof(elx_member);
    case 3: return (int64_t)sizeof(elx_adam_seg);
    case 4: return (int64_t)sizeof(elx_adam_hp);
    case 5: return (int64_t)sizeof(elx_cpu_seg);
    case 6: return (int64_t)sizeof(elx_release_seg);
    default: return -1;
  }
}

}  // extern "C"
