#include "common.h"

#include <atomic>

namespace sg {

static thread_local std::string g_last_error;
static std::atomic<int64_t> g_launches{0};

void count_launch(int n) { g_launches.fetch_add(n, std::memory_order_relaxed); }

void set_error(const char* fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_last_error = buf;
}

}  // namespace sg

extern "C" const char* sg_last_error(void) { return sg::g_last_error.c_str(); }

extern "C" int sg_version(void) { return 1; }

extern "C" int64_t sg_launch_count(void) { return sg::g_launches.load(); }
