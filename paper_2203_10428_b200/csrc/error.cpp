#include <cstdio>

#include "common.h"

namespace {
thread_local char g_msg[1024] = "";
}

namespace pgcn {
int fail(int code, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  std::vsnprintf(g_msg, sizeof(g_msg), fmt, ap);
  va_end(ap);
  return code;
}
}  // namespace pgcn

extern "C" const char* pgcn_last_error(void) { return g_msg; }
extern "C" int pgcn_version(void) { return 100; }
