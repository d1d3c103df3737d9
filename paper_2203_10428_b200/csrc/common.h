// Internal helpers shared by the library's translation units (not part of the ABI).
#pragma once
#include <atomic>
#include <cstdarg>
#include <cstdint>

#include "pgcn.h"

namespace pgcn {

// Records a thread-local message (returned by pgcn_last_error) and returns `code`.
int fail(int code, const char* fmt, ...);

inline int64_t round_up(int64_t x, int64_t a) { return (x + a - 1) / a * a; }
inline int64_t ld_of(int64_t f) { return round_up(f, 4); }

}  // namespace pgcn
