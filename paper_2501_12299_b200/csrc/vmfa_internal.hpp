// vmfa_internal.hpp — shared host-side plumbing of libvmfa_b200.so:
// thread-local error text behind vmfa_last_error(), status helpers.
#pragma once
#include <cstdarg>
#include <cstdio>
#include <string>

#include "vmfa_b200.h"

namespace vmfa_b200 {

void set_error_text(const std::string& s);
const std::string& error_text();

inline int fail(int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  std::vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  set_error_text(buf);
  return code;
}

}  // namespace vmfa_b200
