// Internal helpers shared by the host and CUDA translation units of libfpsa.
#pragma once
#include <string>

namespace fpsa {
// Record `msg` as this thread's last error and return `status`.
int fail(int status, const std::string& msg);
void clear_error();
}  // namespace fpsa
