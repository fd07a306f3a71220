// Internal helpers shared by the host and CUDA translation units of libfpsa.
#pragma once
#include <string>

namespace fpsa {
// Record `msg` as this thread's last error and return `status`.
int fail(int status, const std::string& msg);
void clear_error();
// SM count of the current device (cached per device).
int device_sm_count();
// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) for `func` on the current device, once per
// (function, device): the attribute is per device, so a second GPU needs its own call.
int ensure_smem_attr(const void* func, int bytes, const char* what);
}  // namespace fpsa
