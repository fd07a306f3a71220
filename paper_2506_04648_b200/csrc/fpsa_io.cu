// Host <-> device staging for the streamed host path (HostStreamer) and the
// per-device launch state shared by the kernels' host code.
//
// fpsa_copy2d: a strided 2D copy moves a contiguous run of heads of every
// token between a pinned host [tokens, heads, d] array and a device
// [tokens, chunk, d] buffer, so a head chunk's transfer overlaps the previous
// chunk's kernels.
//
// device_sm_count / ensure_smem_attr: SM count and the dynamic shared-memory
// opt-in are properties of a device, not of the process, so they are cached
// per (device) and (kernel, device): a plan on cuda:1 launched after one on
// cuda:0 gets its own attribute call.
#include <cuda_runtime.h>

#include <cstdint>
#include <mutex>
#include <set>
#include <string>
#include <utility>

#include "../../include/fpsa.h"
#include "fpsa_internal.h"

namespace fpsa {
namespace {
constexpr int kMaxDevices = 64;
std::mutex g_mu;
int g_sms[kMaxDevices] = {0};
std::set<std::pair<const void*, int>> g_attr_done;

int current_device() {
  int dev = 0;
  cudaGetDevice(&dev);
  return dev;
}
}  // namespace

int device_sm_count() {
  const int dev = current_device();
  if (dev < 0 || dev >= kMaxDevices) return 148;
  std::lock_guard<std::mutex> lock(g_mu);
  if (!g_sms[dev]) {
    int n = 0;
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    g_sms[dev] = n > 0 ? n : 148;
  }
  return g_sms[dev];
}

int ensure_smem_attr(const void* func, int bytes, const char* what) {
  const int dev = current_device();
  std::lock_guard<std::mutex> lock(g_mu);
  if (g_attr_done.count({func, dev})) return FPSA_OK;
  if (cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes) != cudaSuccess)
    return fail(FPSA_ECUDA, std::string(what) + " cudaFuncSetAttribute: " + cudaGetErrorString(cudaGetLastError()));
  g_attr_done.insert({func, dev});
  return FPSA_OK;
}
}  // namespace fpsa

extern "C" int fpsa_copy2d(void* dst, int64_t dst_pitch, const void* src, int64_t src_pitch, int64_t width,
                           int64_t rows, void* stream) {
  fpsa::clear_error();
  if (!dst || !src) return fpsa::fail(FPSA_EINVAL, "null buffer");
  if (width < 0 || rows < 0 || dst_pitch < width || src_pitch < width)
    return fpsa::fail(FPSA_EINVAL, "pitches must be >= width >= 0");
  if (width == 0 || rows == 0) return FPSA_OK;
  const cudaError_t e = cudaMemcpy2DAsync(dst, (size_t)dst_pitch, src, (size_t)src_pitch, (size_t)width, (size_t)rows,
                                          cudaMemcpyDefault, static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return fpsa::fail(FPSA_ECUDA, std::string("fpsa_copy2d: ") + cudaGetErrorString(e));
  return FPSA_OK;
}
