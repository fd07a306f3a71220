// Host <-> device staging for the streamed host path (FpsaPlan.run_host):
// a strided 2D copy moves a contiguous run of heads of every token between a
// pinned host [tokens, heads, d] array and a device [tokens, chunk, d] buffer,
// so a head chunk's transfer overlaps the previous chunk's kernels.
#include <cuda_runtime.h>

#include <cstdint>
#include <string>

#include "../../include/fpsa.h"
#include "fpsa_internal.h"

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
