// rrfp_common.h -- shared host-side helpers of the C-ABI library.
#pragma once
#include <stdarg.h>
#include <cuda_runtime.h>

// Sets the thread-local last-error string and returns `code`.
int rrfp_fail(int code, const char* fmt, ...);

#define RRFP_CUDA_TRY(expr)                                                              \
  do {                                                                                   \
    cudaError_t _e = (expr);                                                             \
    if (_e != cudaSuccess)                                                               \
      return rrfp_fail(RRFP_E_CUDA, "%s:%d %s: %s", __FILE__, __LINE__, #expr,           \
                       cudaGetErrorString(_e));                                          \
  } while (0)
