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

// Launch with programmatic dependent launch (PDL) enabled when rrfp_pdl() is
// true: the kernel may start while its predecessor drains; every kernel of
// this library calls griddepcontrol.wait before touching global memory.
bool rrfp_pdl();

template <typename... KArgs, typename... Args>
cudaError_t rrfp_launch(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                        Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = rrfp_pdl() ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...);
}
