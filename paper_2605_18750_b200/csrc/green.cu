// green.cu -- SM partitions of one B200 (CUDA green contexts) for the
// single-GPU pipeline emulation: each emulated stage gets its own disjoint set
// of SMs, so an idle stage's SMs cannot be borrowed by the others (bench.py
// --emulate-pp).  Driver entry points are resolved at run time
// (cudaGetDriverEntryPoint), as gemm_sm100.cu does for the TMA encoder.
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <mutex>
#include <unordered_map>

#include "../../include/rrfp_b200.h"
#include "rrfp_common.h"

namespace {
template <typename F>
F entry(const char* name) {
  void* p = nullptr;
  cudaDriverEntryPointQueryResult q;
  if (cudaGetDriverEntryPoint(name, &p, cudaEnableDefault, &q) != cudaSuccess || q != cudaDriverEntryPointSuccess)
    return nullptr;
  return reinterpret_cast<F>(p);
}
// main stream of each partition -> its green context (released by rrfp_green_destroy)
std::mutex g_mu;
std::unordered_map<void*, CUgreenCtx> g_ctx_of;
}  // namespace

// n partitions of >= min_sms SMs each on `device`; per partition two streams
// (main, side) bound to its green context: streams[2*i], streams[2*i+1].
// *sms = SMs per partition.  Fails if the device cannot be split that way.
extern "C" int rrfp_green_streams(int device, int n, int min_sms, void** streams, int* sms) {
  using get_res_t = CUresult (*)(CUdevice, CUdevResource*, CUdevResourceType);
  using split_t = CUresult (*)(CUdevResource*, unsigned int*, const CUdevResource*, CUdevResource*, unsigned int,
                               unsigned int);
  using gen_t = CUresult (*)(CUdevResourceDesc*, CUdevResource*, unsigned int);
  using create_t = CUresult (*)(CUgreenCtx*, CUdevResourceDesc, CUdevice, unsigned int);
  using stream_t = CUresult (*)(CUstream*, CUgreenCtx, unsigned int, int);
  auto get_res = entry<get_res_t>("cuDeviceGetDevResource");
  auto split = entry<split_t>("cuDevSmResourceSplitByCount");
  auto gen = entry<gen_t>("cuDevResourceGenerateDesc");
  auto create = entry<create_t>("cuGreenCtxCreate");
  auto mkstream = entry<stream_t>("cuGreenCtxStreamCreate");
  if (!get_res || !split || !gen || !create || !mkstream)
    return rrfp_fail(RRFP_E_CUDA, "green-context driver entry points unavailable");
  if (n < 1 || n > 64 || !streams) return rrfp_fail(RRFP_E_INVALID, "rrfp_green_streams: bad arguments");
  RRFP_CUDA_TRY(cudaSetDevice(device));
  RRFP_CUDA_TRY(cudaFree(0));   // make sure the primary context exists
  CUdevice dev = device;
  CUdevResource all;
  if (get_res(dev, &all, CU_DEV_RESOURCE_TYPE_SM) != CUDA_SUCCESS)
    return rrfp_fail(RRFP_E_CUDA, "cuDeviceGetDevResource failed");
  CUdevResource groups[64], rest;
  // the split has a hardware granularity (SM pairs within GPCs): take the largest
  // group size <= min_sms that still yields n groups
  int want = min_sms;
  for (; want >= 2; want -= 2) {
    unsigned int probe = 0;
    if (split(nullptr, &probe, &all, nullptr, 0, want) == CUDA_SUCCESS && (int)probe >= n) break;
  }
  unsigned int ng = n;
  if (want < 2 || split(groups, &ng, &all, &rest, 0, want) != CUDA_SUCCESS || (int)ng < n)
    return rrfp_fail(RRFP_E_INVALID, "cannot split %u SMs into %d groups (asked >= %d SMs each)", all.sm.smCount,
                     n, min_sms);
  for (int i = 0; i < n; ++i) {
    CUdevResourceDesc desc;
    CUgreenCtx g;
    if (gen(&desc, &groups[i], 1) != CUDA_SUCCESS) return rrfp_fail(RRFP_E_CUDA, "cuDevResourceGenerateDesc");
    if (create(&g, desc, dev, CU_GREEN_CTX_DEFAULT_STREAM) != CUDA_SUCCESS)
      return rrfp_fail(RRFP_E_CUDA, "cuGreenCtxCreate");
    CUstream a, b;
    if (mkstream(&a, g, CU_STREAM_NON_BLOCKING, 0) != CUDA_SUCCESS ||
        mkstream(&b, g, CU_STREAM_NON_BLOCKING, 0) != CUDA_SUCCESS)
      return rrfp_fail(RRFP_E_CUDA, "cuGreenCtxStreamCreate");
    streams[2 * i] = a;
    streams[2 * i + 1] = b;
    std::lock_guard<std::mutex> lk(g_mu);
    g_ctx_of[(void*)a] = g;
  }
  if (sms) *sms = (int)groups[0].sm.smCount;
  return RRFP_OK;
}

// Release what rrfp_green_streams created: the 2n streams and the n green
// contexts (the caller has synchronised them).  Unknown streams are skipped.
extern "C" int rrfp_green_destroy(void* const* streams, int n) {
  using sdestroy_t = CUresult (*)(CUstream);
  using gdestroy_t = CUresult (*)(CUgreenCtx);
  auto sdestroy = entry<sdestroy_t>("cuStreamDestroy");
  auto gdestroy = entry<gdestroy_t>("cuGreenCtxDestroy");
  if (!sdestroy || !gdestroy) return rrfp_fail(RRFP_E_CUDA, "green-context driver entry points unavailable");
  if (n < 0 || (n > 0 && !streams)) return rrfp_fail(RRFP_E_INVALID, "rrfp_green_destroy: bad arguments");
  for (int i = 0; i < n; ++i) {
    CUgreenCtx g = nullptr;
    {
      std::lock_guard<std::mutex> lk(g_mu);
      auto it = g_ctx_of.find(streams[2 * i]);
      if (it == g_ctx_of.end()) continue;
      g = it->second;
      g_ctx_of.erase(it);
    }
    sdestroy((CUstream)streams[2 * i]);
    if (streams[2 * i + 1]) sdestroy((CUstream)streams[2 * i + 1]);
    if (gdestroy(g) != CUDA_SUCCESS) return rrfp_fail(RRFP_E_CUDA, "cuGreenCtxDestroy failed");
  }
  return RRFP_OK;
}
