// Shared device/host helpers for the vlgpx sm_100a library.
#pragma once

#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <string>

#define VL_HD __host__ __device__ __forceinline__
#define VL_D __device__ __forceinline__

namespace vl {

constexpr int kWarp = 32;

// ---- status codes (mirrors include/vlgpx.h) --------------------------------
enum Status : int {
  kOk = 0,
  kEConfig = 2,
  kEData = 3,
  kECapability = 5,
  kECapacity = 6,
  kEFactorization = 40,
  kEBreakdown = 41,
  kEConvergence = 42,
  kECuda = 50,
  kEInternal = 51,
};

struct Error {
  int code;
  std::string msg;
};

// Throwing helpers used inside the library; the C-ABI layer catches them.
[[noreturn]] void fail(int code, const std::string& msg);
void cuda_check(cudaError_t e, const char* what, const char* file, int line);

#define VL_CUDA(x) ::vl::cuda_check((x), #x, __FILE__, __LINE__)
#define VL_LAUNCH_CHECK() ::vl::cuda_check(cudaGetLastError(), "kernel launch", __FILE__, __LINE__)

// ---- memory-ordering helpers for the dependency-driven solves --------------
VL_D int ld_acquire(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
VL_D void st_release(int* p, int v) {
  asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
// L2-coherent load (bypasses L1 so a row published by another SM is never
// served from a stale L1 line).
VL_D double ld_cg(const double* p) { return __ldcg(p); }

// ---- warp / group reductions -----------------------------------------------
template <int G>
VL_D double group_sum(double v) {
#pragma unroll
  for (int o = G / 2; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o, G);
  return v;
}
template <int G>
VL_D double group_max(double v) {
#pragma unroll
  for (int o = G / 2; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o, G));
  return v;
}
VL_D double warp_sum(double v) { return group_sum<32>(v); }

}  // namespace vl
