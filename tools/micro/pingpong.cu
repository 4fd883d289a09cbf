// Cross-SM handoff latency through L2 (st.cg -> ld.cg polling), with optional
// background polling load from other CTAs.  nvcc -arch=sm_100a -O3 pingpong.cu
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

__device__ __forceinline__ long long ldcg(const long long* p) {
  long long v;
  asm volatile("ld.global.cg.s64 %0, [%1];" : "=l"(v) : "l"(p));
  return v;
}

template <int NQ>
__global__ void pingpong(long long* flag, int iters, long long* out, long long* bg, int bg_words, int bg_on,
                         volatile int* stop, int sleep_ns) {
  const int nsm2 = gridDim.x;  // unused
  (void)nsm2;
  if (blockIdx.x == 0 || blockIdx.x == 77) {
    if (threadIdx.x != 0) return;
    const int me = blockIdx.x == 0 ? 0 : 1;
    long long t0 = clock64();
    long long g0;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g0));
    for (int i = 0; i < iters; ++i) {
      if ((i & 1) == me) {
        __stcg(flag, (long long)(i + 1));
      } else {
        while (ldcg(flag) != (long long)(i + 1)) {
        }
      }
    }
    long long g1;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g1));
    if (me == 0) {
      out[0] = clock64() - t0;
      out[1] = g1 - g0;
      *stop = 1;
    }
    return;
  }
  if (!bg_on || blockIdx.x < 2 * 148) return;
  // background: every lane polls a random word of bg (never "ready")
  unsigned h = blockIdx.x * 1315423911u + threadIdx.x * 2654435761u;
  long long acc = 0;
  while (!*stop) {
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
      h = h * 1664525u + 1013904223u;
      acc += ldcg(bg + (h % bg_words));
    }
    if (sleep_ns) __nanosleep(sleep_ns);
  }
  if (acc == 42) out[2] = acc;
}

int main(int argc, char** argv) {
  int iters = 20000;
  long long *flag, *out, *bg;
  int* stop;
  const int bg_words = 1 << 20;  // 8 MB
  cudaMalloc(&flag, 8);
  cudaMalloc(&out, 64);
  cudaMalloc(&bg, 8LL * bg_words);
  cudaMalloc(&stop, 4);
  cudaMemset(bg, 0, 8LL * bg_words);
  int nsm = 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  for (int nq : {1, 20})
  for (int sl : {0, 64, 256, 1000})
  for (int bgb : {0, 1, 2}) {  // background CTAs (256 thr) per SM
    cudaMemset(flag, 0, 8);
    cudaMemset(stop, 0, 4);
    const int grid = 2 * nsm + (bgb ? bgb * nsm : 0);
    if (nq == 1) pingpong<1><<<grid, 256>>>(flag, iters, out, bg, bg_words, bgb > 0, stop, sl);
    else pingpong<20><<<grid, 256>>>(flag, iters, out, bg, bg_words, bgb > 0, stop, sl);
    cudaError_t e = cudaDeviceSynchronize();
    long long h[2];
    cudaMemcpy(h, out, 16, cudaMemcpyDeviceToHost);
    printf("loads/round %2d sleep %4d bg CTAs/SM %d: handoff %.1f ns  %s\n", nq, sl, bgb, (double)h[1] / iters,
           cudaGetErrorString(e));
  }
  return 0;
}
