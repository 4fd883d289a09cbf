// Round-trip time of ld.global.cg polling rounds by many warps (1..N loads
// per lane per round) on an 8 MB array, optionally with concurrent st.cg.
#include <cstdio>
#include <cuda_runtime.h>

template <int NQ>
__global__ void poll(double* a, int words, int rounds, int sleep_ns, long long* out, int writers) {
  unsigned h = (blockIdx.x * 256 + threadIdx.x) * 2654435761u + 12345u;
  const bool wr = writers && (threadIdx.x & 31) == 0 && (blockIdx.x & 1);
  long long g0, g1;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g0));
  double acc = 0;
  for (int r = 0; r < rounds; ++r) {
    double v[NQ];
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
      h = h * 1664525u + 1013904223u;
      asm volatile("ld.global.cg.f64 %0, [%1];" : "=d"(v[q]) : "l"(a + (h % words)));
    }
#pragma unroll
    for (int q = 0; q < NQ; ++q) acc += v[q];
    if (wr) __stcg(a + (h % words), acc);
    if (sleep_ns) __nanosleep(sleep_ns);
    __syncwarp();
  }
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g1));
  if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = g1 - g0;
  if (acc == 1.2345) out[1] = 1;
}

int main() {
  const int words = 1 << 20;
  double* a;
  long long* out;
  cudaMalloc(&a, 8LL * words);
  cudaMalloc(&out, 16);
  cudaMemset(a, 0, 8LL * words);
  int nsm;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  const int rounds = 2000;
  for (int bps : {1, 4})
    for (int wr : {0, 1})
      for (int sl : {0, 64}) {
        long long h;
        poll<1><<<nsm * bps / 1, 256>>>(a, words, rounds, sl, out, wr);
        cudaDeviceSynchronize();
        cudaMemcpy(&h, out, 8, cudaMemcpyDeviceToHost);
        double t1 = (double)h / rounds;
        poll<4><<<nsm * bps, 256>>>(a, words, rounds, sl, out, wr);
        cudaDeviceSynchronize();
        cudaMemcpy(&h, out, 8, cudaMemcpyDeviceToHost);
        double t4 = (double)h / rounds;
        poll<20><<<nsm * bps, 256>>>(a, words, rounds, sl, out, wr);
        cudaDeviceSynchronize();
        cudaMemcpy(&h, out, 8, cudaMemcpyDeviceToHost);
        double t20 = (double)h / rounds;
        printf("CTAs/SM %d writers %d sleep %2d: round ns  1 load %.0f  4 loads %.0f  20 loads %.0f\n", bps, wr, sl, t1,
               t4, t20);
      }
  // single warp alone
  long long h;
  poll<1><<<1, 32>>>(a, words, rounds, 0, out, 0);
  cudaDeviceSynchronize();
  cudaMemcpy(&h, out, 8, cudaMemcpyDeviceToHost);
  printf("single warp, 1 load/lane: %.0f ns\n", (double)h / rounds);
  return 0;
}
