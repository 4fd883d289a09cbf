// Row-parallel kernel frameworks over the n x t row-major (storage order)
// vectors of the Vecchia path.
//
//  * rows_kernel   : no dependencies (products with B, B^T, dB, elementwise
//                    passes).  A group of G lanes owns one row; lane gl of a
//                    group owns columns c = gl + G*k (k < NC).
//  * trsv_kernel   : dependency-driven (sync-free) triangular solve.  Rows
//                    are visited in level order; a row spins on the
//                    epoch-tagged ready flags of the rows it reads, so there
//                    is no per-level launch or grid barrier.  The kernel is
//                    launched cooperatively (all CTAs co-resident) and rows
//                    are assigned statically in level order, which makes the
//                    spin deadlock-free.
//
// Both end with a DETERMINISTIC column reduction (NR quantities per column):
// fixed-order warp -> block -> grid (last-block) sums, no float atomics.
#pragma once

#include <cuda_runtime.h>

#include "common.cuh"

namespace vl {

constexpr int kRowsThreads = 256;

template <int NR>
struct Fin0 {
  VL_D void operator()(const double* /*sums*/, int /*t*/) const {}
};

// acc[r][k] for columns c = gl + G*k.  MAXMASK bit r set -> max-reduce (values >= 0).
template <int G, int NC, int NR, int MAXMASK>
VL_D void block_reduce_cols(double (&acc)[NR > 0 ? NR : 1][NC], int t, double* out, double* sh) {
  if (NR == 0) return;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
#pragma unroll
  for (int r = 0; r < NR; ++r)
#pragma unroll
    for (int k = 0; k < NC; ++k)
#pragma unroll
      for (int o = G; o < 32; o <<= 1) {
        double other = __shfl_xor_sync(0xffffffffu, acc[r][k], o);
        acc[r][k] = ((MAXMASK >> r) & 1) ? fmax(acc[r][k], other) : acc[r][k] + other;
      }
  if (lane < G) {
#pragma unroll
    for (int r = 0; r < NR; ++r)
#pragma unroll
      for (int k = 0; k < NC; ++k) sh[((warp * NR + r) * NC + k) * G + lane] = acc[r][k];
  }
  __syncthreads();
  for (int idx = threadIdx.x; idx < NR * t; idx += blockDim.x) {
    int r = idx / t, c = idx - r * t;
    int k = c / G, gl = c - k * G;
    double s = 0.0;
    for (int w = 0; w < nwarps; ++w) {
      double v = sh[((w * NR + r) * NC + k) * G + gl];
      s = ((MAXMASK >> r) & 1) ? fmax(s, v) : s + v;
    }
    out[idx] = s;
  }
}

// Grid-level finalisation by the last CTA to finish (fixed block order).
template <int NR, int MAXMASK, class Fin>
VL_D void grid_finalize(const double* partials, unsigned* counter, int t, const Fin& fin, double* sh) {
  if (NR == 0) return;
  __threadfence();
  __syncthreads();
  __shared__ unsigned s_ticket;
  if (threadIdx.x == 0) s_ticket = atomicAdd(counter, 1u);
  __syncthreads();
  if (s_ticket != gridDim.x - 1) return;
  __threadfence();
  const int nb = gridDim.x;
  for (int idx = threadIdx.x; idx < NR * t; idx += blockDim.x) {
    int r = idx / t;
    double s = 0.0;
    for (int b = 0; b < nb; ++b) {
      double v = __ldcg(partials + (size_t)b * NR * t + idx);
      s = ((MAXMASK >> r) & 1) ? fmax(s, v) : s + v;
    }
    sh[idx] = s;
  }
  __syncthreads();
  fin(sh, t);
  __syncthreads();
  if (threadIdx.x == 0) *counter = 0u;  // ready for the next launch using this slot
}

// shared memory needed by the reductions
template <int G, int NC, int NR>
constexpr size_t red_smem_bytes(int threads, int t) {
  size_t a = (size_t)(threads / 32) * (NR > 0 ? NR : 1) * NC * G * sizeof(double);
  size_t b = (size_t)(NR > 0 ? NR : 1) * t * sizeof(double);
  return a > b ? a : b;
}

// ---------------------------------------------------------------------------
// Body concept for rows_kernel:
//   template<int G,int NC,int NR> VL_D void operator()(int64_t s, bool valid, int gl, int t,
//                                                      double (&acc)[NR][NC]) const;
// Bodies must keep every lane of the warp participating when they use
// group shuffles (valid == false rows just skip memory traffic).
// ---------------------------------------------------------------------------
template <int G, int NC, int NR, int MAXMASK, class Body, class Fin>
__global__ void __launch_bounds__(kRowsThreads) rows_kernel(int64_t n, int t, Body body, Fin fin,
                                                            double* __restrict__ partials,
                                                            unsigned* __restrict__ counter,
                                                            const int* __restrict__ gate) {
  if (gate != nullptr && *((volatile const int*)gate) == 0) return;
  extern __shared__ double rsh[];
  constexpr int GPW = 32 / G;
  const int lane = threadIdx.x & 31;
  const int gl = lane % G;
  const int gi = lane / G;
  const int64_t gwarp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  double acc[NR > 0 ? NR : 1][NC];
#pragma unroll
  for (int r = 0; r < (NR > 0 ? NR : 1); ++r)
#pragma unroll
    for (int k = 0; k < NC; ++k) acc[r][k] = 0.0;
  for (int64_t s0 = gwarp * GPW; s0 < n; s0 += nwarps * GPW) {
    const int64_t s = s0 + gi;
    body.template run<G, NC, (NR > 0 ? NR : 1)>(s, s < n, gl, t, acc);
  }
  if (NR > 0) {
    block_reduce_cols<G, NC, NR, MAXMASK>(acc, t, partials + (size_t)blockIdx.x * NR * t, rsh);
    grid_finalize<NR, MAXMASK>(partials, counter, t, fin, rsh);
  }
}

// ---------------------------------------------------------------------------
// Dependency-driven triangular solve.
//   Solve:  x_s = rhs(s,c) - sum_{e in deps(s)} w_e * x_{dep(e)}
//   deps are read through the Deps functor (ELL rows of B for the forward
//   solve, children CSR of B^T for the backward solve).
// Body concept:
//   VL_D double rhs(int64_t s, int c, double& racc) const;      // right-hand side
//   VL_D void   out(int64_t s, int c, double x, double& racc) const;  // epilogue
// ---------------------------------------------------------------------------
struct DepsEll {
  const int32_t* nbr;
  const int32_t* cnt;
  const double* val;
  int m;
  VL_D int begin(int64_t s) const { return 0; }
  VL_D int end(int64_t s) const { return cnt[s]; }
  VL_D int32_t col(int64_t s, int e) const { return nbr[s * m + e]; }
  VL_D double w(int64_t s, int e) const { return val[s * m + e]; }
};
struct DepsCsr {
  const int32_t* ptr;
  const int32_t* idx;
  const double* val;
  VL_D int begin(int64_t s) const { return ptr[s]; }
  VL_D int end(int64_t s) const { return ptr[s + 1]; }
  VL_D int32_t col(int64_t s, int e) const { return idx[e]; }
  VL_D double w(int64_t s, int e) const { return val[e]; }
};

template <int G, int NC, int NR, class Deps, class Body, class Fin>
__global__ void __launch_bounds__(kRowsThreads) trsv_kernel(int64_t n, int t, const int32_t* __restrict__ order,
                                                            Deps deps, double* __restrict__ x, int* __restrict__ flags,
                                                            int epoch, Body body, Fin fin,
                                                            double* __restrict__ partials,
                                                            unsigned* __restrict__ counter,
                                                            const int* __restrict__ gate) {
  if (gate != nullptr && *((volatile const int*)gate) == 0) return;
  extern __shared__ double rsh[];
  constexpr int GPW = 32 / G;
  const int lane = threadIdx.x & 31;
  const int gl = lane % G;
  const int gi = lane / G;
  const unsigned gmask = (G == 32) ? 0xffffffffu : (((1u << G) - 1u) << (gi * G));
  const int64_t gid = (((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5) * GPW + gi;
  const int64_t ngroups = (((int64_t)gridDim.x * blockDim.x) >> 5) * GPW;
  double acc[NR > 0 ? NR : 1][NC];
#pragma unroll
  for (int r = 0; r < (NR > 0 ? NR : 1); ++r)
#pragma unroll
    for (int k = 0; k < NC; ++k) acc[r][k] = 0.0;

  for (int64_t p = gid; p < n; p += ngroups) {
    const int64_t s = order[p];
    double xs[NC];
#pragma unroll
    for (int k = 0; k < NC; ++k) {
      int c = gl + G * k;
      xs[k] = (c < t) ? body.rhs(s, c, acc[0][k]) : 0.0;
    }
    const int e0 = deps.begin(s), e1 = deps.end(s);
    for (int e = e0; e < e1; ++e) {
      const int32_t j = deps.col(s, e);
      const double w = deps.w(s, e);
      while (ld_acquire(flags + j) != epoch) {
      }
      const double* xj = x + (int64_t)j * t;
#pragma unroll
      for (int k = 0; k < NC; ++k) {
        int c = gl + G * k;
        if (c < t) xs[k] -= w * ld_cg(xj + c);
      }
    }
#pragma unroll
    for (int k = 0; k < NC; ++k) {
      int c = gl + G * k;
      if (c < t) {
        x[s * t + c] = xs[k];
        body.out(s, c, xs[k], acc[0][k]);
      }
    }
    __threadfence();
    __syncwarp(gmask);
    if (gl == 0) st_release(flags + s, epoch);
  }
  if (NR > 0) {
    block_reduce_cols<G, NC, NR, 0>(acc, t, partials + (size_t)blockIdx.x * NR * t, rsh);
    grid_finalize<NR, 0>(partials, counter, t, fin, rsh);
  }
}

}  // namespace vl
