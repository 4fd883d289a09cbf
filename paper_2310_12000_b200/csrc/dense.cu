// Hand-written fp64 dense kernels of the low-rank paths (see dense.h).
//
// dgemm: 64 x 64 output tile per 256-thread CTA, 16-deep k slices staged
// through shared memory (k-major, so the inner product reads are
// conflict-free and the B values broadcast), the next slice prefetched into
// registers while the current one is consumed, 4 x 4 outputs per thread
// (rows tx + 16 r, columns ty + 16 c).  Long contractions (the n-dimension of
// L^T W L, L^T x) are split over blockIdx.z into fixed k ranges whose
// partials are summed in split order by a second kernel, so results are
// deterministic.  fp64 FMA: B200 has the same fp64 rate on its CUDA cores as
// on the tensor cores, and these products are HBM-bound on L (n x k) except
// the k x k x n SYRK.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>

#include "common.cuh"
#include "dense.h"

namespace vl {

namespace {

constexpr int GBM = 64, GBN = 64, GBK = 16, GTH = 256;

template <bool TA, bool TB, bool KW>
__global__ void __launch_bounds__(GTH) dgemm_kernel(int m, int n, int k, int kchunk, double alpha,
                                                    const double* __restrict__ A, int lda,
                                                    const double* __restrict__ B, int ldb, double beta,
                                                    double* __restrict__ Cm, int ldc, const double* __restrict__ kw,
                                                    int lower, double* __restrict__ part) {
  __shared__ double As[GBK][GBM + 1];
  __shared__ double Bs[GBK][GBN + 1];
  const int tid = threadIdx.x;
  const int bm = blockIdx.x * GBM, bn = blockIdx.y * GBN;
  if (lower && bn > bm + GBM - 1) return;  // tile strictly above the diagonal
  const int k0 = blockIdx.z * kchunk;
  const int k1 = min(k, k0 + kchunk);
  const int tx = tid & 15, ty = tid >> 4;
  double acc[4][4];
#pragma unroll
  for (int r = 0; r < 4; ++r)
#pragma unroll
    for (int c = 0; c < 4; ++c) acc[r][c] = 0.0;
  double ra[4], rb[4];
  // element q of this thread's share of a 64 x 16 (A) / 16 x 64 (B) slice
  auto a_ij = [&](int q, int& i, int& kk) {
    const int e = tid + GTH * q;
    if (TA) { kk = e & 15; i = e >> 4; } else { i = e & 63; kk = e >> 6; }
  };
  auto b_ij = [&](int q, int& kk, int& j) {
    const int e = tid + GTH * q;
    if (TB) { j = e & 63; kk = e >> 6; } else { kk = e & 15; j = e >> 4; }
  };
  auto load = [&](int kt) {
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      int i, kk;
      a_ij(q, i, kk);
      const int gi = bm + i, gk = kt + kk;
      ra[q] = (gi < m && gk < k1) ? (TA ? A[gk + (int64_t)gi * lda] : A[gi + (int64_t)gk * lda]) : 0.0;
      int j, kb;
      b_ij(q, kb, j);
      const int gj = bn + j, gkb = kt + kb;
      double v = 0.0;
      if (gj < n && gkb < k1) {
        v = TB ? B[gj + (int64_t)gkb * ldb] : B[gkb + (int64_t)gj * ldb];
        if (KW) v *= kw[gkb];
      }
      rb[q] = v;
    }
  };
  auto stash = [&]() {
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      int i, kk;
      a_ij(q, i, kk);
      As[kk][i] = ra[q];
      int j, kb;
      b_ij(q, kb, j);
      Bs[kb][j] = rb[q];
    }
  };
  if (k0 < k1) load(k0);
  for (int kt = k0; kt < k1; kt += GBK) {
    __syncthreads();
    stash();
    __syncthreads();
    if (kt + GBK < k1) load(kt + GBK);
#pragma unroll
    for (int kk = 0; kk < GBK; ++kk) {
      double a[4], b[4];
#pragma unroll
      for (int r = 0; r < 4; ++r) a[r] = As[kk][tx + 16 * r];
#pragma unroll
      for (int c = 0; c < 4; ++c) b[c] = Bs[kk][ty + 16 * c];
#pragma unroll
      for (int r = 0; r < 4; ++r)
#pragma unroll
        for (int c = 0; c < 4; ++c) acc[r][c] = fma(a[r], b[c], acc[r][c]);
    }
  }
#pragma unroll
  for (int r = 0; r < 4; ++r)
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const int i = bm + tx + 16 * r, j = bn + ty + 16 * c;
      if (i >= m || j >= n || (lower && j > i)) continue;
      if (part != nullptr) {
        part[(size_t)blockIdx.z * m * n + (size_t)j * m + i] = acc[r][c];
      } else {
        double v = alpha * acc[r][c];
        if (beta != 0.0) v += beta * Cm[i + (int64_t)j * ldc];
        Cm[i + (int64_t)j * ldc] = v;
      }
    }
}

// fp64 tensor-core variant (DMMA, mma.sync.m8n8k4.f64): 128 x 128 CTA tile,
// 8 warps as 4 (M) x 2 (N), each warp 32 x 64 = 4 x 8 m8n8 tiles; operands
// staged k-contiguous per output index (As[m][k], Bs[n][k], padded rows) so
// a fragment load -- element (lane / 4, lane % 4) -- is at most 2-way
// bank-conflicted; 16-deep k slices, next slice prefetched into registers.
constexpr int DBM = 128, DBN = 128, DBK = 16, DKP = DBK + 4;

VL_D void dmma884(double (&d)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
               : "+d"(d[0]), "+d"(d[1])
               : "d"(a), "d"(b));
}

template <bool TA, bool TB, bool KW>
__global__ void __launch_bounds__(GTH, 1) dgemm_dmma_kernel(int m, int n, int k, int kchunk, double alpha,
                                                           const double* __restrict__ A, int lda,
                                                           const double* __restrict__ B, int ldb, double beta,
                                                           double* __restrict__ Cm, int ldc,
                                                           const double* __restrict__ kw, int lower,
                                                           double* __restrict__ part) {
  __shared__ double As[DBM][DKP];
  __shared__ double Bs[DBN][DKP];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int bm = blockIdx.x * DBM, bn = blockIdx.y * DBN;
  if (lower && bn > bm + DBM - 1) return;
  const int k0 = blockIdx.z * kchunk;
  const int k1 = min(k, k0 + kchunk);
  const int wm = (warp >> 1) * 32, wn = (warp & 1) * 64;
  double acc[4][8][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
  double ra[8], rb[8];
  auto a_mk = [&](int q, int& mm, int& kk) {
    const int e = tid + GTH * q;
    if (TA) { kk = e & 15; mm = e >> 4; } else { mm = e & 127; kk = e >> 7; }
  };
  auto b_nk = [&](int q, int& nn, int& kk) {
    const int e = tid + GTH * q;
    if (TB) { nn = e & 127; kk = e >> 7; } else { kk = e & 15; nn = e >> 4; }
  };
  auto load = [&](int kt) {
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      int mm, kk;
      a_mk(q, mm, kk);
      const int gi = bm + mm, gk = kt + kk;
      ra[q] = (gi < m && gk < k1) ? (TA ? A[gk + (int64_t)gi * lda] : A[gi + (int64_t)gk * lda]) : 0.0;
      int nn, kb;
      b_nk(q, nn, kb);
      const int gj = bn + nn, gkb = kt + kb;
      double v = 0.0;
      if (gj < n && gkb < k1) {
        v = TB ? B[gj + (int64_t)gkb * ldb] : B[gkb + (int64_t)gj * ldb];
        if (KW) v *= kw[gkb];
      }
      rb[q] = v;
    }
  };
  auto stash = [&]() {
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      int mm, kk;
      a_mk(q, mm, kk);
      As[mm][kk] = ra[q];
      int nn, kb;
      b_nk(q, nn, kb);
      Bs[nn][kb] = rb[q];
    }
  };
  const int fr = lane >> 2, fc = lane & 3;
  if (k0 < k1) load(k0);
  for (int kt = k0; kt < k1; kt += DBK) {
    __syncthreads();
    stash();
    __syncthreads();
    if (kt + DBK < k1) load(kt + DBK);
#pragma unroll
    for (int kk = 0; kk < DBK; kk += 4) {
      double a[4], b[8];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = As[wm + i * 8 + fr][kk + fc];
#pragma unroll
      for (int j = 0; j < 8; ++j) b[j] = Bs[wn + j * 8 + fr][kk + fc];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) dmma884(acc[i][j], a[i], b[j]);
    }
  }
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 8; ++j)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int r = bm + wm + i * 8 + fr, c = bn + wn + j * 8 + fc * 2 + h;
        if (r >= m || c >= n || (lower && c > r)) continue;
        if (part != nullptr) {
          part[(size_t)blockIdx.z * m * n + (size_t)c * m + r] = acc[i][j][h];
        } else {
          double v = alpha * acc[i][j][h];
          if (beta != 0.0) v += beta * Cm[r + (int64_t)c * ldc];
          Cm[r + (int64_t)c * ldc] = v;
        }
      }
}

// Thin products (an output side <= 8: the t = 1 Woodbury apply of every Newton
// CG iteration), memory-bound on the long operand, read once and coalesced:
//  * thin_nt: C (m x nt) = A (m x K, column-major) B^T, B (nt x K): thread per
//    output row over a K range (split over blockIdx.y), B entries broadcast;
//  * thin_tn: C (mt x n) = A^T B, A (K x mt), B (K x n, column-major): warp per
//    output column j, lanes over K (column j of B contiguous), A staged in smem.
constexpr int kThinMax = 8;

template <int NT, bool KW>
__global__ void __launch_bounds__(256) thin_nt_kernel(int m, int K, int kchunk, const double* __restrict__ A, int lda,
                                                     const double* __restrict__ B, int ldb,
                                                     const double* __restrict__ kw, double* __restrict__ part) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const int k0 = blockIdx.y * kchunk, k1 = min(K, k0 + kchunk);
  double acc[NT];
#pragma unroll
  for (int c = 0; c < NT; ++c) acc[c] = 0.0;
  if (i < m) {
#pragma unroll 8
    for (int kk = k0; kk < k1; ++kk) {
      const double a = A[i + (int64_t)kk * lda] * (KW ? kw[kk] : 1.0);
#pragma unroll
      for (int c = 0; c < NT; ++c) acc[c] = fma(a, __ldg(B + c + (int64_t)kk * ldb), acc[c]);
    }
#pragma unroll
    for (int c = 0; c < NT; ++c) part[(size_t)blockIdx.y * m * NT + (size_t)c * m + i] = acc[c];
  }
}

template <int MT>
__global__ void __launch_bounds__(256) thin_tn_kernel(int n, int K, const double* __restrict__ A, int lda,
                                                     const double* __restrict__ B, int ldb, double alpha, double beta,
                                                     double* __restrict__ Cm, int ldc) {
  extern __shared__ double As[];  // K x MT
  for (int e = threadIdx.x; e < K * MT; e += blockDim.x) {
    const int kk = e % K, c = e / K;
    As[e] = A[kk + (int64_t)c * lda];
  }
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int64_t nw = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t j = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); j < n; j += nw) {
    double acc[MT];
#pragma unroll
    for (int c = 0; c < MT; ++c) acc[c] = 0.0;
    const double* bj = B + j * ldb;
#pragma unroll 8
    for (int kk = lane; kk < K; kk += 32) {
      const double b = bj[kk];
#pragma unroll
      for (int c = 0; c < MT; ++c) acc[c] = fma(As[kk + c * K], b, acc[c]);
    }
#pragma unroll
    for (int c = 0; c < MT; ++c) {
      double v = acc[c];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
      if (lane == c) {
        double r = alpha * v;
        if (beta != 0.0) r += beta * Cm[c + j * ldc];
        Cm[c + j * ldc] = r;
      }
    }
  }
}

__global__ void splitk_reduce_kernel(int m, int n, int splits, double alpha, const double* __restrict__ part,
                                     double beta, double* __restrict__ Cm, int ldc, int lower, int64_t zstride) {
  const int64_t total = (int64_t)m * n;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int i = (int)(e % m), j = (int)(e / m);
    if (lower && j > i) continue;
    double s = 0.0;
    for (int z = 0; z < splits; ++z) s += part[(size_t)z * zstride + e];
    double v = alpha * s;
    if (beta != 0.0) v += beta * Cm[i + (int64_t)j * ldc];
    Cm[i + (int64_t)j * ldc] = v;
  }
}

template <bool TA, bool TB>
void launch_gemm(Ctx& C, const Gemm& g, dim3 grid, int kchunk, double* part, bool tc) {
  if (tc) {
    if (g.kw)
      dgemm_dmma_kernel<TA, TB, true><<<grid, GTH, 0, C.stream>>>(g.m, g.n, g.k, kchunk, g.alpha, g.A, g.lda, g.B,
                                                                  g.ldb, g.beta, g.C, g.ldc, g.kw, g.lower ? 1 : 0,
                                                                  part);
    else
      dgemm_dmma_kernel<TA, TB, false><<<grid, GTH, 0, C.stream>>>(g.m, g.n, g.k, kchunk, g.alpha, g.A, g.lda, g.B,
                                                                   g.ldb, g.beta, g.C, g.ldc, nullptr,
                                                                   g.lower ? 1 : 0, part);
    VL_LAUNCH_CHECK();
    return;
  }
  if (g.kw)
    dgemm_kernel<TA, TB, true><<<grid, GTH, 0, C.stream>>>(g.m, g.n, g.k, kchunk, g.alpha, g.A, g.lda, g.B, g.ldb,
                                                           g.beta, g.C, g.ldc, g.kw, g.lower ? 1 : 0, part);
  else
    dgemm_kernel<TA, TB, false><<<grid, GTH, 0, C.stream>>>(g.m, g.n, g.k, kchunk, g.alpha, g.A, g.lda, g.B, g.ldb,
                                                            g.beta, g.C, g.ldc, nullptr, g.lower ? 1 : 0, part);
  VL_LAUNCH_CHECK();
}

// Diagonal 64 x 64 blocks of L^-1: thread j forward-substitutes column j of
// the block in shared memory (no synchronisation inside the solve).
__global__ void trtri_diag_kernel(int k, const double* __restrict__ L, int ldl, double* __restrict__ Li, int ldi) {
  __shared__ double X[64][65];
  const int b0 = blockIdx.x * 64;
  const int bs = min(64, k - b0);
  const int j = threadIdx.x;
  const double* Lb = L + b0 + (int64_t)b0 * ldl;  // Lb(r, c) = Lb[r + c * ldl] (L1-resident)
  if (j < bs) {
    for (int i = 0; i < bs; ++i) {
      double s = (i == j) ? 1.0 : 0.0;
      for (int l = j; l < i; ++l) s -= __ldg(Lb + i + (int64_t)l * ldl) * X[l][j];
      X[i][j] = (i >= j) ? s / __ldg(Lb + i + (int64_t)i * ldl) : 0.0;
    }
  }
  __syncthreads();
  for (int e = j; e < 64 * 64; e += blockDim.x) {
    const int r = e & 63, c = e >> 6;
    if (r < bs && c < bs) Li[(b0 + r) + (int64_t)(b0 + c) * ldi] = X[r][c];
  }
}

__global__ void zero_upper_kernel(int k, double* __restrict__ Li, int ldi) {
  const int64_t total = (int64_t)k * k;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int i = (int)(e % k), j = (int)(e / k);
    if (j > i) Li[i + (int64_t)j * ldi] = 0.0;
  }
}

}  // namespace

template <int NT>
static void thin_nt(Ctx& C, const Gemm& g) {
  const int splits = (int)std::max<int64_t>(1, std::min<int64_t>(256, g.k / 512));
  const int kchunk = (g.k + splits - 1) / splits;
  DevBuf ws;
  ws.alloc(sizeof(double) * (size_t)splits * g.m * NT);
  const dim3 grid((g.m + 255) / 256, splits);
  if (g.kw)
    thin_nt_kernel<NT, true><<<grid, 256, 0, C.stream>>>(g.m, g.k, kchunk, g.A, g.lda, g.B, g.ldb, g.kw,
                                                         ws.as<double>());
  else
    thin_nt_kernel<NT, false><<<grid, 256, 0, C.stream>>>(g.m, g.k, kchunk, g.A, g.lda, g.B, g.ldb, nullptr,
                                                          ws.as<double>());
  VL_LAUNCH_CHECK();
  const int64_t total = (int64_t)g.m * NT;
  const int blocks = (int)std::max<int64_t>(1, std::min<int64_t>((total + 255) / 256, 8LL * C.num_sms));
  // partials are (m x NT) per split; the first g.n columns are the output
  splitk_reduce_kernel<<<blocks, 256, 0, C.stream>>>(g.m, g.n, splits, g.alpha, ws.as<double>(), g.beta, g.C, g.ldc,
                                                     0, g.m * NT);
  VL_LAUNCH_CHECK();
}

template <int MT>
static void thin_tn(Ctx& C, const Gemm& g) {
  const size_t sm = sizeof(double) * (size_t)g.k * MT;
  if (sm > 48 * 1024)
    VL_CUDA(cudaFuncSetAttribute(thin_tn_kernel<MT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
  const int blocks = (int)std::max<int64_t>(1, std::min<int64_t>(((int64_t)g.n + 7) / 8, 4LL * C.num_sms));
  thin_tn_kernel<MT><<<blocks, 256, sm, C.stream>>>(g.n, g.k, g.A, g.lda, g.B, g.ldb, g.alpha, g.beta, g.C, g.ldc);
  VL_LAUNCH_CHECK();
}

void dgemm(Ctx& C, const Gemm& g) {
  if (g.m <= 0 || g.n <= 0) return;
  if (g.lower && g.m != g.n) fail(kEInternal, "dgemm: lower mode needs a square output");
  if (!g.lower && !g.ta && g.tb && g.n <= kThinMax && g.k >= 4096) {
    // C (m x n<=8) = A B^T with a long contraction: thread per row, split over k
    switch (g.n) {
      case 1: thin_nt<1>(C, g); return;
      case 2: thin_nt<2>(C, g); return;
      case 3: thin_nt<3>(C, g); return;
      case 4: thin_nt<4>(C, g); return;
      case 5: thin_nt<5>(C, g); return;
      case 6: thin_nt<6>(C, g); return;
      case 7: thin_nt<7>(C, g); return;
      default: thin_nt<8>(C, g); return;
    }
  }
  if (!g.lower && g.ta && !g.tb && g.m <= kThinMax && g.kw == nullptr &&
      (size_t)g.k * kThinMax * sizeof(double) <= 200 * 1024) {
    switch (g.m) {
      case 1: thin_tn<1>(C, g); return;
      case 2: thin_tn<2>(C, g); return;
      case 3: thin_tn<3>(C, g); return;
      case 4: thin_tn<4>(C, g); return;
      case 5: thin_tn<5>(C, g); return;
      case 6: thin_tn<6>(C, g); return;
      case 7: thin_tn<7>(C, g); return;
      default: thin_tn<8>(C, g); return;
    }
  }
  // tensor-core tiles (128 x 128) unless an output side is thin (GEMV-like products stay on
  // the 64 x 64 FMA tiles, where the padded tensor tile would only add operand traffic)
  static const int tc_mode = [] {
    const char* e = std::getenv("VL_DGEMM_TC");
    return e ? std::atoi(e) : 1;
  }();
  const bool tc = tc_mode != 0 && g.m >= 64 && g.n >= 64;
  const int TBM = tc ? DBM : GBM, TBN = tc ? DBN : GBN;
  const int tm = (g.m + TBM - 1) / TBM, tn = (g.n + TBN - 1) / TBN;
  int64_t tiles = (int64_t)tm * tn;
  if (g.lower) tiles = (tiles + tm) / 2;
  // split the contraction so the grid fills whole waves of one CTA per SM (>= 90% of the last
  // wave busy, at most 4 waves), keeping >= 256 of k per split
  int splits = 1;
  if (g.k > 0 && tiles < 4LL * C.num_sms) {
    const int smax = (int)std::max<int64_t>(1, std::min<int64_t>(64, g.k / 256));
    double best = 0.0;
    for (int sp = 1; sp <= smax; ++sp) {
      const int64_t ctas = tiles * sp;
      if (ctas > 4LL * C.num_sms) break;
      const int64_t waves = (ctas + C.num_sms - 1) / C.num_sms;
      const double eff = (double)ctas / (double)(waves * C.num_sms);
      const double score = eff * std::min<double>(1.0, (double)ctas / (2.0 * C.num_sms));
      if (score > best + 1e-9) { best = score; splits = sp; }
    }
  }
  int kchunk = (g.k + splits - 1) / splits;
  kchunk = (kchunk + GBK - 1) / GBK * GBK;
  if (kchunk == 0) kchunk = GBK;
  splits = g.k > 0 ? (g.k + kchunk - 1) / kchunk : 1;
  double* part = nullptr;
  DevBuf ws;
  if (splits > 1) {
    ws.alloc(sizeof(double) * (size_t)splits * g.m * g.n);
    part = ws.as<double>();
  }
  const dim3 grid(tm, tn, splits);
  if (g.ta) {
    if (g.tb) launch_gemm<true, true>(C, g, grid, kchunk, part, tc);
    else launch_gemm<true, false>(C, g, grid, kchunk, part, tc);
  } else {
    if (g.tb) launch_gemm<false, true>(C, g, grid, kchunk, part, tc);
    else launch_gemm<false, false>(C, g, grid, kchunk, part, tc);
  }
  if (splits > 1) {
    const int64_t total = (int64_t)g.m * g.n;
    const int blocks = (int)std::max<int64_t>(1, std::min<int64_t>((total + 255) / 256, 8LL * C.num_sms));
    splitk_reduce_kernel<<<blocks, 256, 0, C.stream>>>(g.m, g.n, splits, g.alpha, part, g.beta, g.C, g.ldc,
                                                       g.lower ? 1 : 0, (int64_t)g.m * g.n);
    VL_LAUNCH_CHECK();
  }
}

void dtrtri_lower(Ctx& C, int k, const double* L, int ldl, double* Li, int ldi) {
  if (k <= 0) return;
  const int nb = (k + 63) / 64;
  zero_upper_kernel<<<std::max(1, std::min(8 * C.num_sms, (int)(((int64_t)k * k + 255) / 256))), 256, 0, C.stream>>>(
      k, Li, ldi);
  VL_LAUNCH_CHECK();
  trtri_diag_kernel<<<nb, 64, 0, C.stream>>>(k, L, ldl, Li, ldi);
  VL_LAUNCH_CHECK();
  if (nb == 1) return;
  DevBuf T;
  T.alloc(sizeof(double) * 64 * (size_t)k);
  for (int b = 1; b < nb; ++b) {
    const int r0 = b * 64, bs = std::min(64, k - r0);
    // T (bs x r0) = L[r0:r0+bs, 0:r0] Li[0:r0, 0:r0]
    Gemm g1;
    g1.m = bs; g1.n = r0; g1.k = r0;
    g1.A = L + r0; g1.lda = ldl;
    g1.B = Li; g1.ldb = ldi;
    g1.C = T.as<double>(); g1.ldc = bs;
    dgemm(C, g1);
    // Li[r0:r0+bs, 0:r0] = -Li[r0:r0+bs, r0:r0+bs] T
    Gemm g2;
    g2.m = bs; g2.n = r0; g2.k = bs;
    g2.alpha = -1.0;
    g2.A = Li + r0 + (int64_t)r0 * ldi; g2.lda = ldi;
    g2.B = T.as<double>(); g2.ldb = bs;
    g2.C = Li + r0; g2.ldc = ldi;
    dgemm(C, g2);
  }
}

}  // namespace vl
