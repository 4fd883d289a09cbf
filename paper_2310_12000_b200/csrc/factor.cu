// Vecchia factor build + theta-gradient (fused), one warp per row.
//
// Reference: vecchia.py:101-127 (_submatrices, Cholesky PD check),
// vecchia.py:220-283 (build_factor: A = K^-1 k, D = sigma2 - k.A, D floor),
// vecchia.py:286-337 (factor_gradient: dA = K^-1 (dk - dK A),
// dD = dc(0) - dA.k - A.dk; sigma2: dB = 0, dD = D / sigma2).
//
// The reference solves with LU (np.linalg.solve) and uses Cholesky only as
// a PD check; here the Cholesky factor is reused for both solves (the two
// differ by rounding only).
#include <cuda_runtime.h>

#include "common.cuh"
#include "context.h"
#include "launch.cuh"

namespace vl {

struct Matern {
  double s2, rho, c;  // c = sqrt(3)/rho or sqrt(5)/rho or 1/rho (nu = 0.5 uses r / rho)
  int nu;             // 0: 0.5, 1: 1.5, 2: 2.5
  VL_D double val(double r) const {
    if (nu == 0) return s2 * exp(-r / rho);
    double u = c * r;
    if (nu == 1) return s2 * (1.0 + u) * exp(-u);
    return s2 * (1.0 + u + u * u / 3.0) * exp(-u);
  }
  VL_D double drho(double r) const {
    if (nu == 0) {
      double u = r / rho;
      return s2 * exp(-u) * u / rho;
    }
    double u = c * r;
    if (nu == 1) return s2 * u * u * exp(-u) / rho;
    return s2 * u * u * (1.0 + u) * exp(-u) / (3.0 * rho);
  }
};

template <int DIM>
VL_D double pdist(const double* a, const double* b, int d) {
  double s = 0.0;
  if (DIM > 0) {
#pragma unroll
    for (int k = 0; k < DIM; ++k) { double t = a[k] - b[k]; s += t * t; }
  } else {
    for (int k = 0; k < d; ++k) { double t = a[k] - b[k]; s += t * t; }
  }
  return sqrt(s);
}

// Per-warp scratch layout (doubles): X[mp*d] | L[mp*(mp+1)] | kv | dk | A | y | rhs | dA  (mp each)
VL_HD size_t warp_scratch_doubles(int mp, int d) { return (size_t)mp * d + (size_t)mp * (mp + 1) + 6 * (size_t)mp; }

// Forward then backward substitution with the Cholesky factor in Ls (row
// stride ld): solves (L L^T) x = b.  b in bv (smem), x written to xv.  Lanes
// own rows j = lane + 32 q.
template <int Q>
VL_D void chol_solve(const double* Ls, int ld, int c, const double* bv, double* yv, double* xv, int lane) {
  double acc[Q];
#pragma unroll
  for (int q = 0; q < Q; ++q) acc[q] = 0.0;
  for (int col = 0; col < c; ++col) {
    // lane owning col finalises y_col
    if ((col & 31) == lane) {
      int q = col >> 5;
      double a = 0.0;
#pragma unroll
      for (int qq = 0; qq < Q; ++qq) if (qq == q) a = acc[qq];
      yv[col] = (bv[col] - a) / Ls[col * ld + col];
    }
    __syncwarp();
    double ycol = yv[col];
#pragma unroll
    for (int q = 0; q < Q; ++q) {
      int j = lane + 32 * q;
      if (j > col && j < c) acc[q] += Ls[j * ld + col] * ycol;
    }
  }
  __syncwarp();
#pragma unroll
  for (int q = 0; q < Q; ++q) acc[q] = 0.0;
  for (int col = c - 1; col >= 0; --col) {
    if ((col & 31) == lane) {
      int q = col >> 5;
      double a = 0.0;
#pragma unroll
      for (int qq = 0; qq < Q; ++qq) if (qq == q) a = acc[qq];
      xv[col] = (yv[col] - a) / Ls[col * ld + col];
    }
    __syncwarp();
    double xcol = xv[col];
#pragma unroll
    for (int q = 0; q < Q; ++q) {
      int l = lane + 32 * q;
      if (l < col) acc[q] += Ls[col * ld + l] * xcol;
    }
  }
  __syncwarp();
}

template <int Q, int DIM>
__global__ void __launch_bounds__(128) factor_build_kernel(
    int64_t n, int d, int m, const double* __restrict__ xy, const int32_t* __restrict__ nbr,
    const int32_t* __restrict__ cnt, const int32_t* __restrict__ fidx, Matern K, int want_grad,
    double* __restrict__ val, double* __restrict__ Dout, double* __restrict__ dval,
    double* __restrict__ dD_rho, double* __restrict__ dD_sig, int* __restrict__ err,
    double* __restrict__ gscratch, int use_smem, const double* __restrict__ txy, int dfloor) {
  // txy: target coordinates of row s (prediction points) or null (row s = point s of xy);
  // dfloor: report D_s < 1e-10 sigma2 (factor rows; prediction_blocks has no such check)
  extern __shared__ double smem[];
  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;
  const int64_t gw = (int64_t)blockIdx.x * (blockDim.x >> 5) + wib;
  const int64_t nw = (int64_t)gridDim.x * (blockDim.x >> 5);
  const int mp = m > 0 ? m : 1;
  const size_t per = warp_scratch_doubles(mp, d);
  double* base = use_smem ? (smem + per * wib) : (gscratch + per * gw);
  double* X = base;
  double* L = X + (size_t)mp * d;
  const int ld = mp + 1;
  double* kv = L + (size_t)mp * ld;
  double* dk = kv + mp;
  double* A = dk + mp;
  double* yv = A + mp;
  double* rhs = yv + mp;
  double* dA = rhs + mp;
  const double dc0 = K.drho(0.0);

  for (int64_t s = gw; s < n; s += nw) {
    const int c = cnt[s];
    const double* xi = (txy ? txy : xy) + s * d;
    const int fs = fidx ? fidx[s] : (int)s;
    if (c == 0) {
      if (lane == 0) {
        Dout[s] = K.s2;
        if (want_grad) { dD_rho[s] = dc0; dD_sig[s] = K.s2 / K.s2; }
      }
      for (int j = lane; j < m; j += 32) {
        val[s * m + j] = 0.0;
        if (want_grad) dval[s * m + j] = 0.0;
      }
      continue;
    }
    // gather neighbour coordinates
    for (int j = lane; j < c; j += 32) {
      const double* xj = xy + (int64_t)nbr[s * m + j] * d;
      for (int k = 0; k < d; ++k) X[j * d + k] = xj[k];
    }
    __syncwarp();
    // K (lower triangle incl. diagonal) and k
#pragma unroll
    for (int q = 0; q < Q; ++q) {
      int j = lane + 32 * q;
      if (j < c) {
        for (int l = 0; l <= j; ++l) L[j * ld + l] = K.val(pdist<DIM>(X + j * d, X + l * d, d));
        double r = pdist<DIM>(X + j * d, xi, d);
        kv[j] = K.val(r);
        if (want_grad) dk[j] = K.drho(r);
      }
    }
    __syncwarp();
    // right-looking Cholesky
    bool ok = true;
    for (int col = 0; col < c; ++col) {
      double piv = L[col * ld + col];
      if (!(piv > 0.0)) { ok = false; break; }  // warp-uniform (same smem value)
      double dp = sqrt(piv);
      __syncwarp();
#pragma unroll
      for (int q = 0; q < Q; ++q) {
        int j = lane + 32 * q;
        if (j == col) L[j * ld + col] = dp;
        else if (j > col && j < c) L[j * ld + col] /= dp;
      }
      __syncwarp();
#pragma unroll
      for (int q = 0; q < Q; ++q) {
        int j = lane + 32 * q;
        if (j > col && j < c) {
          double ljc = L[j * ld + col];
          for (int l = col + 1; l <= j; ++l) L[j * ld + l] -= ljc * L[l * ld + col];
        }
      }
      __syncwarp();
    }
    if (!ok) {
      if (lane == 0) {
        atomicMin(err + 1, fs);
        atomicMax(err + 0, 1);
      }
      __syncwarp();
      continue;
    }
    // A = K^-1 k ; D = sigma2 - k.A
    chol_solve<Q>(L, ld, c, kv, yv, A, lane);
    double part = 0.0;
#pragma unroll
    for (int q = 0; q < Q; ++q) {
      int j = lane + 32 * q;
      if (j < c) part += kv[j] * A[j];
    }
    double kA = warp_sum(part);
    double Ds = K.s2 - kA;
    if (lane == 0) {
      Dout[s] = Ds;
      if (dfloor && !(Ds >= 1e-10 * K.s2)) { atomicMin(err + 2, fs); atomicMax(err + 0, 1); }
    }
    for (int j = lane; j < m; j += 32) val[s * m + j] = (j < c) ? -A[j] : 0.0;
    if (want_grad) {
      // rhs_j = dk_j - sum_l dK[j,l] A_l   (full symmetric row; vecchia.py:318-321)
#pragma unroll
      for (int q = 0; q < Q; ++q) {
        int j = lane + 32 * q;
        if (j < c) {
          double acc = 0.0;
          for (int l = 0; l < c; ++l) acc += K.drho(pdist<DIM>(X + j * d, X + l * d, d)) * A[l];
          rhs[j] = dk[j] - acc;
        }
      }
      __syncwarp();
      chol_solve<Q>(L, ld, c, rhs, yv, dA, lane);
      double p1 = 0.0, p2 = 0.0;
#pragma unroll
      for (int q = 0; q < Q; ++q) {
        int j = lane + 32 * q;
        if (j < c) { p1 += dA[j] * kv[j]; p2 += A[j] * dk[j]; }
      }
      p1 = warp_sum(p1);
      p2 = warp_sum(p2);
      if (lane == 0) {
        dD_rho[s] = dc0 + (-p1 - p2);
        dD_sig[s] = Ds / K.s2;
      }
      for (int j = lane; j < m; j += 32) dval[s * m + j] = (j < c) ? -dA[j] : 0.0;
    }
    __syncwarp();
  }
}

__global__ void gather_values_kernel(int64_t nnz, const int32_t* __restrict__ map, const double* __restrict__ src,
                                     double* __restrict__ dst) {
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < nnz; p += (int64_t)gridDim.x * blockDim.x)
    dst[p] = src[map[p]];
}

// X = B_HH^-1, one warp per column (see head.cuh).  Column c is zero above
// row c (head order is topological), so substitution starts at row c.
__global__ void __launch_bounds__(128) head_inverse_kernel(int H, int m, const int32_t* __restrict__ head_rows,
                                                           const int32_t* __restrict__ head_nbr,
                                                           const int32_t* __restrict__ cnt,
                                                           const double* __restrict__ val, double* __restrict__ X) {
  extern __shared__ double xc[];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  double* xcol = xc + (size_t)w * H;
  for (int c = blockIdx.x * 4 + w; c < H; c += gridDim.x * 4) {
    for (int r = c; r < H; ++r) {
      const int64_t s = head_rows[r];
      const int cs = cnt[s];
      double part = 0.0;
      if (lane < cs) {
        const int q = head_nbr[(int64_t)r * m + lane];
        if (q >= c) part = val[s * m + lane] * xcol[q];
      }
      part = warp_sum(part);
      const double xr = (r == c ? 1.0 : 0.0) - part;
      if (lane == 0) {
        xcol[r] = xr;
        X[(size_t)c * H + r] = xr;
      }
      __syncwarp();
    }
  }
}

__global__ void transpose_kernel(int H, const double* __restrict__ A, double* __restrict__ B) {
  __shared__ double tile[32][33];
  const int x = blockIdx.x * 32 + threadIdx.x;
  for (int k = 0; k < 32; k += blockDim.y) {
    const int y = blockIdx.y * 32 + threadIdx.y + k;
    tile[threadIdx.y + k][threadIdx.x] = (x < H && y < H) ? A[(size_t)y * H + x] : 0.0;
  }
  __syncthreads();
  const int x2 = blockIdx.y * 32 + threadIdx.x;
  for (int k = 0; k < 32; k += blockDim.y) {
    const int y2 = blockIdx.x * 32 + threadIdx.y + k;
    if (x2 < H && y2 < H) B[(size_t)y2 * H + x2] = tile[threadIdx.x][threadIdx.y + k];
  }
}

void factor_head_inverse(Ctx& C, Factor& F) {
  const Pattern& P = *F.pat;
  if (P.head_H <= 0 || P.m > 32) return;
  const int H = (int)P.head_H;
  F.headX.alloc(sizeof(double) * (size_t)H * H);
  const size_t smem = sizeof(double) * 4 * (size_t)H;
  VL_CUDA(cudaFuncSetAttribute(head_inverse_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  int occ = 0;
  VL_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, head_inverse_kernel, 128, smem));
  const int blocks = std::max(1, std::min((H + 3) / 4, std::max(occ, 1) * C.num_sms));
  ProfScope ps(C, "factor_head_inverse", 0.0);
  C.prof.launches++;
  cudaEvent_t ev = (C.prof.on && C.prof.tag) ? prof_begin(C) : nullptr;
  head_inverse_kernel<<<blocks, 128, smem, C.stream>>>(H, P.m, P.head_rows.as<int32_t>(), P.head_nbr.as<int32_t>(),
                                                       P.cnt.as<int32_t>(), F.val.as<double>(), F.headX.as<double>());
  VL_LAUNCH_CHECK();
  // row-major copy for the forward single-column GEMV (headX is column-major)
  F.headXr.alloc(sizeof(double) * (size_t)H * H);
  transpose_kernel<<<dim3((H + 31) / 32, (H + 31) / 32), dim3(32, 8), 0, C.stream>>>(H, F.headX.as<double>(),
                                                                                     F.headXr.as<double>());
  VL_LAUNCH_CHECK();
  if (ev) prof_end(C, ev);
}

__global__ void slab_values_kernel(int64_t ne, const int32_t* __restrict__ map, const double* __restrict__ val,
                                   double* __restrict__ sv) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < ne; i += (int64_t)gridDim.x * blockDim.x) {
    const int32_t q = map[i];
    sv[i] = q >= 0 ? val[q] : 0.0;
  }
}

void factor_refresh_transpose(Ctx& C, Factor& F) {
  const Pattern& P = *F.pat;
  if (P.nnz_off > 0) {
    int blocks = C.num_sms * 8;
    gather_values_kernel<<<blocks, 256, 0, C.stream>>>(P.nnz_off, P.tmap.as<int32_t>(), F.val.as<double>(),
                                                       F.valT.as<double>());
    VL_LAUNCH_CHECK();
  }
  auto slab = [&](const Pattern::Slabs& S, DevBuf& sv) {
    sv.alloc(sizeof(double) * std::max<int64_t>(S.nent, 1));
    if (S.nent > 0) {
      slab_values_kernel<<<C.num_sms * 8, 256, 0, C.stream>>>(S.nent, S.map.as<int32_t>(), F.val.as<double>(),
                                                              sv.as<double>());
      VL_LAUNCH_CHECK();
    }
  };
  if (P.has_solve_order) {
    const int64_t ne = (int64_t)P.n * P.m;
    F.val_s.alloc(sizeof(double) * ne);
    slab_values_kernel<<<C.num_sms * 8, 256, 0, C.stream>>>(ne, P.map_s.as<int32_t>(), F.val.as<double>(),
                                                            F.val_s.as<double>());
    VL_LAUNCH_CHECK();
  }
  slab(P.fwd_sl, F.sv_fwd);
  slab(P.bwd_sl, F.sv_bwd);
  slab(P.bwdnh_sl, F.sv_bwdnh);
  factor_head_inverse(C, F);  // dense B_HH^-1 for the solves' head block
}

template <int Q, int DIM>
static void launch_build(Ctx& C, const Pattern& P, Factor& F, const Matern& K, int want_grad, double* gscr,
                         int use_smem, size_t per) {
  const int threads = 128;
  const int wpb = threads / 32;
  size_t smem = use_smem ? per * wpb * sizeof(double) : 0;
  if (use_smem && smem > 48 * 1024)
    VL_CUDA(cudaFuncSetAttribute(factor_build_kernel<Q, DIM>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  int blocks;
  if (use_smem) {
    int occ = 0;
    VL_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, factor_build_kernel<Q, DIM>, threads, smem));
    occ = occ > 0 ? occ : 1;
    int64_t need = (P.n + wpb - 1) / wpb;
    blocks = (int)std::min<int64_t>(need, (int64_t)occ * C.num_sms);
  } else {
    blocks = C.num_sms * 2;
  }
  if (blocks < 1) blocks = 1;
  ProfScope ps(C, "factor_build", 0.0);
  C.prof.launches++;
  cudaEvent_t ev = (C.prof.on && C.prof.tag) ? prof_begin(C) : nullptr;
  factor_build_kernel<Q, DIM><<<blocks, threads, smem, C.stream>>>(
      P.n, P.d, P.m, P.xy.as<double>(), P.nbr.as<int32_t>(), P.cnt.as<int32_t>(), P.fidx.as<int32_t>(), K, want_grad,
      F.val.as<double>(), F.D.as<double>(), want_grad ? F.dval.as<double>() : nullptr,
      want_grad ? F.dD_rho.as<double>() : nullptr, want_grad ? F.dD_sig.as<double>() : nullptr, F.err.as<int>(), gscr,
      use_smem, nullptr, 1);
  VL_LAUNCH_CHECK();
  if (ev) prof_end(C, ev);
}

template <int Q>
static void launch_build_q(Ctx& C, const Pattern& P, Factor& F, const Matern& K, int want_grad, double* gscr,
                           int use_smem, size_t per) {
  if (P.d == 2) launch_build<Q, 2>(C, P, F, K, want_grad, gscr, use_smem, per);
  else if (P.d == 1) launch_build<Q, 1>(C, P, F, K, want_grad, gscr, use_smem, per);
  else launch_build<Q, 0>(C, P, F, K, want_grad, gscr, use_smem, per);
}

// Build (B, D) and optionally d/d(sigma2, rho); errors -> FactorizationError
void factor_build(Ctx& C, const Pattern& P, Factor& F, double sigma2, double rho, double nu, bool want_grad) {
  Matern K;
  K.s2 = sigma2;
  K.rho = rho;
  if (nu == 0.5) { K.nu = 0; K.c = 1.0 / rho; }
  else if (nu == 1.5) { K.nu = 1; K.c = sqrt(3.0) / rho; }
  else if (nu == 2.5) { K.nu = 2; K.c = sqrt(5.0) / rho; }
  else fail(kEConfig, "smoothness nu must be one of (0.5, 1.5, 2.5)");
  if (!(sigma2 > 0)) fail(kEConfig, "sigma2 must be > 0");
  if (!(rho > 0)) fail(kEConfig, "rho must be > 0");
  F.pat = &P;
  F.sigma2 = sigma2;
  F.rho = rho;
  F.nu = nu;
  F.has_grad = want_grad;
  const int64_t n = P.n;
  const int mm = std::max(P.m, 1);
  F.val.alloc(sizeof(double) * n * mm);
  F.D.alloc(sizeof(double) * n);
  F.valT.alloc(sizeof(double) * std::max<int64_t>(P.nnz_off, 1));
  F.err.alloc(sizeof(int) * 4);
  if (want_grad) {
    F.dval.alloc(sizeof(double) * n * mm);
    F.dD_rho.alloc(sizeof(double) * n);
    F.dD_sig.alloc(sizeof(double) * n);
  }
  int h_err[4] = {0, INT32_MAX, INT32_MAX, 0};
  VL_CUDA(cudaMemcpyAsync(F.err.p, h_err, sizeof(h_err), cudaMemcpyHostToDevice, C.stream));
  const int mp = mm;
  const size_t per = warp_scratch_doubles(mp, P.d);
  const int use_smem = (per * 4 * sizeof(double) <= 200 * 1024) ? 1 : 0;
  DevBuf gscr;
  if (!use_smem) gscr.alloc(per * sizeof(double) * (size_t)C.num_sms * 2 * 4);
  double* g = gscr.as<double>();
  if (mp <= 32) launch_build_q<1>(C, P, F, K, want_grad, g, use_smem, per);
  else if (mp <= 64) launch_build_q<2>(C, P, F, K, want_grad, g, use_smem, per);
  else if (mp <= 128) launch_build_q<4>(C, P, F, K, want_grad, g, use_smem, per);
  else if (mp <= 256) launch_build_q<8>(C, P, F, K, want_grad, g, use_smem, per);
  else fail(kECapacity, "m > 256 neighbours is not supported");
  factor_refresh_transpose(C, F);
  VL_CUDA(cudaMemcpyAsync(h_err, F.err.p, sizeof(h_err), cudaMemcpyDeviceToHost, C.stream));
  VL_CUDA(cudaStreamSynchronize(C.stream));
  if (h_err[0]) {
    if (h_err[1] != INT32_MAX)
      fail(kEFactorization, "neighbor covariance submatrix of point " + std::to_string(h_err[1]) +
                                " (factor order) is not positive definite (near-duplicate locations?)");
    fail(kEFactorization, "conditional variance D_" + std::to_string(h_err[2]) +
                              " below 1e-10 * sigma2 (near-duplicate inputs)");
  }
}

// ---------------------------------------------------------------------------
// Prediction blocks (vecchia.py:393-441): each prediction point conditions on
// its `take` nearest training points; A = K^-1 k (Bpo row = -A), Dp = sigma2 -
// k.A, by the factor-build warp kernel with external target coordinates.
// ---------------------------------------------------------------------------
template <int Q, int DIM>
static void launch_pred(Ctx& C, const Pattern& P, const Matern& K, int64_t np, int take, const double* qxy,
                        const int32_t* nbr, const int32_t* cnt, double* A, double* Dp, int* err, size_t per) {
  const int threads = 128;
  const int wpb = threads / 32;
  const size_t smem = per * wpb * sizeof(double);
  const int use_smem = smem <= 200 * 1024 ? 1 : 0;
  DevBuf gscr;
  int blocks;
  if (use_smem) {
    if (smem > 48 * 1024)
      VL_CUDA(cudaFuncSetAttribute(factor_build_kernel<Q, DIM>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)smem));
    int occ = 0;
    VL_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, factor_build_kernel<Q, DIM>, threads, smem));
    occ = occ > 0 ? occ : 1;
    blocks = (int)std::max<int64_t>(1, std::min<int64_t>((np + wpb - 1) / wpb, (int64_t)occ * C.num_sms));
  } else {
    blocks = C.num_sms * 2;
    gscr.alloc(per * sizeof(double) * (size_t)blocks * wpb);
  }
  factor_build_kernel<Q, DIM><<<blocks, threads, use_smem ? smem : 0, C.stream>>>(
      np, P.d, take, P.xy.as<double>(), nbr, cnt, nullptr, K, 0, A, Dp, nullptr, nullptr, nullptr, err,
      gscr.as<double>(), use_smem, qxy, 0);
  VL_LAUNCH_CHECK();
}

void pred_build(Ctx& C, const Pattern& P, double sigma2, double rho, double nu, const double* qxy_dev, int64_t np,
                int take, const int32_t* nbr_dev, const int32_t* cnt_dev, double* A_dev, double* Dp_dev) {
  Matern K;
  K.s2 = sigma2;
  K.rho = rho;
  if (nu == 0.5) { K.nu = 0; K.c = 1.0 / rho; }
  else if (nu == 1.5) { K.nu = 1; K.c = sqrt(3.0) / rho; }
  else if (nu == 2.5) { K.nu = 2; K.c = sqrt(5.0) / rho; }
  else fail(kEConfig, "smoothness nu must be one of (0.5, 1.5, 2.5)");
  if (np == 0) return;
  if (take < 1 || take > 256) fail(kECapacity, "prediction neighbour count must be in [1, 256]");
  DevBuf err;
  err.alloc(sizeof(int) * 4);
  int h_err[4] = {0, INT32_MAX, INT32_MAX, 0};
  VL_CUDA(cudaMemcpyAsync(err.p, h_err, sizeof(h_err), cudaMemcpyHostToDevice, C.stream));
  const size_t per = warp_scratch_doubles(take, P.d);
  auto go = [&](auto qq) {
    constexpr int Q = decltype(qq)::value;
    if (P.d == 2) launch_pred<Q, 2>(C, P, K, np, take, qxy_dev, nbr_dev, cnt_dev, A_dev, Dp_dev, err.as<int>(), per);
    else if (P.d == 1) launch_pred<Q, 1>(C, P, K, np, take, qxy_dev, nbr_dev, cnt_dev, A_dev, Dp_dev, err.as<int>(), per);
    else launch_pred<Q, 0>(C, P, K, np, take, qxy_dev, nbr_dev, cnt_dev, A_dev, Dp_dev, err.as<int>(), per);
  };
  if (take <= 32) go(std::integral_constant<int, 1>{});
  else if (take <= 64) go(std::integral_constant<int, 2>{});
  else if (take <= 128) go(std::integral_constant<int, 4>{});
  else go(std::integral_constant<int, 8>{});
  VL_CUDA(cudaMemcpyAsync(h_err, err.p, sizeof(h_err), cudaMemcpyDeviceToHost, C.stream));
  VL_CUDA(cudaStreamSynchronize(C.stream));
  if (h_err[0] && h_err[1] != INT32_MAX)
    fail(kEFactorization, "neighbor covariance submatrix of prediction point " + std::to_string(h_err[1]) +
                              " is not positive definite");
}

}  // namespace vl
