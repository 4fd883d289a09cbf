// Rank-k Lanczos predictive variances on the device (
// predict.py:104-172, iterative.py:181-219).
//
// The reference materialises RT = Bpo^T densely (n x n_p) and forms
// S = Q^T RT.  Here RT stays sparse (take entries per prediction point):
//   S^T = Bpo Q'   (n_p x k, a gather over the take nearest training rows),
// with the variant's transformation moved from RT onto the k Lanczos vectors:
//   none: RT            -> Q' = Q
//   l1  : RT2 = sd^-1 o B^-T RT          -> Q' = B^-1 (Q / sd)
//   l2  : right = is o SigmaTilde RT     -> Q'r = SigmaTilde (is o Q)
//         left  = is o RT / W            -> Q'l = Q o (is / W)
// (sd = sqrt(W + 1/D), is = 1/sqrt(diag(SigmaTilde) + 1/W)), so memory is
// O((n + n_p) k) instead of O(n n_p).  The Lanczos recurrence (full
// reorthogonalisation, applied twice) keeps its basis as k contiguous
// n-vectors; products and solves with B run on the library's own kernels.
#include <cmath>

#include "bodies.cuh"
#include "launch.cuh"
#include "ops.h"
#include "predict.h"

namespace vl {

namespace {

constexpr int kLzThreads = 256;
constexpr int kLzRowsPerBlock = 4096;  // rows of one partial-dot block

// ---- n-vector helpers --------------------------------------------------------
// out_i = a_i * s1_i^p1 * s2_i^p2 (p in {-1, 0, 1}; null scale = 1), optionally + add_i
// (add and out may alias: element-wise)
__global__ void scale_kernel(int64_t n, const double* a, const double* __restrict__ s1, int p1,
                             const double* __restrict__ s2, int p2, const double* add, double* out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    double v = a[i];
    if (s1) v = p1 > 0 ? v * s1[i] : v / s1[i];
    if (s2) v = p2 > 0 ? v * s2[i] : v / s2[i];
    if (add) v += add[i];
    out[i] = v;
  }
}

// sd = sqrt(W + 1/D) (l1) / is = 1/sqrt(dsig + 1/W) (l2)
__global__ void variant_scale_kernel(int64_t n, int l2, const double* __restrict__ W, const double* __restrict__ D,
                                     const double* __restrict__ dsig, double* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = l2 ? 1.0 / sqrt(dsig[i] + 1.0 / W[i]) : sqrt(W[i] + 1.0 / D[i]);
}

__global__ void count_nonpos_kernel(int64_t n, const double* __restrict__ W, int* __restrict__ out) {
  int c = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    c += !(W[i] > 0.0);
  if (c) atomicAdd(out, c);
}

// Partial dots of w against nq basis vectors: part[b * nq + j] = sum over the
// block's rows of Q[j][i] * w[i] (fixed order: thread-strided, xor tree, warp
// order), folded by dots_fold_kernel in block order -> deterministic.
__global__ void __launch_bounds__(kLzThreads) dots_part_kernel(int64_t n, int nq, const double* __restrict__ Q,
                                                               const double* __restrict__ w,
                                                               double* __restrict__ part) {
  __shared__ double red[kLzThreads / 32];
  const int64_t r0 = (int64_t)blockIdx.x * kLzRowsPerBlock;
  const int64_t r1 = r0 + kLzRowsPerBlock < n ? r0 + kLzRowsPerBlock : n;
  constexpr int K = kLzRowsPerBlock / kLzThreads;
  double wv[K];
#pragma unroll
  for (int k = 0; k < K; ++k) {
    const int64_t i = r0 + threadIdx.x + (int64_t)k * kLzThreads;
    wv[k] = i < r1 ? w[i] : 0.0;
  }
  for (int j = 0; j < nq; ++j) {
    const double* q = Q + (int64_t)j * n;
    double s = 0.0;
#pragma unroll
    for (int k = 0; k < K; ++k) {
      const int64_t i = r0 + threadIdx.x + (int64_t)k * kLzThreads;
      if (i < r1) s = fma(q[i], wv[k], s);
    }
    s = warp_sum(s);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
      double tot = 0.0;
#pragma unroll
      for (int k = 0; k < kLzThreads / 32; ++k) tot += red[k];
      part[(int64_t)blockIdx.x * nq + j] = tot;
    }
    __syncthreads();
  }
}

__global__ void dots_fold_kernel(int nb, int nq, const double* __restrict__ part, double* __restrict__ out) {
  const int j = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (j >= nq) return;
  const int lane = threadIdx.x & 31;
  double s = 0.0;
  for (int b = lane; b < nb; b += 32) s += part[(int64_t)b * nq + j];
  s = warp_sum(s);
  if (lane == 0) out[j] = s;
}

// w_i -= sum_j c_j Q[j][i]  (c scaled by cs: the alpha / beta steps reuse it)
__global__ void __launch_bounds__(kLzThreads) axpy_basis_kernel(int64_t n, int nq, const double* __restrict__ Q,
                                                                const double* __restrict__ c,
                                                                double* __restrict__ w) {
  extern __shared__ double cs[];
  for (int j = threadIdx.x; j < nq; j += blockDim.x) cs[j] = c[j];
  __syncthreads();
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    double v = w[i];
    int j = 0;
    for (; j + 4 <= nq; j += 4) {
      const double q0 = Q[(int64_t)j * n + i], q1 = Q[(int64_t)(j + 1) * n + i];
      const double q2 = Q[(int64_t)(j + 2) * n + i], q3 = Q[(int64_t)(j + 3) * n + i];
      v = fma(-cs[j], q0, v);
      v = fma(-cs[j + 1], q1, v);
      v = fma(-cs[j + 2], q2, v);
      v = fma(-cs[j + 3], q3, v);
    }
    for (; j < nq; ++j) v = fma(-cs[j], Q[(int64_t)j * n + i], v);
    w[i] = v;
  }
}

// w -= a q  -  b p   (p may be null)
__global__ void lanczos_sub_kernel(int64_t n, double a, const double* __restrict__ q, double b,
                                   const double* __restrict__ p, double* __restrict__ w) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    double v = w[i] - a * q[i];
    if (p) v -= b * p[i];
    w[i] = v;
  }
}

__global__ void scal_to_kernel(int64_t n, double inv, const double* __restrict__ w, double* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = w[i] / inv;
}

// Basis vectors [c0, c0 + cw) (vector-major, kk x n) -> row-major n x ldo panel,
// each entry scaled by s1^p1 * s2^p2 of its row; through a 32 x 33 tile.
__global__ void panel_kernel(int64_t n, int c0, int cw, const double* __restrict__ Q, const double* __restrict__ s1,
                             int p1, const double* __restrict__ s2, int p2, double* __restrict__ out, int ldo) {
  __shared__ double tile[32][33];
  const int64_t i0 = (int64_t)blockIdx.x * 32;
  const int j0 = blockIdx.y * 32;
  for (int jj = threadIdx.y; jj < 32; jj += blockDim.y) {
    const int j = j0 + jj;
    const int64_t i = i0 + threadIdx.x;
    tile[jj][threadIdx.x] = (j < cw && i < n) ? Q[(int64_t)(c0 + j) * n + i] : 0.0;
  }
  __syncthreads();
  for (int ii = threadIdx.y; ii < 32; ii += blockDim.y) {
    const int64_t i = i0 + ii;
    const int j = j0 + threadIdx.x;
    if (i < n && j < cw) {
      double v = tile[threadIdx.x][ii];
      if (s1) v = p1 > 0 ? v * s1[i] : v / s1[i];
      if (s2) v = p2 > 0 ? v * s2[i] : v / s2[i];
      out[i * ldo + j] = v;
    }
  }
}

// rows of an n x c panel scaled in place by s_i
__global__ void panel_rowscale_kernel(int64_t n, int c, int ld, const double* __restrict__ s, double* __restrict__ X) {
  const int64_t total = n * c;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = e / c;
    const int j = (int)(e - i * c);
    X[i * ld + j] *= s[i];
  }
}

// S^T panel = Bpo X  (as PredRowsBody in predict.cu, own copy with strided output)
struct BpoPanelBody {
  const int32_t* nbr;
  const double* val;
  int take;
  const double* X;
  int ldx;
  double* Z;
  int ldz;
  template <int G, int NU, int U, int NR>
  VL_D void run(int64_t q, bool valid, int gl, int t, double (&)[NR][NU * U]) const {
    if (!valid) return;
    double a[NU * U];
    zero(a);
    const int32_t* nb = nbr + q * take;
    const double* vv = val + q * take;
    gather<G, NU, U>(
        take, gl, t, [&](int e) { return nb[e]; }, [&](int e) { return vv[e]; }, LoadU<U>{X, ldx}, a);
    store_row<G, NU, U>(Z, ldz, q, gl, t, a);
  }
};

// corr_p = sl_p^T T^-1 sr_p with T = L diag(d) L^T (unit lower bidiagonal L,
// sub-diagonal l): forward sweep, diagonal scaling, backward sweep per
// prediction point; the row's k entries stay in L1 between the sweeps.
__global__ void tri_corr_kernel(int64_t np, int kk, int ld, const double* __restrict__ Sr,
                                const double* __restrict__ Sl, const double* __restrict__ dl,
                                const double* __restrict__ Dp, double* __restrict__ work, double* __restrict__ var) {
  const double* dd = dl;        // kk pivots
  const double* ll = dl + kk;   // kk - 1 multipliers
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < np; p += (int64_t)gridDim.x * blockDim.x) {
    const double* sr = Sr + p * ld;
    const double* sl = Sl + p * ld;
    double* y = work + p * ld;
    double prev = sr[0];
    y[0] = prev;
    for (int j = 1; j < kk; ++j) {
      prev = sr[j] - ll[j - 1] * prev;
      y[j] = prev;
    }
    double x = y[kk - 1] / dd[kk - 1];
    double acc = sl[kk - 1] * x;
    for (int j = kk - 2; j >= 0; --j) {
      x = y[j] / dd[j] - ll[j] * x;
      acc += sl[j] * x;
    }
    var[p] = Dp[p] + acc;
  }
}

__global__ void copy_dp_kernel(int64_t np, const double* __restrict__ Dp, double* __restrict__ var) {
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < np; p += (int64_t)gridDim.x * blockDim.x)
    var[p] = Dp[p];
}

inline int nblocks(Ctx& C, int64_t n) {
  return (int)std::max<int64_t>(1, std::min<int64_t>((n + kLzThreads - 1) / kLzThreads, 8LL * C.num_sms));
}

struct Lz {
  Ctx& C;
  const Factor& F;
  int64_t n;
  DevBuf part, dbuf, tmp1, tmp2;

  Lz(Ctx& c, const Factor& f, int k) : C(c), F(f), n(f.pat->n) {
    tmp1.alloc(sizeof(double) * n);
    tmp2.alloc(sizeof(double) * n);
    dbuf.alloc(sizeof(double) * 8);
    part.alloc(sizeof(double) * (size_t)((n + kLzRowsPerBlock - 1) / kLzRowsPerBlock) * std::max(k, 1));
  }
  void scale(const double* a, const double* s1, int p1, const double* s2, int p2, const double* add, double* out) {
    scale_kernel<<<nblocks(C, n), kLzThreads, 0, C.stream>>>(n, a, s1, p1, s2, p2, add, out);
    VL_LAUNCH_CHECK();
  }
  // dots of w against nq contiguous n-vectors starting at Q -> host (synchronises)
  void dots(int nq, const double* Q, const double* w, double* out_dev, std::vector<double>* out_host) {
    const int nb = (int)((n + kLzRowsPerBlock - 1) / kLzRowsPerBlock);
    dots_part_kernel<<<nb, kLzThreads, 0, C.stream>>>(n, nq, Q, w, part.as<double>());
    VL_LAUNCH_CHECK();
    dots_fold_kernel<<<(nq + 7) / 8, 256, 0, C.stream>>>(nb, nq, part.as<double>(), out_dev);
    VL_LAUNCH_CHECK();
    if (out_host) {
      out_host->resize(nq);
      VL_CUDA(cudaMemcpyAsync(out_host->data(), out_dev, sizeof(double) * nq, cudaMemcpyDeviceToHost, C.stream));
      VL_CUDA(cudaStreamSynchronize(C.stream));
    }
  }
  double dot(const double* a, const double* b) {
    std::vector<double> h;
    dots(1, a, b, dbuf.as<double>(), &h);
    return h[0];
  }
  // precision product y = B^T (D^-1 (B x))  (vecchia.py:176-180)
  void precision(const double* x, double* y) {
    op_spmm(C, F, 0, 1, 1, x, tmp1.as<double>());
    scale(tmp1.as<double>(), F.D.as<double>(), -1, nullptr, 0, nullptr, tmp2.as<double>());
    op_spmm(C, F, 1, 1, 1, tmp2.as<double>(), y);
  }
  // SigmaTilde x = B^-1 (D o B^-T x)  (vecchia.py:182-186)
  void sigma_tilde(const double* x, double* y) {
    op_trsv(C, F, true, 1, 1, x, tmp1.as<double>());
    scale(tmp1.as<double>(), F.D.as<double>(), 1, nullptr, 0, nullptr, tmp2.as<double>());
    op_trsv(C, F, false, 1, 1, tmp2.as<double>(), y);
  }
};

}  // namespace

int pred_lanczos(Ctx& C, const Factor& F, const PredBlocks& B, const double* W, int variant, int k,
                 const double* start_raw, const double* dsig, double breakdown_tol, double* var_out) {
  const int64_t n = F.pat->n, np = B.np;
  if (k < 1 || k > n) fail(kEConfig, "rank k must be in [1, n]");
  if (variant < 0 || variant > 2) fail(kEConfig, "unknown Lanczos variant");
  if (variant == 2 && !dsig) fail(kEConfig, "l2 variant needs diag(SigmaTilde)");
  ProfScope ps(C, "pred_lanczos", 0.0);
  Lz z(C, F, k);
  const double* D = F.D.as<double>();
  DevBuf sc, x1, x2, wv, cbuf;
  sc.alloc(sizeof(double) * n);
  x1.alloc(sizeof(double) * n);
  x2.alloc(sizeof(double) * n);
  wv.alloc(sizeof(double) * n);
  cbuf.alloc(sizeof(double) * (size_t)k);
  double* s = sc.as<double>();
  if (variant == 2) {
    DevBuf cnt;
    cnt.alloc(sizeof(int));
    VL_CUDA(cudaMemsetAsync(cnt.p, 0, sizeof(int), C.stream));
    count_nonpos_kernel<<<nblocks(C, n), kLzThreads, 0, C.stream>>>(n, W, cnt.as<int>());
    VL_LAUNCH_CHECK();
    int bad = 0;
    VL_CUDA(cudaMemcpyAsync(&bad, cnt.p, sizeof(int), cudaMemcpyDeviceToHost, C.stream));
    VL_CUDA(cudaStreamSynchronize(C.stream));
    if (bad) fail(kECapability, "l2 variant needs W > 0 everywhere");
  }
  if (variant) {
    variant_scale_kernel<<<nblocks(C, n), kLzThreads, 0, C.stream>>>(n, variant == 2, W, D, dsig, s);
    VL_LAUNCH_CHECK();
  }

  // operator of the variant (predict.py:139-168)
  auto matvec = [&](const double* v, double* y) {
    if (variant == 0) {
      z.precision(v, x1.as<double>());
      z.scale(v, W, 1, nullptr, 0, x1.as<double>(), y);
    } else if (variant == 1) {
      z.scale(v, s, -1, nullptr, 0, nullptr, x1.as<double>());
      op_trsv(C, F, false, 1, 1, x1.as<double>(), x2.as<double>());        // x = B^-1 (v / sd)
      z.precision(x2.as<double>(), x1.as<double>());
      z.scale(x2.as<double>(), W, 1, nullptr, 0, x1.as<double>(), x1.as<double>());  // W x + Q x
      op_trsv(C, F, true, 1, 1, x1.as<double>(), x2.as<double>());
      z.scale(x2.as<double>(), s, -1, nullptr, 0, nullptr, y);
    } else {
      z.scale(v, s, 1, nullptr, 0, nullptr, x1.as<double>());              // x = is o v
      z.sigma_tilde(x1.as<double>(), x2.as<double>());
      z.scale(x1.as<double>(), W, -1, nullptr, 0, x2.as<double>(), x2.as<double>());  // SigmaTilde x + x / W
      z.scale(x2.as<double>(), s, 1, nullptr, 0, nullptr, y);
    }
  };

  // start vector = column mean of the variant's RT_right (linear in RT: apply the
  // transformation to the mean of the sparse columns)
  DevBuf Q;
  Q.alloc(sizeof(double) * (size_t)n * k);
  double* q0 = Q.as<double>();
  if (variant == 0) {
    VL_CUDA(cudaMemcpyAsync(wv.p, start_raw, sizeof(double) * n, cudaMemcpyDeviceToDevice, C.stream));
  } else if (variant == 1) {
    op_trsv(C, F, true, 1, 1, start_raw, x1.as<double>());
    z.scale(x1.as<double>(), s, -1, nullptr, 0, nullptr, wv.as<double>());
  } else {
    z.sigma_tilde(start_raw, x1.as<double>());
    z.scale(x1.as<double>(), s, 1, nullptr, 0, nullptr, wv.as<double>());
  }
  const double norm0 = std::sqrt(z.dot(wv.as<double>(), wv.as<double>()));
  auto no_correction = [&]() {
    if (np) {
      copy_dp_kernel<<<nblocks(C, np), kLzThreads, 0, C.stream>>>(np, B.Dp.as<double>(), var_out);
      VL_LAUNCH_CHECK();
    }
    return 0;
  };
  if (!(norm0 >= breakdown_tol)) return no_correction();
  scal_to_kernel<<<nblocks(C, n), kLzThreads, 0, C.stream>>>(n, norm0, wv.as<double>(), q0);
  VL_LAUNCH_CHECK();

  // ---- Lanczos with full reorthogonalisation, twice (iterative.py:181-219) ----
  std::vector<double> al(k), be(std::max(k - 1, 0)), hc;
  int achieved = k;
  double* w = wv.as<double>();
  for (int j = 0; j < k; ++j) {
    const double* qj = q0 + (int64_t)j * n;
    matvec(qj, w);
    al[j] = z.dot(qj, w);
    lanczos_sub_kernel<<<nblocks(C, n), kLzThreads, 0, C.stream>>>(n, al[j], qj, j > 0 ? be[j - 1] : 0.0,
                                                                   j > 0 ? qj - n : nullptr, w);
    VL_LAUNCH_CHECK();
    for (int rep = 0; rep < 2; ++rep) {
      z.dots(j + 1, q0, w, cbuf.as<double>(), nullptr);
      axpy_basis_kernel<<<nblocks(C, n), kLzThreads, sizeof(double) * (j + 1), C.stream>>>(n, j + 1, q0,
                                                                                            cbuf.as<double>(), w);
      VL_LAUNCH_CHECK();
    }
    if (j == k - 1) break;
    const double beta = std::sqrt(z.dot(w, w));
    if (beta < breakdown_tol) {
      achieved = j + 1;
      break;
    }
    be[j] = beta;
    scal_to_kernel<<<nblocks(C, n), kLzThreads, 0, C.stream>>>(n, beta, w, q0 + (int64_t)(j + 1) * n);
    VL_LAUNCH_CHECK();
  }
  const int kk = achieved;
  if (np == 0) return kk;

  // ---- T = L diag(d) L^T on the host (T is SPD: Lanczos of an SPD operator) ----
  std::vector<double> dl(2 * kk, 0.0);
  dl[0] = al[0];
  for (int j = 1; j < kk; ++j) {
    const double l = be[j - 1] / dl[j - 1];
    dl[kk + j - 1] = l;
    dl[j] = al[j] - l * be[j - 1];
  }
  for (int j = 0; j < kk; ++j)
    if (!(dl[j] > 0.0) || !std::isfinite(dl[j])) fail(kEBreakdown, "Lanczos tridiagonal is not positive definite");
  DevBuf dld;
  dld.alloc(sizeof(double) * 2 * kk);
  VL_CUDA(cudaMemcpyAsync(dld.p, dl.data(), sizeof(double) * 2 * kk, cudaMemcpyHostToDevice, C.stream));

  // ---- S^T = Bpo Q' in column panels (<= 128 columns per launch) ----
  const int ldz = kk + (kk & 1);
  DevBuf Zr, Zl, Zw, P1, P2;
  Zr.alloc(sizeof(double) * (size_t)np * ldz);
  Zw.alloc(sizeof(double) * (size_t)np * ldz);
  if (variant == 2) Zl.alloc(sizeof(double) * (size_t)np * ldz);
  constexpr int kPanel = 128;
  P1.alloc(sizeof(double) * (size_t)n * kPanel);
  if (variant) P2.alloc(sizeof(double) * (size_t)n * kPanel);
  auto panel = [&](int c0, int cw, int ld, const double* s1, int p1, const double* s2, int p2, double* out) {
    dim3 grid((unsigned)((n + 31) / 32), (unsigned)((cw + 31) / 32));
    panel_kernel<<<grid, dim3(32, 8), 0, C.stream>>>(n, c0, cw, q0, s1, p1, s2, p2, out, ld);
    VL_LAUNCH_CHECK();
  };
  auto bpo = [&](const double* X, int ld, int cw, double* Z) {
    dispatch_cols(cw, ld, [&](auto g, auto nu, auto uu) {
      constexpr int G = decltype(g)::value, NU = decltype(nu)::value, U = decltype(uu)::value;
      launch_rows<G, NU, U, 0, 0>(C, np, cw,
                                  BpoPanelBody{B.nbr.as<int32_t>(), B.val.as<double>(), B.take, X, ld, Z, ldz},
                                  Fin0<0>{});
    });
  };
  for (int c0 = 0; c0 < kk; c0 += kPanel) {
    const int cw = std::min(kPanel, kk - c0);
    // an odd panel is widened by one zero column (contiguous 16-byte column units: ld == t
    // even), so the solves and the gather treat the pad like any other column
    const int ct = cw + (cw & 1);
    if (ct != cw) VL_CUDA(cudaMemsetAsync(P1.p, 0, sizeof(double) * (size_t)n * ct, C.stream));
    if (variant == 0) {
      panel(c0, cw, ct, nullptr, 0, nullptr, 0, P1.as<double>());
      bpo(P1.as<double>(), ct, ct, Zr.as<double>() + c0);
    } else if (variant == 1) {
      panel(c0, cw, ct, s, -1, nullptr, 0, P1.as<double>());
      op_trsv(C, F, false, ct, ct, P1.as<double>(), P2.as<double>());
      bpo(P2.as<double>(), ct, ct, Zr.as<double>() + c0);
    } else {
      panel(c0, cw, ct, s, 1, W, -1, P1.as<double>());                     // left: Q o is / W
      bpo(P1.as<double>(), ct, ct, Zl.as<double>() + c0);
      panel(c0, cw, ct, s, 1, nullptr, 0, P1.as<double>());                // right: SigmaTilde (is o Q)
      op_trsv(C, F, true, ct, ct, P1.as<double>(), P2.as<double>());
      panel_rowscale_kernel<<<nblocks(C, n * ct), kLzThreads, 0, C.stream>>>(n, ct, ct, D, P2.as<double>());
      VL_LAUNCH_CHECK();
      op_trsv(C, F, false, ct, ct, P2.as<double>(), P1.as<double>());
      bpo(P1.as<double>(), ct, ct, Zr.as<double>() + c0);
    }
  }
  tri_corr_kernel<<<nblocks(C, np), kLzThreads, 0, C.stream>>>(np, kk, ldz, Zr.as<double>(),
                                                               variant == 2 ? Zl.as<double>() : Zr.as<double>(),
                                                               dld.as<double>(), B.Dp.as<double>(), Zw.as<double>(),
                                                               var_out);
  VL_LAUNCH_CHECK();
  VL_CUDA(cudaStreamSynchronize(C.stream));
  return kk;
}

}  // namespace vl
