// LRAC: low-rank pivoted Cholesky of the exact covariance + diag(1/W),
// Woodbury solves, eq7 operator SigmaTilde + W^-1 (preconditioners.py:167-214,
// 249-320; laplace.py:118-182).
//
// Hand-written: the pivoted Cholesky step (Matern row of the pivot + the
// n x j GEMV against the previous columns + diagonal update + deterministic
// argmax of the next pivot, all in one kernel per step), the sparse
// operator applies, all elementwise/reduction passes.  Library: the plain
// n x k GEMMs / k x k triangular solves of the Woodbury core (cuBLAS) and the
// k x k Cholesky of M (cuSOLVER potrf).
#include <cusolverDn.h>

#include <cmath>
#include <mutex>

#include "bodies.cuh"
#include "launch.cuh"
#include "lrac.h"
#include "dense.h"
#include "ops.h"
#include "pcg_common.cuh"

namespace vl {

namespace {

std::mutex g_h_mu;
cusolverDnHandle_t g_solv[16] = {};

cusolverDnHandle_t solver(Ctx& C) {
  std::lock_guard<std::mutex> lk(g_h_mu);
  cusolverDnHandle_t& h = g_solv[C.device & 15];
  if (!h) {
    if (cusolverDnCreate(&h) != CUSOLVER_STATUS_SUCCESS) fail(kECuda, "cusolverDnCreate failed");
  }
  cusolverDnSetStream(h, C.stream);
  return h;
}

struct MaternK {
  double s2, rho, c;
  int nu;
  VL_D double val(double r) const {
    if (nu == 0) return s2 * exp(-r / rho);
    const double u = c * r;
    if (nu == 1) return s2 * (1.0 + u) * exp(-u);
    return s2 * (1.0 + u + u * u / 3.0) * exp(-u);
  }
};

MaternK make_matern(const Factor& F) {
  MaternK K;
  K.s2 = F.sigma2;
  K.rho = F.rho;
  if (F.nu == 0.5) { K.nu = 0; K.c = 1.0 / F.rho; }
  else if (F.nu == 1.5) { K.nu = 1; K.c = std::sqrt(3.0) / F.rho; }
  else { K.nu = 2; K.c = std::sqrt(5.0) / F.rho; }
  return K;
}

// pivoted-Cholesky state (device): [0] pivot storage index, [1] stop, [2] err, [3] keff ; dp in doubles
struct PcState {
  int* i;
  double* dp;
};

constexpr int kPcThreads = 256;

__global__ void fill_kernel(int64_t n, double v, double* d) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    d[i] = v;
}

// One greedy step j (preconditioners.py:308-319): col = (Sigma[:, p] - L[:, :j] L[p, :j]) / sqrt(d_p),
// col_p = sqrt(d_p), d -= col^2, d_p = 0; then min(d), sum(max(d, 0)) and the argmax (ties -> lowest
// factor index) for step j+1, finalised by the last CTA.
__global__ void __launch_bounds__(kPcThreads) pchol_step_kernel(int64_t n, int dim, const double* __restrict__ xy,
                                                               const int32_t* __restrict__ fidx, MaternK K, int j,
                                                               int k, double* __restrict__ L, double* __restrict__ d,
                                                               PcState st, double tol, double* __restrict__ part,
                                                               unsigned* __restrict__ counter,
                                                               int32_t* __restrict__ piv_s,
                                                               const double* __restrict__ qc,
                                                               double* __restrict__ LT) {
  // qc: dense column of the matrix at the pivot (precision accessor) or null (Matern row of Sigma)
  // LT: column-major copy of L (k x n, column c contiguous over rows) for the
  // thread-per-row dot products (coalesced across the warp; L itself is
  // row-major for the Woodbury GEMMs)
  if (((volatile int*)st.i)[1] != 0) return;
  __shared__ double s_min[kPcThreads / 32], s_sum[kPcThreads / 32], s_max[kPcThreads / 32];
  __shared__ int s_arg[kPcThreads / 32];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int p = st.i[0];
  const double dp = *st.dp;
  const double sq = sqrt(dp);
  const double* Lp = L + (int64_t)p * k;
  const double* xp = xy + (int64_t)p * dim;
  double wmin = 1e300, wsum = 0.0, wmax = -1.0;
  int warg = 0x7fffffff;  // factor index of the best
  int wsrow = -1;
  // two threads per row: half-warp h (lanes 16h..16h+15) covers rows
  // base..base+15 and columns [h*jh, min(j, (h+1)*jh)); 8 independent loads
  // in flight per thread (coalesced 128 B per half-warp and column)
  const int half = lane >> 4;
  const int jh = (j + 1) >> 1;
  const int c0 = half * jh, c1 = min(j, c0 + jh);
  const int64_t rows_per_grid = ((int64_t)gridDim.x * blockDim.x) >> 1;
  const int64_t r0 = ((blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5) * 16 + (lane & 15);
  const int64_t nround = (n + rows_per_grid - 1) / rows_per_grid;
  for (int64_t rr = 0; rr < nround; ++rr) {
    const int64_t i = r0 + rr * rows_per_grid;
    const bool on = i < n;
    // dot = L[i, :j] . L[p, :j] in column order (Lp[c] is a warp-wide broadcast)
    double da = 0.0, db = 0.0;
    if (on) {
      const double* li = LT + i;
      int c = c0;
      for (; c + 8 <= c1; c += 8) {
        double a[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) a[q] = li[(int64_t)(c + q) * n];
#pragma unroll
        for (int q = 0; q < 8; q += 2) {
          da = fma(a[q], Lp[c + q], da);
          db = fma(a[q + 1], Lp[c + q + 1], db);
        }
      }
      for (; c < c1; ++c) da = fma(li[(int64_t)c * n], Lp[c], da);
    }
    double dot = da + db;
    dot += __shfl_xor_sync(0xffffffffu, dot, 16);  // the row's other half
    if (!on || half) continue;
    double src;
    if (qc) {
      src = qc[i];
    } else {
      double r2 = 0.0;
      for (int q = 0; q < dim; ++q) {
        const double df = xy[i * dim + q] - xp[q];
        r2 += df * df;
      }
      src = K.val(sqrt(r2));
    }
    double col = (src - dot) / sq;
    double di = fmax(d[i], 0.0);  // np.clip(d, 0) of this step
    if (i == p) col = sq;
    L[i * k + j] = col;
    LT[(int64_t)j * n + i] = col;
    di = di - col * col;
    if (i == p) di = 0.0;
    d[i] = di;
    wmin = fmin(wmin, di);
    const double dc = fmax(di, 0.0);
    wsum += dc;
    const int fi = fidx[i];
    if (dc > wmax || (dc == wmax && fi < warg)) {
      wmax = dc;
      warg = fi;
      wsrow = (int)i;
    }
  }
  // warp reduction (fixed xor tree), then lane 0 of each warp holds the warp's values
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    wmin = fmin(wmin, __shfl_xor_sync(0xffffffffu, wmin, o));
    wsum += __shfl_xor_sync(0xffffffffu, wsum, o);
    const double mx = __shfl_xor_sync(0xffffffffu, wmax, o);
    const int f = __shfl_xor_sync(0xffffffffu, warg, o);
    const int row = __shfl_xor_sync(0xffffffffu, wsrow, o);
    if (row >= 0 && (mx > wmax || (mx == wmax && f < warg))) {
      wmax = mx;
      warg = f;
      wsrow = row;
    }
  }
  // block reduction (lane 0 of each warp holds the warp's values)
  if (lane == 0) {
    s_min[wib] = wmin;
    s_sum[wib] = wsum;
    s_max[wib] = wmax;
    s_arg[wib] = wsrow;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double bmin = 1e300, bsum = 0.0, bmax = -1.0;
    int brow = -1, bf = 0x7fffffff;
    for (int w = 0; w < kPcThreads / 32; ++w) {
      bmin = fmin(bmin, s_min[w]);
      bsum += s_sum[w];
      if (s_arg[w] >= 0) {
        const int f = fidx[s_arg[w]];
        if (s_max[w] > bmax || (s_max[w] == bmax && f < bf)) {
          bmax = s_max[w];
          bf = f;
          brow = s_arg[w];
        }
      }
    }
    double* pb = part + (size_t)blockIdx.x * 4;
    pb[0] = bmin;
    pb[1] = bsum;
    pb[2] = bmax;
    pb[3] = (double)brow;
    __threadfence();
    s_arg[0] = (int)atomicAdd(counter, 1u);
  }
  __syncthreads();
  if (s_arg[0] != (int)gridDim.x - 1) return;
  // last CTA: all threads fold the per-block partials (thread-strided, then a
  // fixed shuffle / shared-memory tree: deterministic, and ~gridDim / 256
  // independent loads per thread instead of one thread walking gridDim
  // dependent loads).  Ties of the maximum go to the lowest factor index.
  __threadfence();
  double gmin = 1e300, gsum = 0.0, gmax = -1.0;
  int grow = -1, gf = 0x7fffffff;
  auto better = [&](double mx, int f) { return mx > gmax || (mx == gmax && f < gf); };
  for (unsigned bq = threadIdx.x; bq < gridDim.x; bq += blockDim.x) {
    const double* q = part + (size_t)bq * 4;
    gmin = fmin(gmin, __ldcg(q));
    gsum += __ldcg(q + 1);
    const int row = (int)__ldcg(q + 3);
    const double mx = __ldcg(q + 2);
    if (row >= 0) {
      const int f = fidx[row];
      if (better(mx, f)) {
        gmax = mx;
        gf = f;
        grow = row;
      }
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    gmin = fmin(gmin, __shfl_xor_sync(0xffffffffu, gmin, o));
    gsum += __shfl_xor_sync(0xffffffffu, gsum, o);
    const double mx = __shfl_xor_sync(0xffffffffu, gmax, o);
    const int f = __shfl_xor_sync(0xffffffffu, gf, o);
    const int row = __shfl_xor_sync(0xffffffffu, grow, o);
    if (row >= 0 && better(mx, f)) {
      gmax = mx;
      gf = f;
      grow = row;
    }
  }
  __syncthreads();  // s_* reused below
  if (lane == 0) {
    s_min[wib] = gmin;
    s_sum[wib] = gsum;
    s_max[wib] = gmax;
    s_arg[wib] = grow;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    gmin = 1e300;
    gsum = 0.0;
    gmax = -1.0;
    grow = -1;
    gf = 0x7fffffff;
    for (int w = 0; w < kPcThreads / 32; ++w) {
      gmin = fmin(gmin, s_min[w]);
      gsum += s_sum[w];
      if (s_arg[w] >= 0) {
        const int f = fidx[s_arg[w]];
        if (better(s_max[w], f)) {
          gmax = s_max[w];
          gf = f;
          grow = s_arg[w];
        }
      }
    }
    piv_s[j] = p;
    st.i[3] = j + 1;
    if (j + 1 < k) {
      if (gmin < -1e-10) {
        st.i[2] = 1;
        st.i[1] = 1;
      } else if (gsum <= tol || !(gmax > 0.0)) {
        st.i[1] = 1;
      } else {
        st.i[0] = grow;
        *st.dp = gmax;
      }
    }
    *counter = 0u;
  }
}


__global__ void add_identity_kernel(int k, double* M) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < k; i += gridDim.x * blockDim.x) M[(size_t)i * k + i] += 1.0;
}

__global__ void sumlog_diag_kernel(int k, const double* __restrict__ M, double* out) {
  __shared__ double sh[256];
  double s = 0.0;
  for (int i = threadIdx.x; i < k; i += blockDim.x) s += log(M[(size_t)i * k + i]);
  sh[threadIdx.x] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double a = 0.0;
    for (int i = 0; i < (int)blockDim.x; ++i) a += sh[i];
    *out = 2.0 * a;
  }
}

// ---- elementwise bodies -----------------------------------------------------------
struct MulWBody {  // x = W o r
  const double* W;
  const double* r;
  double* x;
  int ld;
  template <int G, int NU, int U, int NR>
  VL_D void run(int64_t s, bool valid, int gl, int t, double (&)[NR][NU * U]) const {
    if (!valid) return;
    double a[NU * U];
    load_row<G, NU, U>(r, ld, s, gl, t, a);
    const double w = W[s];
#pragma unroll
    for (int i = 0; i < NU * U; ++i) a[i] *= w;
    store_row<G, NU, U>(x, ld, s, gl, t, a);
  }
};
template <bool DOT>
struct WoodFinishBody {  // z = x - W o y ; acc += r . z
  const double* W;
  const double* x;
  const double* y;
  const double* r;
  double* z;
  int ld;
  template <int G, int NU, int U, int NR>
  VL_D void run(int64_t s, bool valid, int gl, int t, double (&acc)[NR][NU * U]) const {
    if (!valid) return;
    double a[NU * U], b[NU * U], rr[NU * U];
    load_row<G, NU, U>(x, ld, s, gl, t, a);
    load_row<G, NU, U>(y, ld, s, gl, t, b);
    const double w = W[s];
#pragma unroll
    for (int i = 0; i < NU * U; ++i) a[i] = a[i] - w * b[i];
    store_row<G, NU, U>(z, ld, s, gl, t, a);
    if (DOT) {
      load_row<G, NU, U>(r, ld, s, gl, t, rr);
#pragma unroll
      for (int i = 0; i < NU * U; ++i) acc[0][i] += rr[i] * a[i];
    }
  }
};
struct Eq7FinishBody {  // v = sx + h / W ; acc += h . v
  const double* W;
  const double* sx;
  const double* h;
  double* v;
  int ld;
  template <int G, int NU, int U, int NR>
  VL_D void run(int64_t s, bool valid, int gl, int t, double (&acc)[NR][NU * U]) const {
    if (!valid) return;
    double a[NU * U], hs[NU * U];
    load_row<G, NU, U>(sx, ld, s, gl, t, a);
    load_row<G, NU, U>(h, ld, s, gl, t, hs);
    const double w = W[s];
#pragma unroll
    for (int i = 0; i < NU * U; ++i) {
      a[i] = a[i] + hs[i] / w;
      acc[0][i] += hs[i] * a[i];
    }
    store_row<G, NU, U>(v, ld, s, gl, t, a);
  }
};
struct UpdBody {  // r -= alpha v ; u += alpha h ; acc += r^2  (active columns)
  double* r;
  double* u;
  const double* v;
  const double* h;
  const double* alpha;
  const int* active;
  int ld;
  template <int G, int NU, int U, int NR>
  VL_D void run(int64_t s, bool valid, int gl, int t, double (&acc)[NR][NU * U]) const {
    if (!valid) return;
#pragma unroll
    for (int i = 0; i < NU * U; ++i) {
      const int c = vl::Cols<G, NU, U>::col(gl, i);
      if (c >= t || !active[c]) continue;
      const int64_t o = s * ld + c;
      const double al = alpha[c];
      const double rn = r[o] - al * v[o];
      r[o] = rn;
      u[o] = u[o] + al * h[o];
      acc[0][i] += rn * rn;
    }
  }
};
struct DivWBody {  // y = x / W
  const double* W;
  const double* x;
  double* y;
  int ld;
  template <int G, int NU, int U, int NR>
  VL_D void run(int64_t s, bool valid, int gl, int t, double (&)[NR][NU * U]) const {
    if (!valid) return;
    double a[NU * U];
    load_row<G, NU, U>(x, ld, s, gl, t, a);
    const double w = W[s];
#pragma unroll
    for (int i = 0; i < NU * U; ++i) a[i] /= w;
    store_row<G, NU, U>(y, ld, s, gl, t, a);
  }
};
struct RhsScaleD {  // trsv rhs = D o w
  const double* w;
  const double* D;
  int ld;
  VL_D double rhs(int64_t s, int c, double&) const { return w[s * ld + c] * D[s]; }
  VL_D void out(int64_t, int, double, double&) const {}
};
struct PrecK1Body {  // tmp = D^-1 (B h)
  BView B;
  const double* h;
  double* tmp;
  const double* D;
  int ld;
  template <int G, int NU, int U, int NR>
  VL_D void run(int64_t s, bool valid, int gl, int t, double (&)[NR][NU * U]) const {
    double a[NU * U];
    zero(a);
    gather_B<G, NU, U>(B, B.val, s, valid, gl, t, LoadU<U>{h, ld}, a);
    if (!valid) return;
    double hs[NU * U];
    load_row<G, NU, U>(h, ld, s, gl, t, hs);
    const double di = 1.0 / D[s];
#pragma unroll
    for (int i = 0; i < NU * U; ++i) a[i] = di * (hs[i] + a[i]);
    store_row<G, NU, U>(tmp, ld, s, gl, t, a);
  }
};
struct PrecK2Body {  // v = W h + B^T tmp ; acc += h . v
  BView B;
  const double* h;
  const double* tmp;
  double* v;
  const double* W;
  int ld;
  template <int G, int NU, int U, int NR>
  VL_D void run(int64_t s, bool valid, int gl, int t, double (&acc)[NR][NU * U]) const {
    double a[NU * U];
    zero(a);
    gather_Bt<G, NU, U>(B, s, valid, gl, t, LoadU<U>{tmp, ld}, a);
    if (!valid) return;
    double ts[NU * U], hs[NU * U];
    load_row<G, NU, U>(tmp, ld, s, gl, t, ts);
    load_row<G, NU, U>(h, ld, s, gl, t, hs);
    const double ws = W[s];
#pragma unroll
    for (int i = 0; i < NU * U; ++i) {
      a[i] = ws * hs[i] + (ts[i] + a[i]);
      acc[0][i] += hs[i] * a[i];
    }
    store_row<G, NU, U>(v, ld, s, gl, t, a);
  }
};
struct RzFin {
  cg::CgCols K;
  VL_D void operator()(const double* sums, int t) const {
    for (int c = threadIdx.x; c < t; c += blockDim.x) K.rz[c] = sums[c];
  }
};

}  // namespace

void lrac_free_handles() {
  std::lock_guard<std::mutex> lk(g_h_mu);
  for (auto& h : g_solv)
    if (h) { cusolverDnDestroy(h); h = nullptr; }
}

void lrac_pchol(Ctx& C, const Factor& F, LracFactor& LF, int k, double tol) {
  const Pattern& P = *F.pat;
  const int64_t n = P.n;
  if (k < 1 || k > n) fail(kEConfig, "rank k must be in [1, " + std::to_string(n) + "]");
  LF.k = k;
  LF.L.alloc(sizeof(double) * (size_t)n * k);
  VL_CUDA(cudaMemsetAsync(LF.L.p, 0, sizeof(double) * (size_t)n * k, C.stream));
  LF.piv_s.alloc(sizeof(int32_t) * k);
  DevBuf d, st, part;
  d.alloc(sizeof(double) * n);
  st.alloc(64);
  const int grid = std::min<int64_t>(C.num_sms * 8, (2 * n + kPcThreads - 1) / kPcThreads);
  DevBuf LT;  // column-major copy of L for the step kernel's dot products
  LT.alloc(sizeof(double) * (size_t)n * k);
  part.alloc(sizeof(double) * 4 * (size_t)grid);
  fill_kernel<<<C.num_sms * 4, 256, 0, C.stream>>>(n, F.sigma2, d.as<double>());
  int h_i[4] = {P.iperm[0], 0, 0, 0};  // first pivot: all d equal -> lowest factor index
  double h_dp = F.sigma2;
  VL_CUDA(cudaMemcpyAsync(st.p, h_i, sizeof(h_i), cudaMemcpyHostToDevice, C.stream));
  VL_CUDA(cudaMemcpyAsync(st.as<char>() + 32, &h_dp, sizeof(double), cudaMemcpyHostToDevice, C.stream));
  PcState S{st.as<int>(), reinterpret_cast<double*>(st.as<char>() + 32)};
  const MaternK K = make_matern(F);
  unsigned* counter = next_counter(C);
  ProfScope ps(C, "lrac_pchol", 0.0);
  cudaEvent_t pev = (C.prof.on && C.prof.tag) ? prof_begin(C) : nullptr;  // the k steps as one timed region
  for (int j = 0; j < k; ++j) {
    pchol_step_kernel<<<grid, kPcThreads, 0, C.stream>>>(n, P.d, P.xy.as<double>(), P.fidx.as<int32_t>(), K, j, k,
                                                         LF.L.as<double>(), d.as<double>(), S, tol,
                                                         part.as<double>(), counter, LF.piv_s.as<int32_t>(), nullptr,
                                                         LT.as<double>());
    VL_LAUNCH_CHECK();
    C.prof.launches++;
  }
  if (pev) prof_end(C, pev);
  VL_CUDA(cudaMemcpyAsync(h_i, st.p, sizeof(h_i), cudaMemcpyDeviceToHost, C.stream));
  VL_CUDA(cudaStreamSynchronize(C.stream));
  if (h_i[2]) fail(kEFactorization, "pivoted Cholesky: diagonal went negative; input not PSD");
  LF.keff = h_i[3];
  std::vector<int32_t> ps_(LF.keff);
  if (LF.keff) VL_CUDA(cudaMemcpy(ps_.data(), LF.piv_s.p, sizeof(int32_t) * LF.keff, cudaMemcpyDeviceToHost));
  LF.piv_f.resize(LF.keff);
  for (int q = 0; q < LF.keff; ++q) LF.piv_f[q] = P.sperm[ps_[q]];
}

void lrac_prepare(Ctx& C, const Factor& F, const LracFactor& LF, const double* W, LracPrec& Pr) {
  lowrank_prepare(C, F, &LF, W, nullptr, 0, Pr);
}

void lowrank_prepare(Ctx& C, const Factor& F, const LracFactor* LFp, const double* Wop, const double* einv, int eq6,
                     LracPrec& Pr) {
  const Pattern& P = *F.pat;
  const int64_t n = P.n;
  Pr.F = &F;
  Pr.LF = LFp ? LFp : &Pr.empty;
  const LracFactor& LF = *Pr.LF;
  const double* W = einv ? einv : Wop;
  const int k = LF.keff;
  Pr.W = W;
  Pr.Wop = Wop;
  Pr.eq6 = eq6;
  Pr.sumlogW = lrac_sumlogW(C, n, W);
  if (k == 0) {
    Pr.logdetM = 0.0;
    return;
  }
  ProfScope ps(C, "lrac_prepare", 0.0);
  DevBuf info, ld;
  Pr.Lm.alloc(sizeof(double) * (size_t)k * k);
  // M = L^T diag(W) L (lower triangle): L (n x LF.k row-major) is the column-major (LF.k x n)
  // matrix A, so M = A diag(W) A^T -- the hand-written weighted SYRK (dense.cu), no scaled copy of L
  {
    Gemm g;
    g.tb = true;
    g.m = k; g.n = k; g.k = (int)n;
    g.A = LF.L.as<double>(); g.lda = LF.k;
    g.B = LF.L.as<double>(); g.ldb = LF.k;
    g.C = Pr.Lm.as<double>(); g.ldc = k;
    g.kw = W;
    g.lower = true;
    dgemm(C, g);
  }
  add_identity_kernel<<<8, 256, 0, C.stream>>>(k, Pr.Lm.as<double>());
  VL_LAUNCH_CHECK();
  cusolverDnHandle_t sh = solver(C);
  int lwork = 0;
  if (cusolverDnDpotrf_bufferSize(sh, CUBLAS_FILL_MODE_LOWER, k, Pr.Lm.as<double>(), k, &lwork) !=
      CUSOLVER_STATUS_SUCCESS)
    fail(kECuda, "potrf buffer size");
  DevBuf work;
  work.alloc(sizeof(double) * std::max(lwork, 1));
  info.alloc(64);
  if (cusolverDnDpotrf(sh, CUBLAS_FILL_MODE_LOWER, k, Pr.Lm.as<double>(), k, work.as<double>(), lwork,
                       info.as<int>()) != CUSOLVER_STATUS_SUCCESS)
    fail(kECuda, "potrf");
  ld.alloc(64);
  sumlog_diag_kernel<<<1, 256, 0, C.stream>>>(k, Pr.Lm.as<double>(), ld.as<double>());
  int h_info = 0;
  VL_CUDA(cudaMemcpyAsync(&h_info, info.p, sizeof(int), cudaMemcpyDeviceToHost, C.stream));
  VL_CUDA(cudaMemcpyAsync(&Pr.logdetM, ld.p, sizeof(double), cudaMemcpyDeviceToHost, C.stream));
  VL_CUDA(cudaStreamSynchronize(C.stream));
  if (h_info != 0) fail(kEFactorization, "LRAC Woodbury core M is not positive definite");
  // explicit Lm^-1 and M^-1 = Lm^-T Lm^-1: the Woodbury solves become one k x k product
  Pr.Lmi.alloc(sizeof(double) * (size_t)k * k);
  Pr.Minv.alloc(sizeof(double) * (size_t)k * k);
  dtrtri_lower(C, k, Pr.Lm.as<double>(), k, Pr.Lmi.as<double>(), k);
  Gemm g;
  g.ta = true;
  g.m = k; g.n = k; g.k = k;
  g.A = Pr.Lmi.as<double>(); g.lda = k;
  g.B = Pr.Lmi.as<double>(); g.ldb = k;
  g.C = Pr.Minv.as<double>(); g.ldc = k;
  dgemm(C, g);
}

// z = W o r - W o (L M^-1 L^T (W o r))
template <bool DOT, class Fin>
static void woodbury(Ctx& C, const LracPrec& Pr, int t, const double* r, double* z, const Fin& fin, const int* gate) {
  const Pattern& P = *Pr.F->pat;
  const int64_t n = P.n;
  const int k = Pr.LF->keff, kl = Pr.LF->k;
  DevBuf x, y, w;
  x.alloc(sizeof(double) * (size_t)n * t);
  y.alloc(sizeof(double) * (size_t)n * t);
  w.alloc(sizeof(double) * (size_t)std::max(k, 1) * t);
  dispatch_cols(t, t, [&](auto g, auto nu, auto uu) {
    constexpr int G = decltype(g)::value, NU = decltype(nu)::value, U = decltype(uu)::value;
    launch_rows<G, NU, U, 0, 0>(C, n, t, MulWBody{Pr.W, r, x.as<double>(), t}, Fin0<0>{}, gate);
  });
  if (k > 0) {
    DevBuf u;
    u.alloc(sizeof(double) * (size_t)k * t);
    // w (k x t) = A (k x n) x^T ; A = L^T viewed column-major (lda = kl), x viewed (t x n, ld t)
    Gemm g1;
    g1.tb = true;
    g1.m = k; g1.n = t; g1.k = (int)n;
    g1.A = Pr.LF->L.as<double>(); g1.lda = kl;
    g1.B = x.as<double>(); g1.ldb = t;
    g1.C = w.as<double>(); g1.ldc = k;
    dgemm(C, g1);
    // u = M^-1 w
    Gemm g2;
    g2.m = k; g2.n = t; g2.k = k;
    g2.A = Pr.Minv.as<double>(); g2.lda = k;
    g2.B = w.as<double>(); g2.ldb = k;
    g2.C = u.as<double>(); g2.ldc = k;
    dgemm(C, g2);
    // y (t x n, column-major) = u^T (t x k) A (k x n)
    Gemm g3;
    g3.ta = true;
    g3.m = t; g3.n = (int)n; g3.k = k;
    g3.A = u.as<double>(); g3.lda = k;
    g3.B = Pr.LF->L.as<double>(); g3.ldb = kl;
    g3.C = y.as<double>(); g3.ldc = t;
    dgemm(C, g3);
  } else {
    VL_CUDA(cudaMemsetAsync(y.p, 0, sizeof(double) * (size_t)n * t, C.stream));
  }
  dispatch_cols(t, t, [&](auto g, auto nu, auto uu) {
    constexpr int G = decltype(g)::value, NU = decltype(nu)::value, U = decltype(uu)::value;
    launch_rows<G, NU, U, DOT ? 1 : 0, 0>(C, n, t, WoodFinishBody<DOT>{Pr.W, x.as<double>(), y.as<double>(), r, z, t},
                                         fin, gate);
  });
}

void lrac_apply_inv(Ctx& C, const LracPrec& Pr, int t, const double* r, double* z) {
  woodbury<false>(C, Pr, t, r, z, Fin0<0>{}, nullptr);
}

void apply_sigma_tilde(Ctx& C, const Factor& F, int t, const double* x, double* y, double* scratch) {
  const Pattern& P = *F.pat;
  DepsEll dfw = deps_fwd(F);
  DepsCsr dbw{P.tptr.as<int32_t>(), P.tidx.as<int32_t>(), F.valT.as<double>()};
  dispatch_cols(t, t, [&](auto g, auto nu, auto uu) {
    constexpr int G = decltype(g)::value, NU = decltype(nu)::value, U = decltype(uu)::value;
    launch_trsv<G, NU, U, 0>(C, F, false, t, t, dbw, scratch, TrsvPlain{x, t}, Fin0<0>{});
    launch_trsv<G, NU, U, 0>(C, F, true, t, t, dfw, y, RhsScaleD{scratch, F.D.as<double>(), t}, Fin0<0>{});
  });
}

void pcg_lrac(Ctx& C, const LracPrec& Pr, int t, const double* b, double* u, double tol, int max_iter, bool capture,
              PcgResult* out) {
  using namespace cg;
  const Factor& F = *Pr.F;
  const Pattern& P = *F.pat;
  const int64_t n = P.n;
  if (!(tol > 0)) fail(kEConfig, "tol must be > 0");
  const size_t vb = sizeof(double) * (size_t)n * t;
  DevBuf r, z, v, h, sx, scr;
  r.alloc(vb); z.alloc(vb); v.alloc(vb); h.alloc(vb); sx.alloc(vb); scr.alloc(vb);
  const int cap = capture ? std::max(max_iter, 1) : 1;
  DevBuf colsd, colsi, hist;
  colsd.alloc(sizeof(double) * (7 * (size_t)t + 1));
  colsi.alloc(sizeof(int) * (3 * (size_t)t + 4));
  hist.alloc(sizeof(double) * 2 * (size_t)cap * t);
  CgCols K;
  double* cd = colsd.as<double>();
  K.nb = cd; K.rz = cd + t; K.alpha = cd + 2 * t; K.beta = cd + 3 * t; K.res = cd + 4 * t; K.tolnb = cd + 5 * t;
  K.errval = cd + 7 * t;
  int* ci = colsi.as<int>();
  K.active = ci; K.iters = ci + t; K.conv = ci + 2 * t; K.status = ci + 3 * t;
  K.ah = hist.as<double>();
  K.bh = K.ah + (size_t)cap * t;
  const int* gate = K.status;
  const Pattern& PP = P;
  DepsEll dfw = deps_fwd(F);
  DepsCsr dbw{PP.tptr.as<int32_t>(), PP.tidx.as<int32_t>(), F.valT.as<double>()};
  int status[3] = {0, 0, 0};
  dispatch_cols(t, t, [&](auto g, auto nu, auto uu) {
    constexpr int G = decltype(g)::value, NU = decltype(nu)::value, U = decltype(uu)::value;
    ProfScope ps(C, t == 1 ? "lrac1_cg" : "lracT_cg", 0.0);
    launch_rows<G, NU, U, 1, 0>(C, n, t, InitBody{b, r.as<double>(), u, h.as<double>(), t}, InitFin{K, tol});
    woodbury<true>(C, Pr, t, r.as<double>(), z.as<double>(), RzFin{K}, gate);
    int l = 0, chunk = 4;
    while (l < max_iter) {
      const int lim = std::min(max_iter, l + chunk);
      for (; l < lim; ++l) {
        launch_rows<G, NU, U, 0, 0>(C, n, t, HUpdBody{z.as<double>(), h.as<double>(), K.beta, t}, Fin0<0>{}, gate);
        // v = SigmaTilde h + h / W  (eq7)  or  W h + Q h  (eq6)
        if (Pr.eq6) {  // v = W h + B^T D^-1 B h
          launch_rows<G, NU, U, 0, 0>(C, n, t, PrecK1Body{bview(F, false), h.as<double>(), sx.as<double>(),
                                                          F.D.as<double>(), t},
                                      Fin0<0>{}, gate);
          launch_rows<G, NU, U, 1, 0>(C, n, t, PrecK2Body{bview(F, false), h.as<double>(), sx.as<double>(),
                                                          v.as<double>(), Pr.Wop, t},
                                      K2Fin{K, l, cap}, gate);
        } else {
          launch_trsv<G, NU, U, 0>(C, F, false, t, t, dbw, scr.as<double>(), TrsvPlain{h.as<double>(), t},
                                   Fin0<0>{}, gate);
          launch_trsv<G, NU, U, 0>(C, F, true, t, t, dfw, sx.as<double>(),
                                   RhsScaleD{scr.as<double>(), F.D.as<double>(), t}, Fin0<0>{}, gate);
          launch_rows<G, NU, U, 1, 0>(C, n, t,
                                      Eq7FinishBody{Pr.Wop, sx.as<double>(), h.as<double>(), v.as<double>(), t},
                                      K2Fin{K, l, cap}, gate);
        }
        launch_rows<G, NU, U, 1, 0>(C, n, t,
                                    UpdBody{r.as<double>(), u, v.as<double>(), h.as<double>(), K.alpha, K.active, t},
                                    K3Fin{K, l}, gate);
        woodbury<true>(C, Pr, t, r.as<double>(), z.as<double>(), K4Fin{K, l, cap}, gate);
      }
      VL_CUDA(cudaMemcpyAsync(status, K.status, sizeof(status), cudaMemcpyDeviceToHost, C.stream));
      VL_CUDA(cudaStreamSynchronize(C.stream));
      if (status[1] != 0 || status[0] == 0) break;
      chunk = std::min(chunk * 2, 16);
    }
  });
  if (status[1] != 0) {
    double ev = 0;
    VL_CUDA(cudaMemcpy(&ev, K.errval, sizeof(double), cudaMemcpyDeviceToHost));
    char buf[200];
    snprintf(buf, sizeof(buf), "CG breakdown in column %d: curvature %.3e <= 0", status[2], ev);
    fail(kEBreakdown, buf);
  }
  if (out) {
    out->iters.assign(t, 0);
    out->converged.assign(t, 0);
    out->res.assign(t, 0.0);
    VL_CUDA(cudaMemcpyAsync(out->iters.data(), K.iters, sizeof(int) * t, cudaMemcpyDeviceToHost, C.stream));
    VL_CUDA(cudaMemcpyAsync(out->converged.data(), K.conv, sizeof(int) * t, cudaMemcpyDeviceToHost, C.stream));
    VL_CUDA(cudaMemcpyAsync(out->res.data(), K.res, sizeof(double) * t, cudaMemcpyDeviceToHost, C.stream));
    VL_CUDA(cudaStreamSynchronize(C.stream));
    int mx = 0;
    for (int c = 0; c < t; ++c) mx = std::max(mx, out->iters[c]);
    out->max_iters = mx;
    if (capture && mx > 0) {
      out->alpha.assign((size_t)mx * t, 0.0);
      out->beta.assign((size_t)mx * t, 0.0);
      VL_CUDA(cudaMemcpy(out->alpha.data(), K.ah, sizeof(double) * mx * t, cudaMemcpyDeviceToHost));
      VL_CUDA(cudaMemcpy(out->beta.data(), K.bh, sizeof(double) * mx * t, cudaMemcpyDeviceToHost));
    }
  }
}

namespace {
struct SumLogWBody {
  const double* W;
  template <int G, int NU, int U, int NR>
  VL_D void run(int64_t s, bool valid, int, int, double (&acc)[NR][NU * U]) const {
    if (valid) acc[0][0] += log(W[s]);
  }
};
struct CopySum1 {
  double* dst;
  VL_D void operator()(const double* sums, int) const {
    if (threadIdx.x == 0) dst[0] = sums[0];
  }
};
struct ProbeZLBody {  // Z = sqrt(1/W) o Gn + ZL ; (ZL already = L Gk)
  const double* W;
  const double* Gn;
  double* Z;
  int ld;
  template <int G, int NU, int U, int NR>
  VL_D void run(int64_t s, bool valid, int gl, int t, double (&)[NR][NU * U]) const {
    if (!valid) return;
    double g[NU * U], z[NU * U];
    load_row<G, NU, U>(Gn, ld, s, gl, t, g);
    load_row<G, NU, U>(Z, ld, s, gl, t, z);
    const double se = sqrt(1.0 / W[s]);
#pragma unroll
    for (int i = 0; i < NU * U; ++i) z[i] = se * g[i] + z[i];
    store_row<G, NU, U>(Z, ld, s, gl, t, z);
  }
};
struct DotZVBody {
  const double* Z;
  const double* V;
  int ld;
  template <int G, int NU, int U, int NR>
  VL_D void run(int64_t s, bool valid, int gl, int t, double (&acc)[NR][NU * U]) const {
    if (!valid) return;
    double a[NU * U], b[NU * U];
    load_row<G, NU, U>(Z, ld, s, gl, t, a);
    load_row<G, NU, U>(V, ld, s, gl, t, b);
#pragma unroll
    for (int i = 0; i < NU * U; ++i) acc[0][i] += a[i] * b[i];
  }
};
template <int NRv>
struct CopySumsL {
  double* dst;
  VL_D void operator()(const double* sums, int t) const {
    for (int i = threadIdx.x; i < NRv * t; i += blockDim.x) dst[i] = sums[i];
  }
};
}  // namespace

double lrac_sumlogW(Ctx& C, int64_t n, const double* W) {
  double* d = C.dev_scalars.as<double>();
  launch_rows<1, 1, 1, 1, 0>(C, n, 1, SumLogWBody{W}, CopySum1{d});
  double h;
  VL_CUDA(cudaMemcpyAsync(&h, d, sizeof(double), cudaMemcpyDeviceToHost, C.stream));
  VL_CUDA(cudaStreamSynchronize(C.stream));
  return h;
}

// Z = sqrt(e) o Gn + L Gk (preconditioners.py:204-207), V = P^-1 Z, w_c = z_c . v_c
void lrac_probes(Ctx& C, const LracPrec& Pr, int t, const double* Gn, const double* Gk, double* Z, double* V,
                 double* w_host) {
  const int64_t n = Pr.F->pat->n;
  const int k = Pr.LF->keff, kl = Pr.LF->k;
  ProfScope ps(C, "lrac_probes", 0.0);
  if (k > 0) {
    // Z (t x n, column-major) = Gk (t x k, column-major view of the k x t row-major draws) A (k x n)
    Gemm g;
    g.m = t; g.n = (int)n; g.k = k;
    g.A = Gk; g.lda = t;
    g.B = Pr.LF->L.as<double>(); g.ldb = kl;
    g.C = Z; g.ldc = t;
    dgemm(C, g);
  } else {
    VL_CUDA(cudaMemsetAsync(Z, 0, sizeof(double) * (size_t)n * t, C.stream));
  }
  double* sums = C.dev_scalars.as<double>();
  dispatch_cols(t, t, [&](auto g, auto nu, auto uu) {
    constexpr int G = decltype(g)::value, NU = decltype(nu)::value, U = decltype(uu)::value;
    launch_rows<G, NU, U, 0, 0>(C, n, t, ProbeZLBody{Pr.W, Gn, Z, t}, Fin0<0>{});
  });
  lrac_apply_inv(C, Pr, t, Z, V);
  dispatch_cols(t, t, [&](auto g, auto nu, auto uu) {
    constexpr int G = decltype(g)::value, NU = decltype(nu)::value, U = decltype(uu)::value;
    launch_rows<G, NU, U, 1, 0>(C, n, t, DotZVBody{Z, V, t}, CopySumsL<1>{sums});
  });
  VL_CUDA(cudaMemcpyAsync(w_host, sums, sizeof(double) * t, cudaMemcpyDeviceToHost, C.stream));
  VL_CUDA(cudaStreamSynchronize(C.stream));
}

// ---------------------------------------------------------------------------
// Gradient pieces (laplace.py:369-386 _lrac_dL, 421-431 LRAC mu-derivative,
// 527-533 LRAC dP_trace / dP_op, eq7 dA_op = -SigmaTilde dQ SigmaTilde)
// ---------------------------------------------------------------------------
namespace {

__global__ void colnorm2_kernel(int64_t n, int k, int ldk, const double* __restrict__ Y, double* __restrict__ g2) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const double* c = Y + i * ldk;
    double s = 0.0;
    for (int l = 0; l < k; ++l) s += c[l] * c[l];
    g2[i] = s;
  }
}

// dS[i][q] = d Sigma(x_i, x_piv_q) / d rho   (n x k row-major, lda kl)
__global__ void dsigma_kernel(int64_t n, int dim, int k, int kl, const double* __restrict__ xy,
                              const int32_t* __restrict__ piv_s, MaternK K, double* __restrict__ dS) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n * k; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = e / k;
    const int q = (int)(e % k);
    const int64_t p = piv_s[q];
    double r2 = 0.0;
    for (int a = 0; a < dim; ++a) {
      const double df = xy[i * dim + a] - xy[p * dim + a];
      r2 += df * df;
    }
    const double r = sqrt(r2);
    double v;
    if (K.nu == 0) {
      const double u = r / K.rho;
      v = K.s2 * exp(-u) * u / K.rho;
    } else {
      const double u = K.c * r;
      v = (K.nu == 1) ? K.s2 * u * u * exp(-u) / K.rho : K.s2 * u * u * (1.0 + u) * exp(-u) / (3.0 * K.rho);
    }
    dS[i * kl + q] = v;
  }
}

// rows at the pivots: out (k x k, column-major, ld k): out[a + b*k] = src[piv_a][b]
__global__ void gather_piv_rows_kernel(int k, int kl, const int32_t* __restrict__ piv_s, const double* __restrict__ src,
                                       double* __restrict__ out) {
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < k * k; e += gridDim.x * blockDim.x) {
    const int a = e % k, b = e / k;
    out[a + (size_t)b * k] = src[(int64_t)piv_s[a] * kl + b];
  }
}

// Phi = tril(X, -1) + 0.5 diag(X) in place (column-major)
__global__ void phi_kernel(int k, double* X) {
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < k * k; e += gridDim.x * blockDim.x) {
    const int a = e % k, b = e / k;
    if (a < b) X[e] = 0.0;
    else if (a == b) X[e] *= 0.5;
  }
}

__global__ void diag_sum_kernel(int k, const double* __restrict__ A, double* out) {
  __shared__ double sh[256];
  double s = 0.0;
  for (int i = threadIdx.x; i < k; i += blockDim.x) s += A[(size_t)i * k + i];
  sh[threadIdx.x] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double a = 0.0;
    for (int i = 0; i < (int)blockDim.x; ++i) a += sh[i];
    *out = a;
  }
}

template <int G>
VL_D double gsum_l(double v) {
#pragma unroll
  for (int o = 1; o < G; o <<= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// LRAC mu-derivative (laplace.py:421-431): H = U V / W^2, R = (V/W)^2, per-row
// control variate c; s = 0.5 md3 (1/W + c (G2 - 1/W) - mean(H - c R)).
// Column sums for the xi STE: h_xi = -sum m3/W^2 U V, r_xi = -sum m3/W^2 V^2.
template <bool XI>
struct LracMuBody {
  const double* U_;
  const double* V_;
  const double* W;
  const double* G2;
  const double* d3;
  const double* md3x;
  double* s_out;
  int ld;
  int plain;  // no control variate (l2, laplace.py:433-434)
  template <int G, int NU, int U, int NR>
  VL_D void run(int64_t s, bool valid, int gl, int t, double (&acc)[NR][NU * U]) const {
    constexpr int NC = NU * U;
    double us[NC], vs[NC], H[NC], R[NC];
    load_row<G, NU, U>(U_, ld, valid ? s : 0, gl, valid ? t : 0, us);
    load_row<G, NU, U>(V_, ld, valid ? s : 0, gl, valid ? t : 0, vs);
    const double w = valid ? W[s] : 1.0;
    double sh = 0.0, sr = 0.0;
#pragma unroll
    for (int i = 0; i < NC; ++i) {
      const int c = vl::Cols<G, NU, U>::col(gl, i);
      const bool on = valid && c < t;
      H[i] = on ? us[i] * vs[i] / (w * w) : 0.0;
      const double vw = vs[i] / w;
      R[i] = on ? vw * vw : 0.0;
      sh += H[i];
      sr += R[i];
    }
    sh = gsum_l<G>(sh);
    sr = gsum_l<G>(sr);
    const double hm = sh / t, rm = sr / t;
    double svr = 0.0, scv = 0.0;
#pragma unroll
    for (int i = 0; i < NC; ++i) {
      const int c = vl::Cols<G, NU, U>::col(gl, i);
      if (valid && c < t) {
        svr += (R[i] - rm) * (R[i] - rm);
        scv += (H[i] - hm) * (R[i] - rm);
      }
    }
    svr = gsum_l<G>(svr);
    scv = gsum_l<G>(scv);
    double cw = 0.0;
    if (t >= 2 && !plain) {
      const double vr = svr / (t - 1), cv = scv / (t - 1);
      cw = (vr >= 1e-300) ? cv / vr : 0.0;
    }
    double sm = 0.0;
#pragma unroll
    for (int i = 0; i < NC; ++i) {
      const int c = vl::Cols<G, NU, U>::col(gl, i);
      if (valid && c < t) sm += H[i] - cw * R[i];
    }
    sm = gsum_l<G>(sm);
    if (!valid) return;
    if (gl == 0) {
      const double exact = 1.0 / w + cw * (G2[s] - 1.0 / w);
      s_out[s] = 0.5 * ((-d3[s]) * (exact - sm / t));
    }
    if constexpr (XI) {
      const double q = md3x[s] / (w * w);
#pragma unroll
      for (int i = 0; i < NC; ++i) {
        const int c = vl::Cols<G, NU, U>::col(gl, i);
        if (c >= t) continue;
        acc[0][i] += -(q * us[i] * vs[i]);
        acc[1][i] += -(q * vs[i] * vs[i]);
      }
    }
  }
};

// h_k = -(SigmaTilde u)^T dQ_k (SigmaTilde v): forward-only dQ dot with
// U' = SigmaTilde U, V' = SigmaTilde V (columns: h_sigma2, h_rho)
struct DQDotBody {
  BView B;
  const double* dval;
  const double* U_;
  const double* V_;
  const double* D;
  const double* dDs;
  const double* dDr;
  int ld;
  template <int G, int NU, int U, int NR>
  VL_D void run(int64_t s, bool valid, int gl, int t, double (&acc)[NR][NU * U]) const {
    constexpr int NC = NU * U;
    double BU[NC], BV[NC], dBU[NC], dBV[NC], us[NC], vs[NC];
    zero(BU);
    zero(BV);
    zero(dBU);
    zero(dBV);
    gather_B<G, NU, U>(B, B.val, s, valid, gl, t, LoadU<U>{U_, ld}, BU);
    gather_B<G, NU, U>(B, B.val, s, valid, gl, t, LoadU<U>{V_, ld}, BV);
    gather_B<G, NU, U>(B, dval, s, valid, gl, t, LoadU<U>{U_, ld}, dBU);
    gather_B<G, NU, U>(B, dval, s, valid, gl, t, LoadU<U>{V_, ld}, dBV);
    if (!valid) return;
    load_row<G, NU, U>(U_, ld, s, gl, t, us);
    load_row<G, NU, U>(V_, ld, s, gl, t, vs);
#pragma unroll
    for (int i = 0; i < NC; ++i) {
      BU[i] += us[i];
      BV[i] += vs[i];
    }
    const double Dinv = 1.0 / D[s];
    const double qs = dDs[s] * Dinv * Dinv, qr = dDr[s] * Dinv * Dinv;
#pragma unroll
    for (int i = 0; i < NC; ++i) {
      const int c = vl::Cols<G, NU, U>::col(gl, i);
      if (c >= t) continue;
      acc[0][i] += (BU[i] * qs * BV[i]);  // -(-qs ...) : h = -(u'^T dQ v')
      acc[1][i] += -((dBU[i] * BV[i] + BU[i] * dBV[i]) * Dinv - BU[i] * qr * BV[i]);
    }
  }
};

// Probe-sharded LRAC mu-derivative (multi-GPU; the per-row control variate
// needs all t probes), mirroring the VADU split of laplace.cu:
//   MODE 1: rowA = [sum_c H, sum_c R] over the local columns (+ xi column sums)
//   MODE 2: rowB = [sum_c (H - hbar)(R - rbar), sum_c (R - rbar)^2], global means rowA / tg
template <int MODE, bool XI>
struct LracMuSplitBody {
  const double* U_;
  const double* V_;
  const double* W;
  const double* md3x;
  double* rowA;
  double* rowB;
  int tg;
  int ld;
  template <int G, int NU, int U, int NR>
  VL_D void run(int64_t s, bool valid, int gl, int t, double (&acc)[NR][NU * U]) const {
    constexpr int NC = NU * U;
    double us[NC], vs[NC], H[NC], R[NC];
    load_row<G, NU, U>(U_, ld, valid ? s : 0, gl, valid ? t : 0, us);
    load_row<G, NU, U>(V_, ld, valid ? s : 0, gl, valid ? t : 0, vs);
    const double w = valid ? W[s] : 1.0;
#pragma unroll
    for (int i = 0; i < NC; ++i) {
      const int c = vl::Cols<G, NU, U>::col(gl, i);
      const bool on = valid && c < t;
      H[i] = on ? us[i] * vs[i] / (w * w) : 0.0;
      const double vw = vs[i] / w;
      R[i] = on ? vw * vw : 0.0;
    }
    if constexpr (MODE == 1) {
      double sh = 0.0, sr = 0.0;
#pragma unroll
      for (int i = 0; i < NC; ++i) {
        sh += H[i];
        sr += R[i];
      }
      sh = gsum_l<G>(sh);
      sr = gsum_l<G>(sr);
      if (valid && gl == 0) {
        rowA[2 * s] = sh;
        rowA[2 * s + 1] = sr;
      }
      if constexpr (XI) {
        if (!valid) return;
        const double q = md3x[s] / (w * w);
#pragma unroll
        for (int i = 0; i < NC; ++i) {
          const int c = vl::Cols<G, NU, U>::col(gl, i);
          if (c >= t) continue;
          acc[0][i] += -(q * us[i] * vs[i]);
          acc[1][i] += -(q * vs[i] * vs[i]);
        }
      }
    } else {
      const double hm = valid ? rowA[2 * s] / tg : 0.0, rm = valid ? rowA[2 * s + 1] / tg : 0.0;
      double svr = 0.0, scv = 0.0;
#pragma unroll
      for (int i = 0; i < NC; ++i) {
        const int c = vl::Cols<G, NU, U>::col(gl, i);
        if (valid && c < t) {
          svr += (R[i] - rm) * (R[i] - rm);
          scv += (H[i] - hm) * (R[i] - rm);
        }
      }
      svr = gsum_l<G>(svr);
      scv = gsum_l<G>(scv);
      if (valid && gl == 0) {
        rowB[2 * s] = scv;
        rowB[2 * s + 1] = svr;
      }
    }
  }
};

// MODE 3 of the split: s = 0.5 (-d3) (1/W + c (G2 - 1/W) - mean(H - c R)) from the reduced row sums
struct LracMuFinishBody {
  const double* rowA;
  const double* rowB;
  const double* G2;
  const double* W;
  const double* d3;
  double* s_out;
  int tg;
  int plain;
  template <int G, int NU, int U, int NR>
  VL_D void run(int64_t s, bool valid, int, int, double (&)[NR][NU * U]) const {
    if (!valid) return;
    double cw = 0.0;
    if (tg >= 2 && !plain) {
      const double vr = rowB[2 * s + 1] / (tg - 1), cv = rowB[2 * s] / (tg - 1);
      cw = (vr >= 1e-300) ? cv / vr : 0.0;
    }
    const double w = W[s];
    const double exact = 1.0 / w + cw * (G2[s] - 1.0 / w);
    s_out[s] = 0.5 * ((-d3[s]) * (exact - (rowA[2 * s] - cw * rowA[2 * s + 1]) / tg));
  }
};

// [sum G2 m3, sum m3 / W] (the xi dP_trace pieces) as a device reduction
struct XiSumsBody {
  const double* G2;
  const double* m3;
  const double* W;
  template <int G, int NU, int U, int NR>
  VL_D void run(int64_t s, bool valid, int, int, double (&acc)[NR][NU * U]) const {
    if (!valid) return;
    acc[0][0] += G2[s] * m3[s];
    acc[1][0] += m3[s] / W[s];
  }
};

}  // namespace

// out: s (n, device); hcols (2 x t: h_s2, h_rho), rcols (2 x t: r_s2, r_rho),
// dPt (2); with md3x: xih (t), xir (t), xi_scalars [sum G2 m3, sum m3 / W]
namespace {
// G2 = diag(L M^-1 L^T) = column norms of Lm^-1 L^T (zero without a low-rank part)
void lrac_G2(Ctx& C, const LracPrec& Pr, DevBuf& G2) {
  const int64_t n = Pr.F->pat->n;
  const int k = Pr.LF->keff, kl = Pr.LF->k;
  DevBuf Y;
  // G2 = diag(L M^-1 L^T) = column norms of Lm^-1 L^T
  Y.alloc(sizeof(double) * (size_t)n * kl);
  G2.alloc(sizeof(double) * n);
  if (k > 0) {
    Gemm g;  // Y (k x n, ld kl) = Lm^-1 A, A = L^T viewed column-major
    g.m = k; g.n = (int)n; g.k = k;
    g.A = Pr.Lmi.as<double>(); g.lda = k;
    g.B = Pr.LF->L.as<double>(); g.ldb = kl;
    g.C = Y.as<double>(); g.ldc = kl;
    dgemm(C, g);
    colnorm2_kernel<<<C.num_sms * 4, 256, 0, C.stream>>>(n, k, kl, Y.as<double>(), G2.as<double>());
  } else {
    VL_CUDA(cudaMemsetAsync(G2.p, 0, sizeof(double) * n, C.stream));
  }
}

// The per-probe-column and scalar parts of the LRAC gradient (everything except
// the mu-derivative): h (sigma2, rho) through SigmaTilde U / V and the dQ dot,
// r = 2 (L^T v).(dL^T v), dP_trace, and the xi scalars.
void lrac_grad_columns(Ctx& C, const LracPrec& Pr, int t, const double* U, const double* V, const double* md3x,
                       const DevBuf& G2, double* hcols, double* rcols, double* dPt, double* xis) {
  const Factor& F = *Pr.F;
  const Pattern& P = *F.pat;
  const int64_t n = P.n;
  const int k = Pr.LF->keff, kl = Pr.LF->k;
  double* sums = C.dev_scalars.as<double>();
  // h via SigmaTilde U, SigmaTilde V and the forward-only dQ dot
  DevBuf SU, SV, scr;
  SU.alloc(sizeof(double) * (size_t)n * t);
  SV.alloc(sizeof(double) * (size_t)n * t);
  scr.alloc(sizeof(double) * (size_t)n * t);
  apply_sigma_tilde(C, F, t, U, SU.as<double>(), scr.as<double>());
  apply_sigma_tilde(C, F, t, V, SV.as<double>(), scr.as<double>());
  BView Bv = bview(F, false);
  dispatch_cols(t, t, [&](auto g, auto nu, auto uu) {
    constexpr int G_ = decltype(g)::value, NU = decltype(nu)::value, U_ = decltype(uu)::value;
    launch_rows<G_, NU, U_, 2, 0>(C, n, t,
                                  DQDotBody{Bv, F.dval.as<double>(), SU.as<double>(), SV.as<double>(), F.D.as<double>(),
                                            F.dD_sig.as<double>(), F.dD_rho.as<double>(), t},
                                  CopySumsL<2>{sums});
  });
  VL_CUDA(cudaMemcpyAsync(hcols, sums, sizeof(double) * 2 * t, cudaMemcpyDeviceToHost, C.stream));
  VL_CUDA(cudaStreamSynchronize(C.stream));
  if (md3x && xis) {
    // xi dP_trace pieces: sum G2 m3, sum m3 / W (device reduction)
    launch_rows<1, 1, 1, 2, 0>(C, n, 1, XiSumsBody{G2.as<double>(), md3x, Pr.Wop}, CopySumsL<2>{sums});
    VL_CUDA(cudaMemcpyAsync(xis, sums, sizeof(double) * 2, cudaMemcpyDeviceToHost, C.stream));
    VL_CUDA(cudaStreamSynchronize(C.stream));
  }
  if (k == 0) {
    for (int i = 0; i < 2 * t; ++i) rcols[i] = 0.0;
    dPt[0] = dPt[1] = 0.0;
    return;
  }
  // dense chain on the hand-written GEMM (dense.cu); triangular solves as products with inverses
  auto gemm = [&](bool ta, bool tb, int m_, int n_, int k_, double alpha, const double* A_, int lda_, const double* B_,
                  int ldb_, double beta, double* C_, int ldc_, const double* kw = nullptr) {
    Gemm g;
    g.ta = ta; g.tb = tb; g.m = m_; g.n = n_; g.k = k_; g.alpha = alpha; g.beta = beta;
    g.A = A_; g.lda = lda_; g.B = B_; g.ldb = ldb_; g.C = C_; g.ldc = ldc_; g.kw = kw;
    dgemm(C, g);
  };
  const double* Lp = Pr.LF->L.as<double>();  // column-major (kl x n) view of L^T
  // A1 = L^T V (k x t)
  DevBuf A1, A2, tr;
  A1.alloc(sizeof(double) * (size_t)k * t);
  A2.alloc(sizeof(double) * (size_t)k * t);
  tr.alloc(64);
  gemm(false, true, k, t, (int)n, 1.0, Lp, kl, V, t, 0.0, A1.as<double>(), k);
  std::vector<double> a1((size_t)k * t), a2((size_t)k * t);
  VL_CUDA(cudaMemcpyAsync(a1.data(), A1.p, sizeof(double) * a1.size(), cudaMemcpyDeviceToHost, C.stream));
  // --- sigma2: dL = L / (2 sigma2): r = 2 (L^T v).(dL^T v) = (L^T v)^2 / sigma2 ;
  //     dPt = 2 tr(M^-1 L^T W L) / (2 sigma2) = (k - tr M^-1) / sigma2
  const double* Minv = Pr.Minv.as<double>();
  diag_sum_kernel<<<1, 256, 0, C.stream>>>(k, Minv, tr.as<double>());
  double trMinv = 0.0;
  VL_CUDA(cudaMemcpyAsync(&trMinv, tr.p, sizeof(double), cudaMemcpyDeviceToHost, C.stream));
  VL_CUDA(cudaStreamSynchronize(C.stream));
  for (int c = 0; c < t; ++c) {
    double s = 0.0;
    for (int l = 0; l < k; ++l) s += a1[(size_t)c * k + l] * a1[(size_t)c * k + l];
    rcols[c] = s / Pr.F->sigma2;
  }
  dPt[0] = ((double)k - trMinv) / Pr.F->sigma2;
  // --- rho: dL = (dS - L dR^T) R^-T, dR = R Phi(R^-1 dS_pp R^-T), R = L[piv]
  const MaternK Km = make_matern(F);
  DevBuf dS, dL, R, Ri, X, X1, dR;
  dS.alloc(sizeof(double) * (size_t)n * kl);
  dL.alloc(sizeof(double) * (size_t)n * kl);
  R.alloc(sizeof(double) * (size_t)k * k);
  Ri.alloc(sizeof(double) * (size_t)k * k);
  X.alloc(sizeof(double) * (size_t)k * k);
  X1.alloc(sizeof(double) * (size_t)k * k);
  dR.alloc(sizeof(double) * (size_t)k * k);
  dsigma_kernel<<<C.num_sms * 8, 256, 0, C.stream>>>(n, P.d, k, kl, P.xy.as<double>(), Pr.LF->piv_s.as<int32_t>(), Km,
                                                     dS.as<double>());
  gather_piv_rows_kernel<<<64, 256, 0, C.stream>>>(k, kl, Pr.LF->piv_s.as<int32_t>(), Lp, R.as<double>());
  gather_piv_rows_kernel<<<64, 256, 0, C.stream>>>(k, kl, Pr.LF->piv_s.as<int32_t>(), dS.as<double>(), X.as<double>());
  VL_LAUNCH_CHECK();
  dtrtri_lower(C, k, R.as<double>(), k, Ri.as<double>(), k);
  // X = R^-1 dS_pp R^-T, then Phi(X) in place
  gemm(false, false, k, k, k, 1.0, Ri.as<double>(), k, X.as<double>(), k, 0.0, X1.as<double>(), k);
  gemm(false, true, k, k, k, 1.0, X1.as<double>(), k, Ri.as<double>(), k, 0.0, X.as<double>(), k);
  phi_kernel<<<64, 256, 0, C.stream>>>(k, X.as<double>());
  VL_LAUNCH_CHECK();
  // dR = R Phi
  gemm(false, false, k, k, k, 1.0, R.as<double>(), k, X.as<double>(), k, 0.0, dR.as<double>(), k);
  // dL^T (k x n view, ld kl) = R^-1 (dS^T - dR L^T)
  gemm(false, false, k, (int)n, k, -1.0, dR.as<double>(), k, Lp, kl, 1.0, dS.as<double>(), kl);
  gemm(false, false, k, (int)n, k, 1.0, Ri.as<double>(), k, dS.as<double>(), kl, 0.0, dL.as<double>(), kl);
  // A2 = dL^T V
  gemm(false, true, k, t, (int)n, 1.0, dL.as<double>(), kl, V, t, 0.0, A2.as<double>(), k);
  // T1 = L^T diag(W) dL (k x k), MT = M^-1 T1 -> tr(M^-1 T1)
  DevBuf T1, MT;
  T1.alloc(sizeof(double) * (size_t)k * k);
  MT.alloc(sizeof(double) * (size_t)k * k);
  gemm(false, true, k, k, (int)n, 1.0, Lp, kl, dL.as<double>(), kl, 0.0, T1.as<double>(), k, Pr.W);
  gemm(false, false, k, k, k, 1.0, Minv, k, T1.as<double>(), k, 0.0, MT.as<double>(), k);
  diag_sum_kernel<<<1, 256, 0, C.stream>>>(k, MT.as<double>(), tr.as<double>());
  double trMT = 0.0;
  VL_CUDA(cudaMemcpyAsync(&trMT, tr.p, sizeof(double), cudaMemcpyDeviceToHost, C.stream));
  VL_CUDA(cudaMemcpyAsync(a2.data(), A2.p, sizeof(double) * a2.size(), cudaMemcpyDeviceToHost, C.stream));
  VL_CUDA(cudaStreamSynchronize(C.stream));
  dPt[1] = 2.0 * trMT;
  for (int c = 0; c < t; ++c) {
    double s = 0.0;
    for (int l = 0; l < k; ++l) s += a1[(size_t)c * k + l] * a2[(size_t)c * k + l];
    rcols[t + c] = 2.0 * s;
  }
}
}  // namespace

// out: s (n, device); hcols (2 x t: h_s2, h_rho), rcols (2 x t: r_s2, r_rho),
// dPt (2); with md3x: xih (t), xir (t), xi_scalars [sum G2 m3, sum m3 / W]
void lrac_grad(Ctx& C, const LracPrec& Pr, int t, const double* U, const double* V, const double* d3,
               const double* md3x, double* s_out, double* hcols, double* rcols, double* dPt, double* xicols,
               double* xis, int plain) {
  const Factor& F = *Pr.F;
  const int64_t n = F.pat->n;
  if (!F.has_grad) fail(kEConfig, "factor was built without gradient");
  ProfScope ps(C, "lrac_grad", 0.0);
  DevBuf G2;
  lrac_G2(C, Pr, G2);
  double* sums = C.dev_scalars.as<double>();
  dispatch_cols(t, t, [&](auto g, auto nu, auto uu) {
    constexpr int G_ = decltype(g)::value, NU = decltype(nu)::value, U_ = decltype(uu)::value;
    if (md3x)
      launch_rows<G_, NU, U_, 2, 0>(C, n, t, LracMuBody<true>{U, V, Pr.Wop, G2.as<double>(), d3, md3x, s_out, t, plain},
                                    CopySumsL<2>{sums});
    else
      launch_rows<G_, NU, U_, 0, 0>(C, n, t, LracMuBody<false>{U, V, Pr.Wop, G2.as<double>(), d3, nullptr, s_out, t,
                                                               plain},
                                    Fin0<0>{});
  });
  if (md3x) {
    VL_CUDA(cudaMemcpyAsync(xicols, sums, sizeof(double) * 2 * t, cudaMemcpyDeviceToHost, C.stream));
    VL_CUDA(cudaStreamSynchronize(C.stream));
  }
  lrac_grad_columns(C, Pr, t, U, V, md3x, G2, hcols, rcols, dPt, xis);
}

void lrac_grad_split(Ctx& C, const LracPrec& Pr, int mode, int t, int t_glob, const double* U, const double* V,
                     const double* d3, const double* md3x, double* rowA, double* rowB, double* s_out, double* hcols,
                     double* rcols, double* dPt, double* xicols, double* xis, int plain) {
  const Factor& F = *Pr.F;
  const int64_t n = F.pat->n;
  if (!F.has_grad) fail(kEConfig, "factor was built without gradient");
  ProfScope ps(C, "lrac_grad_split", 0.0);
  double* sums = C.dev_scalars.as<double>();
  if (mode == 3) {
    DevBuf G2;
    lrac_G2(C, Pr, G2);
    launch_rows<1, 1, 1, 0, 0>(C, n, 1, LracMuFinishBody{rowA, rowB, G2.as<double>(), Pr.Wop, d3, s_out, t_glob, plain},
                               Fin0<0>{});
    return;
  }
  if (t < 1 || 2 * t > 8192) fail(kECapacity, "invalid probe shard width");
  if (mode == 2) {
    dispatch_cols(t, t, [&](auto g, auto nu, auto uu) {
      constexpr int G_ = decltype(g)::value, NU = decltype(nu)::value, U_ = decltype(uu)::value;
      launch_rows<G_, NU, U_, 0, 0>(C, n, t, LracMuSplitBody<2, false>{U, V, Pr.Wop, nullptr, rowA, rowB, t_glob, t},
                                    Fin0<0>{});
    });
    return;
  }
  if (mode != 1) fail(kEConfig, "unknown split mode");
  DevBuf G2;
  lrac_G2(C, Pr, G2);
  dispatch_cols(t, t, [&](auto g, auto nu, auto uu) {
    constexpr int G_ = decltype(g)::value, NU = decltype(nu)::value, U_ = decltype(uu)::value;
    if (md3x)
      launch_rows<G_, NU, U_, 2, 0>(C, n, t, LracMuSplitBody<1, true>{U, V, Pr.Wop, md3x, rowA, rowB, t_glob, t},
                                    CopySumsL<2>{sums});
    else
      launch_rows<G_, NU, U_, 0, 0>(C, n, t, LracMuSplitBody<1, false>{U, V, Pr.Wop, nullptr, rowA, rowB, t_glob, t},
                                    Fin0<0>{});
  });
  if (md3x) {
    VL_CUDA(cudaMemcpyAsync(xicols, sums, sizeof(double) * 2 * t, cudaMemcpyDeviceToHost, C.stream));
    VL_CUDA(cudaStreamSynchronize(C.stream));
  }
  lrac_grad_columns(C, Pr, t, U, V, md3x, G2, hcols, rcols, dPt, xis);
}

void lrac_solve_system(Ctx& C, const LracPrec& Pr, int t, const double* rhs, double* u, double tol, int max_iter,
                       PcgResult* out) {
  const int64_t n = Pr.F->pat->n;
  DevBuf srhs, scr, us;
  srhs.alloc(sizeof(double) * (size_t)n * t);
  scr.alloc(sizeof(double) * (size_t)n * t);
  us.alloc(sizeof(double) * (size_t)n * t);
  if (Pr.eq6) {  // laplace.py:180-181
    pcg_lrac(C, Pr, t, rhs, u, tol, max_iter, false, out);
    return;
  }
  apply_sigma_tilde(C, *Pr.F, t, rhs, srhs.as<double>(), scr.as<double>());
  pcg_lrac(C, Pr, t, srhs.as<double>(), us.as<double>(), tol, max_iter, false, out);
  dispatch_cols(t, t, [&](auto g, auto nu, auto uu) {
    constexpr int G = decltype(g)::value, NU = decltype(nu)::value, U = decltype(uu)::value;
    launch_rows<G, NU, U, 0, 0>(C, n, t, DivWBody{Pr.Wop, us.as<double>(), u, t}, Fin0<0>{});
  });
}


// ---------------------------------------------------------------------------
// Other low-rank-plus-diagonal preconditioners (preconditioners.py:161-246,
// 323-387) and diag(SigmaTilde) for l2 (vecchia.py:198-212).
// ---------------------------------------------------------------------------
namespace {

// Column p of Q = B^T D^-1 B into the dense vector qc (sequential, fixed order):
// Q[i, p] = sum over rows r with B_rp != 0 (r = p and the children of p) of B_ri B_rp / D_r.
__global__ void qcol_kernel(const int32_t* __restrict__ nbr, const int32_t* __restrict__ cnt,
                            const double* __restrict__ val, const int32_t* __restrict__ tptr,
                            const int32_t* __restrict__ tidx, const double* __restrict__ valT,
                            const double* __restrict__ D, int m, PcState st, double* __restrict__ qc,
                            int32_t* __restrict__ touched, int* __restrict__ ntouched) {
  if (threadIdx.x != 0 || ((volatile int*)st.i)[1] != 0) return;
  const int32_t p = st.i[0];
  int nt = 0;
  auto add_row = [&](int32_t r, double brp) {
    const double w = brp / D[r];
    qc[r] += w;  // B_rr = 1
    touched[nt++] = r;
    for (int e = 0; e < cnt[r]; ++e) {
      const int32_t i = nbr[(int64_t)r * m + e];
      qc[i] += val[(int64_t)r * m + e] * w;
      touched[nt++] = i;
    }
  };
  add_row(p, 1.0);
  for (int32_t e = tptr[p]; e < tptr[p + 1]; ++e) add_row(tidx[e], valT[e]);
  *ntouched = nt;
}

__global__ void qclear_kernel(double* __restrict__ qc, const int32_t* __restrict__ touched,
                              const int* __restrict__ ntouched) {
  const int nt = *ntouched;
  for (int e = threadIdx.x; e < nt; e += blockDim.x) qc[touched[e]] = 0.0;
}

struct DiagQBody {  // diag(B^T D^-1 B)
  BView B;
  const double* D;
  double* out;
  template <int G, int NU, int U, int NR>
  VL_D void run(int64_t s, bool valid, int, int, double (&)[NR][NU * U]) const {
    if (!valid) return;
    double q = 1.0 / D[s];
    for (int32_t e = B.tptr[s]; e < B.tptr[s + 1]; ++e) q += B.valT[e] * B.valT[e] / D[B.tidx[e]];
    out[s] = q;
  }
};

struct RowScoreBody {  // (1 + sum_e B_se^2) / D_s
  BView B;
  const double* D;
  double* out;
  template <int G, int NU, int U, int NR>
  VL_D void run(int64_t s, bool valid, int, int, double (&)[NR][NU * U]) const {
    if (!valid) return;
    double q = 1.0;
    for (int e = 0; e < B.cnt[s]; ++e) {
      const double b = B.val[s * B.m + e];
      q += b * b;
    }
    out[s] = q / D[s];
  }
};

// U[:, c] = B_{r_c,:}^T / sqrt(D_{r_c}) into the dense n x kl row-major factor
__global__ void rowsel_scatter_kernel(int k, int kl, int m, const int32_t* __restrict__ rows,
                                      const int32_t* __restrict__ nbr, const int32_t* __restrict__ cnt,
                                      const double* __restrict__ val, const double* __restrict__ D,
                                      double* __restrict__ L) {
  for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < k; c += gridDim.x * blockDim.x) {
    const int32_t r = rows[c];
    const double f = 1.0 / sqrt(D[r]);
    L[(int64_t)r * kl + c] = f;
    for (int e = 0; e < cnt[r]; ++e) L[(int64_t)nbr[(int64_t)r * m + e] * kl + c] = val[(int64_t)r * m + e] * f;
  }
}

__global__ void eye_block_kernel(int64_t n, int a, int w, double* __restrict__ E) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n * w; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = e / w;
    const int c = (int)(e % w);
    E[e] = (i == a + c) ? 1.0 : 0.0;
  }
}

struct DX2Body {  // acc[c] += D_s X_sc^2
  const double* D;
  const double* X;
  int ld;
  template <int G, int NU, int U, int NR>
  VL_D void run(int64_t s, bool valid, int gl, int t, double (&acc)[NR][NU * U]) const {
    if (!valid) return;
    double a[NU * U];
    load_row<G, NU, U>(X, ld, s, gl, t, a);
    const double ds = D[s];
#pragma unroll
    for (int i = 0; i < NU * U; ++i) acc[0][i] += ds * a[i] * a[i];
  }
};

}  // namespace

namespace {
// Deterministic device argmax over storage rows: largest v[s], ties to the
// lowest factor index fidx[s] (the reference's argmax / lexsort tie rule);
// pass 1 per block, pass 2 one block over the block winners.
constexpr int kAmThreads = 256;
VL_D bool am_better(double va, int32_t fa, double vb, int32_t fb) { return va > vb || (va == vb && fa < fb); }

__global__ void __launch_bounds__(kAmThreads) argmax_pass1(int64_t n, const double* __restrict__ v,
                                                           const int32_t* __restrict__ fidx, double* __restrict__ bv,
                                                           int32_t* __restrict__ bsr) {
  __shared__ double sv[kAmThreads];
  __shared__ int32_t sf[kAmThreads], ss[kAmThreads];
  double best = -INFINITY;
  int32_t bf = INT32_MAX, bs = -1;
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n; r += (int64_t)gridDim.x * blockDim.x) {
    const double x = v[r];
    const int32_t f = fidx[r];
    if (bs < 0 || am_better(x, f, best, bf)) { best = x; bf = f; bs = (int32_t)r; }
  }
  sv[threadIdx.x] = best; sf[threadIdx.x] = bf; ss[threadIdx.x] = bs;
  __syncthreads();
  for (int o = kAmThreads / 2; o > 0; o >>= 1) {
    if (threadIdx.x < o) {
      const int q = threadIdx.x + o;
      if (ss[q] >= 0 && (ss[threadIdx.x] < 0 || am_better(sv[q], sf[q], sv[threadIdx.x], sf[threadIdx.x]))) {
        sv[threadIdx.x] = sv[q]; sf[threadIdx.x] = sf[q]; ss[threadIdx.x] = ss[q];
      }
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) { bv[blockIdx.x] = sv[0]; bsr[blockIdx.x] = ss[0]; }
}

// pass 2: winner -> out_s / out_v (pivoted-Cholesky state: i[0] = row, i[1..3] = 0);
// with knock_out, v[winner] = -inf (the next round of a top-k selection)
__global__ void __launch_bounds__(kAmThreads) argmax_pass2(int nb, const double* __restrict__ bv,
                                                           const int32_t* __restrict__ bsr,
                                                           const int32_t* __restrict__ fidx, int* out_i,
                                                           double* out_v, int32_t* sel_f, int32_t* sel_s, int slot,
                                                           double* knock_out) {
  __shared__ double sv[kAmThreads];
  __shared__ int32_t sf[kAmThreads], ss[kAmThreads];
  double best = -INFINITY;
  int32_t bf = INT32_MAX, bs = -1;
  for (int b = threadIdx.x; b < nb; b += blockDim.x) {
    const int32_t r = bsr[b];
    if (r < 0) continue;
    const int32_t f = fidx[r];
    if (bs < 0 || am_better(bv[b], f, best, bf)) { best = bv[b]; bf = f; bs = r; }
  }
  sv[threadIdx.x] = best; sf[threadIdx.x] = bf; ss[threadIdx.x] = bs;
  __syncthreads();
  for (int o = kAmThreads / 2; o > 0; o >>= 1) {
    if (threadIdx.x < o) {
      const int q = threadIdx.x + o;
      if (ss[q] >= 0 && (ss[threadIdx.x] < 0 || am_better(sv[q], sf[q], sv[threadIdx.x], sf[threadIdx.x]))) {
        sv[threadIdx.x] = sv[q]; sf[threadIdx.x] = sf[q]; ss[threadIdx.x] = ss[q];
      }
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    if (out_i) { out_i[0] = ss[0]; out_i[1] = out_i[2] = out_i[3] = 0; }
    if (out_v) *out_v = sv[0];
    if (sel_f) { sel_f[slot] = sf[0]; sel_s[slot] = ss[0]; }
    if (knock_out && ss[0] >= 0) knock_out[ss[0]] = -INFINITY;
  }
}

void device_argmax(Ctx& C, int64_t n, double* v, const int32_t* fidx, DevBuf& scratch, int* out_i, double* out_v,
                   int32_t* sel_f, int32_t* sel_s, int slot, bool knock_out) {
  const int nb = (int)std::max<int64_t>(1, std::min<int64_t>(4LL * C.num_sms, (n + kAmThreads - 1) / kAmThreads));
  scratch.alloc((sizeof(double) + sizeof(int32_t)) * nb);
  double* bv = scratch.as<double>();
  int32_t* bsr = reinterpret_cast<int32_t*>(bv + nb);
  argmax_pass1<<<nb, kAmThreads, 0, C.stream>>>(n, v, fidx, bv, bsr);
  argmax_pass2<<<1, kAmThreads, 0, C.stream>>>(nb, bv, bsr, fidx, out_i, out_v, sel_f, sel_s, slot,
                                               knock_out ? v : nullptr);
  VL_LAUNCH_CHECK();
}
}  // namespace

void pchol_precision(Ctx& C, const Factor& F, LracFactor& LF, int k, double tol) {
  const Pattern& P = *F.pat;
  const int64_t n = P.n;
  if (k < 1 || k > n) fail(kEConfig, "rank k must be in [1, " + std::to_string(n) + "]");
  LF.k = k;
  LF.L.alloc(sizeof(double) * (size_t)n * k);
  VL_CUDA(cudaMemsetAsync(LF.L.p, 0, sizeof(double) * (size_t)n * k, C.stream));
  LF.piv_s.alloc(sizeof(int32_t) * k);
  DevBuf d, st, part, qc, touched, nt;
  d.alloc(sizeof(double) * n);
  qc.alloc(sizeof(double) * n);
  VL_CUDA(cudaMemsetAsync(qc.p, 0, sizeof(double) * n, C.stream));
  const int64_t tmax = (int64_t)(P.max_children + 1) * (P.m + 1);
  touched.alloc(sizeof(int32_t) * std::max<int64_t>(tmax, 1));
  nt.alloc(64);
  st.alloc(64);
  const int grid = std::min<int64_t>(C.num_sms * 8, (2 * n + kPcThreads - 1) / kPcThreads);
  DevBuf LT;  // column-major copy of L for the step kernel's dot products
  LT.alloc(sizeof(double) * (size_t)n * k);
  part.alloc(sizeof(double) * 4 * (size_t)grid);
  BView Bv = bview(F, false);
  launch_rows<1, 1, 1, 0, 0>(C, n, 1, DiagQBody{Bv, F.D.as<double>(), d.as<double>()}, Fin0<0>{});
  // first pivot: argmax of diag(Q), ties to the lowest factor index (preconditioners.py:311), on the device
  PcState S{st.as<int>(), reinterpret_cast<double*>(st.as<char>() + 32)};
  DevBuf amw;
  device_argmax(C, n, d.as<double>(), P.fidx.as<int32_t>(), amw, S.i, S.dp, nullptr, nullptr, 0, false);
  int h_i[4] = {0, 0, 0, 0};
  const MaternK K = make_matern(F);
  unsigned* counter = next_counter(C);
  ProfScope ps(C, "pchol_precision", 0.0);
  for (int j = 0; j < k; ++j) {
    qcol_kernel<<<1, 32, 0, C.stream>>>(P.nbr.as<int32_t>(), P.cnt.as<int32_t>(), F.val.as<double>(),
                                        P.tptr.as<int32_t>(), P.tidx.as<int32_t>(), F.valT.as<double>(),
                                        F.D.as<double>(), P.m, S, qc.as<double>(), touched.as<int32_t>(), nt.as<int>());
    pchol_step_kernel<<<grid, kPcThreads, 0, C.stream>>>(n, P.d, P.xy.as<double>(), P.fidx.as<int32_t>(), K, j, k,
                                                         LF.L.as<double>(), d.as<double>(), S, tol,
                                                         part.as<double>(), counter, LF.piv_s.as<int32_t>(),
                                                         qc.as<double>(), LT.as<double>());
    qclear_kernel<<<1, 256, 0, C.stream>>>(qc.as<double>(), touched.as<int32_t>(), nt.as<int>());
    VL_LAUNCH_CHECK();
    C.prof.launches += 3;
  }
  VL_CUDA(cudaMemcpyAsync(h_i, st.p, sizeof(h_i), cudaMemcpyDeviceToHost, C.stream));
  VL_CUDA(cudaStreamSynchronize(C.stream));
  if (h_i[2]) fail(kEFactorization, "pivoted Cholesky: diagonal went negative; input not PSD");
  LF.keff = h_i[3];
  std::vector<int32_t> ps_(LF.keff);
  if (LF.keff) VL_CUDA(cudaMemcpy(ps_.data(), LF.piv_s.p, sizeof(int32_t) * LF.keff, cudaMemcpyDeviceToHost));
  LF.piv_f.resize(LF.keff);
  for (int q = 0; q < LF.keff; ++q) LF.piv_f[q] = P.sperm[ps_[q]];
}

void rowsel_factor(Ctx& C, const Factor& F, LracFactor& LF, int k) {
  const Pattern& P = *F.pat;
  const int64_t n = P.n;
  if (k < 1 || k > n) fail(kEConfig, "rank k must be in [1, " + std::to_string(n) + "]");
  DevBuf sc;
  sc.alloc(sizeof(double) * n);
  launch_rows<1, 1, 1, 0, 0>(C, n, 1, RowScoreBody{bview(F, false), F.D.as<double>(), sc.as<double>()}, Fin0<0>{});
  // top-k of the scores with lexsort((arange, -scores)) semantics -- descending score, ties to
  // the lower factor index -- as k device argmax rounds (each knocks its winner out); only the
  // k winners come back to the host
  DevBuf amw, selb;
  selb.alloc(sizeof(int32_t) * 2 * (size_t)k);
  int32_t* sel_f = selb.as<int32_t>();
  int32_t* sel_s = sel_f + k;
  for (int c = 0; c < k; ++c)
    device_argmax(C, n, sc.as<double>(), P.fidx.as<int32_t>(), amw, nullptr, nullptr, sel_f, sel_s, c, true);
  std::vector<int32_t> sel(k);
  VL_CUDA(cudaMemcpyAsync(sel.data(), sel_f, sizeof(int32_t) * k, cudaMemcpyDeviceToHost, C.stream));
  VL_CUDA(cudaStreamSynchronize(C.stream));
  std::sort(sel.begin(), sel.end());  // S_k ascending (preconditioners.py:375)
  std::vector<int32_t> rows(k);
  for (int c = 0; c < k; ++c) rows[c] = P.iperm[sel[c]];
  LF.k = k;
  LF.keff = k;
  LF.piv_f = sel;
  LF.piv_s.alloc(sizeof(int32_t) * k);
  VL_CUDA(cudaMemcpyAsync(LF.piv_s.p, rows.data(), sizeof(int32_t) * k, cudaMemcpyHostToDevice, C.stream));
  LF.L.alloc(sizeof(double) * (size_t)n * k);
  VL_CUDA(cudaMemsetAsync(LF.L.p, 0, sizeof(double) * (size_t)n * k, C.stream));
  rowsel_scatter_kernel<<<std::max(1, (k + 127) / 128), 128, 0, C.stream>>>(
      k, k, P.m, LF.piv_s.as<int32_t>(), P.nbr.as<int32_t>(), P.cnt.as<int32_t>(), F.val.as<double>(),
      F.D.as<double>(), LF.L.as<double>());
  VL_LAUNCH_CHECK();
  VL_CUDA(cudaStreamSynchronize(C.stream));
}

void diag_sigma_tilde(Ctx& C, const Factor& F, double* out) {
  const Pattern& P = *F.pat;
  const int64_t n = P.n;
  constexpr int Wd = 64;
  DevBuf E, X;
  E.alloc(sizeof(double) * (size_t)n * Wd);
  X.alloc(sizeof(double) * (size_t)n * Wd);
  DepsCsr dbw{P.tptr.as<int32_t>(), P.tidx.as<int32_t>(), F.valT.as<double>()};
  double* sums = C.dev_scalars.as<double>();
  ProfScope ps(C, "diag_sigma_tilde", 0.0);
  for (int64_t a = 0; a < n; a += Wd) {
    const int w = (int)std::min<int64_t>(Wd, n - a);
    eye_block_kernel<<<C.num_sms * 4, 256, 0, C.stream>>>(n, (int)a, w, E.as<double>());
    VL_LAUNCH_CHECK();
    dispatch_cols(w, w, [&](auto g, auto nu, auto uu) {
      constexpr int G = decltype(g)::value, NU = decltype(nu)::value, U = decltype(uu)::value;
      launch_trsv<G, NU, U, 0>(C, F, false, w, w, dbw, X.as<double>(), TrsvPlain{E.as<double>(), w}, Fin0<0>{});
      launch_rows<G, NU, U, 1, 0>(C, n, w, DX2Body{F.D.as<double>(), X.as<double>(), w}, CopySumsL<1>{sums});
    });
    VL_CUDA(cudaMemcpyAsync(out + a, sums, sizeof(double) * w, cudaMemcpyDeviceToDevice, C.stream));
  }
}

}  // namespace vl
