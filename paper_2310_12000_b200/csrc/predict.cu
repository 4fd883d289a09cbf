// Prediction path on the device (predict.py:45-101,
// vecchia.py:364-441):
//   blocks  : Bpo rows (= -A, A = K^-1 k over the take nearest training
//             points) and Dp, built by the factor-build warp kernel;
//   mean    : omega = F_p - Bpo b*;
//   sim var : per sample z3 = W^1/2 z1 + B^T D^-1/2 z2, u = (W + Q)^-1 z3
//             (multi-RHS PCG, one column per sample), z4 = Bpo u,
//             acc += z4^2 in sample order (and the full n_p x n_p second
//             moment with a rank-c update when requested).
#include "dense.h"

#include "bodies.cuh"
#include "launch.cuh"
#include "ops.h"
#include "predict.h"

namespace vl {

void pred_build(Ctx& C, const Pattern& P, double sigma2, double rho, double nu, const double* qxy_dev, int64_t np,
                int take, const int32_t* nbr_dev, const int32_t* cnt_dev, double* A_dev, double* Dp_dev);

namespace {

__global__ void map_nbr_kernel(int64_t ne, const int32_t* __restrict__ fac, const int32_t* __restrict__ iperm,
                               int32_t* __restrict__ out) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < ne; e += (int64_t)gridDim.x * blockDim.x)
    out[e] = iperm[fac[e]];
}

__global__ void fill_int_kernel(int64_t n, int v, int32_t* __restrict__ out) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x)
    out[e] = v;
}

// y_q = sum_e Bpo[q,e] X[nbr[q,e], :]  (column groups as in rows_kernel)
template <class Out>
struct PredRowsBody {
  const int32_t* nbr;
  const double* val;  // Bpo values (-A)
  int take;
  const double* X;
  int ld;
  Out out;
  template <int G, int NU, int U, int NR>
  VL_D void run(int64_t q, bool valid, int gl, int t, double (&acc)[NR][NU * U]) const {
    if (!valid) return;
    double a[NU * U];
    zero(a);
    const int32_t* nb = nbr + q * take;
    const double* vv = val + q * take;
    gather<G, NU, U>(
        take, gl, t, [&](int e) { return nb[e]; }, [&](int e) { return vv[e]; }, LoadU<U>{X, ld}, a);
    out.template put<G, NU, U>(q, gl, t, a);
  }
};

struct MeanOut {  // omega = F_p + (-(Bpo b))
  const double* Fp;
  double* omega;
  template <int G, int NU, int U>
  VL_D void put(int64_t q, int gl, int, double (&a)[NU * U]) const {
    if (gl == 0) omega[q] = Fp[q] + (-a[0]);
  }
};

struct StoreOut {  // z4 (np x ld)
  double* Z;
  int ld;
  template <int G, int NU, int U>
  VL_D void put(int64_t q, int gl, int t, double (&a)[NU * U]) const {
    store_row<G, NU, U>(Z, ld, q, gl, t, a);
  }
};

// z3 = sqrt(W) o z1 + B^T (D^-1/2 o z2)
struct Z3Body {
  BView B;
  const double* W;
  const double* D;
  const double* z1;
  const double* z2;
  double* z3;
  int ld;
  template <int G, int NU, int U, int NR>
  VL_D void run(int64_t s, bool valid, int gl, int t, double (&)[NR][NU * U]) const {
    auto load = [&](int64_t j, int c, double* out) {
      load_unit<U>(z2 + j * ld + c, out);
      const double f = 1.0 / sqrt(D[j]);
#pragma unroll
      for (int i = 0; i < U; ++i) out[i] *= f;
    };
    double a[NU * U];
    zero(a);
    gather_Bt<G, NU, U>(B, s, valid, gl, t, load, a);
    if (!valid) return;
    double v2[NU * U], v1[NU * U];
    load_row<G, NU, U>(z2, ld, s, gl, t, v2);
    load_row<G, NU, U>(z1, ld, s, gl, t, v1);
    const double ds = 1.0 / sqrt(D[s]);
    const double ws = sqrt(W[s]);
#pragma unroll
    for (int i = 0; i < NU * U; ++i) a[i] = ws * v1[i] + (ds * v2[i] + a[i]);
    store_row<G, NU, U>(z3, ld, s, gl, t, a);
  }
};

__global__ void accum_sq_kernel(int64_t np, int c, const double* __restrict__ Z, double* __restrict__ acc) {
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < np; q += (int64_t)gridDim.x * blockDim.x) {
    double a = acc[q];
    for (int k = 0; k < c; ++k) {
      const double z = Z[q * c + k];
      a += z * z;
    }
    acc[q] = a;
  }
}


}  // namespace

void pred_create(Ctx& C, const Pattern& P, double sigma2, double rho, double nu, const double* qxy_host, int64_t np,
                 const int32_t* nbr_factor_host, int take, PredBlocks& B) {
  B.np = np;
  B.take = take;
  B.d = P.d;
  B.qxy.alloc(sizeof(double) * std::max<int64_t>(np * P.d, 1));
  B.nbr.alloc(sizeof(int32_t) * std::max<int64_t>(np * take, 1));
  B.cnt.alloc(sizeof(int32_t) * std::max<int64_t>(np, 1));
  B.val.alloc(sizeof(double) * std::max<int64_t>(np * take, 1));
  B.Dp.alloc(sizeof(double) * std::max<int64_t>(np, 1));
  if (np == 0) return;
  for (int64_t e = 0; e < np * take; ++e)
    if (nbr_factor_host[e] < 0 || nbr_factor_host[e] >= P.n) fail(kEConfig, "prediction neighbour out of range");
  DevBuf fac, ip;
  fac.alloc(sizeof(int32_t) * np * take);
  ip.alloc(sizeof(int32_t) * P.n);
  VL_CUDA(cudaMemcpyAsync(B.qxy.p, qxy_host, sizeof(double) * np * P.d, cudaMemcpyHostToDevice, C.stream));
  VL_CUDA(cudaMemcpyAsync(fac.p, nbr_factor_host, sizeof(int32_t) * np * take, cudaMemcpyHostToDevice, C.stream));
  VL_CUDA(cudaMemcpyAsync(ip.p, P.iperm.data(), sizeof(int32_t) * P.n, cudaMemcpyHostToDevice, C.stream));
  map_nbr_kernel<<<C.num_sms * 4, 256, 0, C.stream>>>(np * take, fac.as<int32_t>(), ip.as<int32_t>(),
                                                       B.nbr.as<int32_t>());
  fill_int_kernel<<<C.num_sms * 4, 256, 0, C.stream>>>(np, take, B.cnt.as<int32_t>());
  VL_LAUNCH_CHECK();
  pred_build(C, P, sigma2, rho, nu, B.qxy.as<double>(), np, take, B.nbr.as<int32_t>(), B.cnt.as<int32_t>(),
             B.val.as<double>(), B.Dp.as<double>());
}

void pred_mean(Ctx& C, const PredBlocks& B, const double* b_dev, const double* Fp_dev, double* omega_dev) {
  if (B.np == 0) return;
  ProfScope ps(C, "pred_mean", 0.0);
  launch_rows<1, 1, 1, 0, 0>(C, B.np, 1,
                             PredRowsBody<MeanOut>{B.nbr.as<int32_t>(), B.val.as<double>(), B.take, b_dev, 1,
                                                   MeanOut{Fp_dev, omega_dev}},
                             Fin0<0>{});
}

void pred_z3(Ctx& C, const Factor& F, const double* W, int c, const double* z1, const double* z2, double* z3) {
  const int64_t n = F.pat->n;
  ProfScope ps(C, "pred_z3", 0.0);
  BView Bv = bview(F, false);
  dispatch_cols(c, c, [&](auto g, auto nu, auto uu) {
    constexpr int G = decltype(g)::value, NU = decltype(nu)::value, U = decltype(uu)::value;
    launch_rows<G, NU, U, 0, 0>(C, n, c, Z3Body{Bv, W, F.D.as<double>(), z1, z2, z3, c}, Fin0<0>{});
  });
}

void pred_accum(Ctx& C, const PredBlocks& B, const double* U_dev, int c, double* acc_dev, double* cov_dev) {
  if (B.np == 0 || c == 0) return;
  ProfScope ps(C, "pred_accum", 0.0);
  DevBuf Z;
  Z.alloc(sizeof(double) * (size_t)B.np * c);
  dispatch_cols(c, c, [&](auto g, auto nu, auto uu) {
    constexpr int G = decltype(g)::value, NU = decltype(nu)::value, U = decltype(uu)::value;
    launch_rows<G, NU, U, 0, 0>(C, B.np, c,
                                PredRowsBody<StoreOut>{B.nbr.as<int32_t>(), B.val.as<double>(), B.take, U_dev, c,
                                                       StoreOut{Z.as<double>(), c}},
                                Fin0<0>{});
  });
  accum_sq_kernel<<<C.num_sms * 4, 256, 0, C.stream>>>(B.np, c, Z.as<double>(), acc_dev);
  VL_LAUNCH_CHECK();
  if (cov_dev) {
    // cov (np x np, symmetric, both triangles) += Z Z^T ; Z row-major np x c == column-major c x np
    Gemm g;
    g.ta = true;
    g.m = (int)B.np; g.n = (int)B.np; g.k = c;
    g.A = Z.as<double>(); g.lda = c;
    g.B = Z.as<double>(); g.ldb = c;
    g.beta = 1.0;
    g.C = cov_dev; g.ldc = (int)B.np;
    dgemm(C, g);
  }
}

}  // namespace vl
