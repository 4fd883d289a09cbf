// Multi-RHS preconditioned CG for the VADU-preconditioned Laplace system
// (laplace.py:156-182 eq6 operator, preconditioners.py:101-132 VADU solve,
// iterative.py:104-178 pcg_solve).  Each column runs the reference's scalar
// recurrence independently; converged columns are frozen by a device-side
// mask so results equal a per-column stop at the reference's iteration.
//
// One iteration = 4 kernels:
//   K1  h = z + beta h_prev (fused into the gather),  tmp = D^-1 (B h)
//   K2  v = W h + B^T tmp,  h.v -> alpha            (last-CTA finalize)
//   K3  w = B^-T (r - alpha v),  ||r - alpha v|| -> converged?
//   K4  z = B^-1 (w / d),  (r - alpha v).z -> beta
// The r/u updates themselves (r -= alpha v, u += alpha h) are deferred to
// the next iteration's elementwise h-update (and a final flush), so the
// solves' rows read two vectors instead of read-modify-writing four.
#include <cmath>
#include <cstring>

#include "bodies.cuh"
#include "launch.cuh"
#include "ops.h"
#include "pcg.h"
#include "pcg_common.cuh"

namespace vl {

namespace {
using namespace cg;

// ---- preconditioner solve pieces ------------------------------------------
struct RhsPlainActive {  // w = B^-T r  (init)
  const double* r;
  int ld;
  VL_D double rhs(int64_t s, int c, double&) const { return r[s * ld + c]; }
  VL_D void out(int64_t, int, double, double&) const {}
};
template <bool DEFER>
struct RhsScaleDot {  // z = B^-1 (w * dinv) ; acc += (r - alpha v) . z
  const double* w;
  const double* dinv;
  const double* r;
  const double* v;
  const double* alpha;
  int ld;
  VL_D double rhs(int64_t s, int c, double&) const { return w[s * ld + c] * dinv[s]; }
  VL_D void out(int64_t s, int c, double x, double& acc) const {
    const int64_t o = s * ld + c;
    const double rn = DEFER ? fma(-alpha[c], v[o], r[o]) : r[o];
    acc += rn * x;
  }
};
struct RzInitFin {
  CgCols K;
  VL_D void operator()(const double* sums, int t) const {
    for (int c = threadIdx.x; c < t; c += blockDim.x) K.rz[c] = sums[c];
  }
};

// ---- K1: tmp = Dinv (B h) ------------------------------------------------------
struct K1Body {
  BView B;
  const double* h;
  double* tmp;
  const double* Dinv;
  int ld;
  template <int G, int NU, int U, int NR>
  VL_D void run(int64_t s, bool valid, int gl, int t, double (&)[NR][NU * U]) const {
    double a[NU * U];
    zero(a);
    gather_B<G, NU, U>(B, B.val, s, valid, gl, t, LoadU<U>{h, ld}, a);
    if (!valid) return;
    double hs[NU * U];
    load_row<G, NU, U>(h, ld, s, gl, t, hs);
    const double di = Dinv[s];
#pragma unroll
    for (int i = 0; i < NU * U; ++i) a[i] = di * (hs[i] + a[i]);
    store_row<G, NU, U>(tmp, ld, s, gl, t, a);
  }
};

// ---- K2: v = W h + B^T tmp; h.v -> alpha -----------------------------------
struct K2Body {
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
// ---- K3: r -= alpha v, u += alpha h (rhs of w = B^-T r); ||r|| -------------
struct K3Rhs {
  const double* r;
  const double* v;
  const double* alpha;
  int ld;
  VL_D double rhs(int64_t s, int c, double& acc) const {
    const int64_t o = s * ld + c;
    const double rn = fma(-alpha[c], v[o], r[o]);  // alpha = 0 for frozen columns
    acc += rn * rn;
    return rn;
  }
  VL_D void out(int64_t, int, double, double&) const {}
};
// t > 1: the update stays fused into the solve's rhs (the solve is gather-
// bound there, and deferring would add a pass over r, u, v per iteration)
struct K3RhsFused {
  double* r;
  double* u;
  const double* v;
  const double* h;
  const double* alpha;
  int ld;
  VL_D double rhs(int64_t s, int c, double& acc) const {
    const int64_t o = s * ld + c;
    const double al = alpha[c];  // 0 for frozen columns
    const double rn = fma(-al, v[o], r[o]);
    r[o] = rn;
    u[o] = fma(al, h[o], u[o]);
    acc += rn * rn;
    return rn;
  }
  VL_D void out(int64_t, int, double, double&) const {}
};
// ---- diagonal preconditioners (diag / identity): elementwise P^-1 -----------
struct DiagInitBody {  // z = r / d ; acc += r . z
  const double* r;
  const double* dinv;
  double* z;
  int ld;
  template <int G, int NU, int U, int NR>
  VL_D void run(int64_t s, bool valid, int gl, int t, double (&acc)[NR][NU * U]) const {
    if (!valid) return;
    double a[NU * U];
    load_row<G, NU, U>(r, ld, s, gl, t, a);
    const double di = dinv[s];
#pragma unroll
    for (int i = 0; i < NU * U; ++i) {
      const double zz = a[i] * di;
      acc[0][i] += a[i] * zz;
      a[i] = zz;
    }
    store_row<G, NU, U>(z, ld, s, gl, t, a);
  }
};
template <bool STORE>  // false: ||r - alpha v||^2 (K3) ; true: z = (r - alpha v)/d, (r - alpha v).z (K4)
struct DiagStepBody {
  const double* r;
  const double* v;
  const double* alpha;
  const double* dinv;
  double* z;
  int ld;
  template <int G, int NU, int U, int NR>
  VL_D void run(int64_t s, bool valid, int gl, int t, double (&acc)[NR][NU * U]) const {
    if (!valid) return;
    constexpr int NC = NU * U;
    double rs[NC], vs[NC];
    load_row<G, NU, U>(r, ld, s, gl, t, rs);
    load_row<G, NU, U>(v, ld, s, gl, t, vs);
    const double di = STORE ? dinv[s] : 0.0;
#pragma unroll
    for (int i = 0; i < NC; ++i) {
      const int c = vl::Cols<G, NU, U>::col(gl, i);
      const double rn = fma(-(c < t ? alpha[c] : 0.0), vs[i], rs[i]);
      if (STORE) {
        rs[i] = rn * di;
        acc[0][i] += rn * rs[i];
      } else {
        acc[0][i] += rn * rn;
      }
    }
    if (STORE) store_row<G, NU, U>(z, ld, s, gl, t, rs);
  }
};
// ---- deferred update: r -= alpha v, u += alpha h; then h = z + beta h -------
template <bool HUPD>
struct DeferBody {
  const double* z;
  double* h;
  double* r;
  double* u;
  const double* v;
  const double* alpha;
  const double* beta;
  int ld;
  template <int G, int NU, int U, int NR>
  VL_D void run(int64_t s, bool valid, int gl, int t, double (&)[NR][NU * U]) const {
    if (!valid) return;
    constexpr int NC = NU * U;
    double hs[NC], rs[NC], us[NC], vs[NC];
    load_row<G, NU, U>(h, ld, s, gl, t, hs);
    load_row<G, NU, U>(r, ld, s, gl, t, rs);
    load_row<G, NU, U>(u, ld, s, gl, t, us);
    load_row<G, NU, U>(v, ld, s, gl, t, vs);
#pragma unroll
    for (int i = 0; i < NC; ++i) {
      const int c = vl::Cols<G, NU, U>::col(gl, i);
      const double al = c < t ? alpha[c] : 0.0;
      rs[i] = fma(-al, vs[i], rs[i]);
      us[i] = fma(al, hs[i], us[i]);
    }
    store_row<G, NU, U>(r, ld, s, gl, t, rs);
    store_row<G, NU, U>(u, ld, s, gl, t, us);
    if constexpr (HUPD) {
      double zs[NC];
      load_row<G, NU, U>(z, ld, s, gl, t, zs);
#pragma unroll
      for (int i = 0; i < NC; ++i) {
        const int c = vl::Cols<G, NU, U>::col(gl, i);
        hs[i] = zs[i] + (c < t ? beta[c] : 0.0) * hs[i];
      }
      store_row<G, NU, U>(h, ld, s, gl, t, hs);
    }
  }
};
// ---- K4: z = B^-1 (w / d); r.z -> beta -------------------------------------
}  // namespace

void pcg_vadu(Ctx& C, const SysVadu& S, int t, int ld, const double* b, double* u, double tol, int max_iter,
              bool capture, PcgResult* out) {
  const Factor& F = *S.F;
  const Pattern& P = *F.pat;
  const int64_t n = P.n;
  if (!(tol > 0)) fail(kEConfig, "tol must be > 0");
  if (max_iter < 0) fail(kEConfig, "max_iter must be >= 0");
  const size_t vb = sizeof(double) * (size_t)n * ld;
  DevBuf r, z, w, v, tmp, h0, h1;
  r.alloc(vb); z.alloc(vb); w.alloc(vb); v.alloc(vb); tmp.alloc(vb); h0.alloc(vb); h1.alloc(vb);
  VL_CUDA(cudaMemsetAsync(v.p, 0, vb, C.stream));  // read (times alpha = 0) by the first deferred update
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
  BView B = bview(F, false);
  DepsEll dfw{P.nbr.as<int32_t>(), P.cnt.as<int32_t>(), F.val.as<double>(), P.m};
  DepsCsr dbw{P.tptr.as<int32_t>(), P.tidx.as<int32_t>(), F.valT.as<double>()};
  double* hb[2] = {h0.as<double>(), h1.as<double>()};

  dispatch_cols(t, ld, [&](auto g, auto nu, auto uu) {
    constexpr int G = decltype(g)::value, NU = decltype(nu)::value, U = decltype(uu)::value;
    constexpr bool DEFER = (G == 1 && NU == 1 && U == 1);  // single RHS: r/u updates deferred
    const bool diagp = S.pkind == 1;  // diagonal preconditioner: elementwise P^-1, updates deferred
    // init
    ProfScope ps_init(C, t == 1 ? "cg1_init" : "cgT_init", 0.0);
    launch_rows<G, NU, U, 1, 0>(C, n, t, InitBody{b, r.as<double>(), u, hb[0], ld}, InitFin{K, tol});
    if (diagp) {
      launch_rows<G, NU, U, 1, 0>(C, n, t, DiagInitBody{r.as<double>(), S.dinv, z.as<double>(), ld}, RzInitFin{K},
                                  gate);
    } else {
      launch_trsv<G, NU, U, 0>(C, F, false, t, ld, dbw, w.as<double>(),
                               RhsPlainActive{r.as<double>(), ld}, Fin0<0>{}, gate);
      launch_trsv<G, NU, U, 1>(C, F, true, t, ld, dfw, z.as<double>(),
                               RhsScaleDot<false>{w.as<double>(), S.dinv, r.as<double>(), nullptr, nullptr, ld},
                               RzInitFin{K}, gate);
    }
    int status[3] = {0, 0, 0};
    int l = 0;
    int chunk = 4;
    while (l < max_iter) {
      const int lim = std::min(max_iter, l + chunk);
      for (; l < lim; ++l) {
        double* hn = hb[0];
        {
          ProfScope ps(C, t == 1 ? "cg1_hupd" : "cgT_hupd", 24.0 * n * t);
          if (DEFER || diagp)
            launch_rows<G, NU, U, 0, 0>(C, n, t,
                                        DeferBody<true>{z.as<double>(), hn, r.as<double>(), u, v.as<double>(),
                                                        K.alpha, K.beta, ld},
                                        Fin0<0>{}, gate);
          else
            launch_rows<G, NU, U, 0, 0>(C, n, t, HUpdBody{z.as<double>(), hn, K.beta, ld}, Fin0<0>{}, gate);
        }
        {
          ProfScope ps(C, t == 1 ? "cg1_spmm_B" : "cgT_spmm_B", bapply_bytes(P, t, 1));
          launch_rows<G, NU, U, 0, 0>(C, n, t, K1Body{B, hn, tmp.as<double>(), S.Dinv, ld}, Fin0<0>{}, gate);
        }
        {
          ProfScope ps(C, t == 1 ? "cg1_spmm_Bt" : "cgT_spmm_Bt", bapply_bytes(P, t, 1));
          launch_rows<G, NU, U, 1, 0>(C, n, t, K2Body{B, hn, tmp.as<double>(), v.as<double>(), S.W, ld},
                                      K2Fin{K, l, cap}, gate);
        }
        {
          ProfScope ps(C, t == 1 ? "cg1_trsv_Bt" : "cgT_trsv_Bt", bapply_bytes(P, t, 0));
          if (diagp)
            launch_rows<G, NU, U, 1, 0>(C, n, t,
                                        DiagStepBody<false>{r.as<double>(), v.as<double>(), K.alpha, nullptr,
                                                            nullptr, ld},
                                        K3Fin{K, l}, gate);
          else if constexpr (DEFER)
            launch_trsv<G, NU, U, 1>(C, F, false, t, ld, dbw, w.as<double>(),
                                     K3Rhs{r.as<double>(), v.as<double>(), K.alpha, ld}, K3Fin{K, l}, gate);
          else
            launch_trsv<G, NU, U, 1>(C, F, false, t, ld, dbw, w.as<double>(),
                                     K3RhsFused{r.as<double>(), u, v.as<double>(), hn, K.alpha, ld}, K3Fin{K, l},
                                     gate);
        }
        {
          ProfScope ps(C, t == 1 ? "cg1_trsv_B" : "cgT_trsv_B", bapply_bytes(P, t, 1));
          if (diagp)
            launch_rows<G, NU, U, 1, 0>(C, n, t,
                                        DiagStepBody<true>{r.as<double>(), v.as<double>(), K.alpha, S.dinv,
                                                           z.as<double>(), ld},
                                        K4Fin{K, l, cap}, gate);
          else
            launch_trsv<G, NU, U, 1>(C, F, true, t, ld, dfw, z.as<double>(),
                                     RhsScaleDot<DEFER>{w.as<double>(), S.dinv, r.as<double>(), v.as<double>(),
                                                        K.alpha, ld},
                                     K4Fin{K, l, cap}, gate);
        }
      }
      VL_CUDA(cudaMemcpyAsync(status, K.status, sizeof(status), cudaMemcpyDeviceToHost, C.stream));
      VL_CUDA(cudaStreamSynchronize(C.stream));
      if (status[1] != 0 || status[0] == 0) break;
      chunk = std::min(chunk * 2, 16);
    }
    // flush the last deferred update (alpha = 0 when nothing is pending)
    if (DEFER || diagp)
      launch_rows<G, NU, U, 0, 0>(C, n, t,
                                  DeferBody<false>{nullptr, hb[0], r.as<double>(), u, v.as<double>(), K.alpha,
                                                   nullptr, ld},
                                  Fin0<0>{});
    if (status[1] != 0) {
      double ev = 0;
      VL_CUDA(cudaMemcpy(&ev, K.errval, sizeof(double), cudaMemcpyDeviceToHost));
      char buf[256];
      snprintf(buf, sizeof(buf), "CG breakdown in column %d: curvature %.3e <= 0 (operator or preconditioner not PD)",
               status[2], ev);
      fail(kEBreakdown, buf);
    }
  });
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
      VL_CUDA(cudaMemcpyAsync(out->alpha.data(), K.ah, sizeof(double) * mx * t, cudaMemcpyDeviceToHost, C.stream));
      VL_CUDA(cudaMemcpyAsync(out->beta.data(), K.bh, sizeof(double) * mx * t, cudaMemcpyDeviceToHost, C.stream));
      VL_CUDA(cudaStreamSynchronize(C.stream));
    }
  }
}

}  // namespace vl
