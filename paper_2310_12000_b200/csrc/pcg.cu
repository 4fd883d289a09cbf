// Multi-RHS preconditioned CG for the VADU-preconditioned Laplace system
// (laplace.py:156-182 eq6 operator, preconditioners.py:101-132 VADU solve,
// iterative.py:104-178 pcg_solve).  Each column runs the reference's scalar
// recurrence independently; converged columns are frozen by a device-side
// mask so results equal a per-column stop at the reference's iteration.
//
// Sandwich preconditioners P = B^T diag(d) B (vadu, lva, l1), product modes
// 1 and 2 (Ctx::pmode1 / pmodeT): 3 kernels per iteration, no B h pass.
// With y = B^-T r and z = B^-1 (y/d) the preconditioned direction satisfies
// B z = y/d exactly, so  B^T D^-1 B z = B^T (om o y),  om = 1/(D d).
// Carrying q = B^T D^-1 B h by the same recurrence as h gives A h = W h + q:
//   E    u += alpha h (deferred from the last solves; mode 2 also r -= alpha (W h + q));
//        h = z + beta h;  q = p + beta q;  h.(W h + q) -> alpha   (last-CTA finalize)
//   Bwd  y = B^-T (r - alpha (W h + q));  ||r - alpha(W h + q)|| -> converged?
//        mode 1: p = B^T(om o y) from the same gathers (PsumOf), r stored
//   Fwd  z = B^-1 (y / d);  (r - alpha (W h + q)).z -> beta
//        mode 2: p = B^T(om o y) on a side stream, concurrent with Fwd
// Mode 3 (single RHS): mode 0 with D^-1 B h carried by recurrence (no K1).
// Mode 0 (and the diagonal preconditioners):
//   K1  tmp = D^-1 (B h);  K2  v = W h + B^T tmp, h.v -> alpha
//   K3  ||r - alpha v||;   K4  z = (r - alpha v)/d, r.z -> beta
// with the r/u updates deferred to the next elementwise h-update.
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
  VL_D void prefetch(int64_t s) const {  // single-RHS items: next item's lines into L2
    prefetch_l2(w + s * ld);
    prefetch_l2(dinv + s);
    prefetch_l2(r + s * ld);
    if (DEFER) prefetch_l2(v + s * ld);
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
// ---- sandwich form, product mode 3 (single RHS): B h by recurrence ----------
// D^-1 B h_l = om o y_l + beta D^-1 B h_{l-1}  (B z_l = y_l / d exactly), so
// the K1 pass becomes part of the deferred elementwise update.
struct DeferGBody {
  const double* z;
  const double* y;
  const double* om;
  double* h;
  double* gt;
  double* r;
  double* u;
  const double* v;
  const double* alpha;
  const double* beta;
  template <int G, int NU, int U, int NR>
  VL_D void run(int64_t s, bool valid, int, int, double (&)[NR][NU * U]) const {
    if (!valid) return;
    const double al = alpha[0], be = beta[0];
    const double hs = h[s];
    r[s] = fma(-al, v[s], r[s]);
    u[s] = fma(al, hs, u[s]);
    h[s] = z[s] + be * hs;
    gt[s] = om[s] * y[s] + be * gt[s];
  }
};
// ---- sandwich form, product mode 0: B h and B^T tmp passes ----------------
struct RhsPlainActive {  // w = B^-T r  (init)
  const double* r;
  int ld;
  VL_D double rhs(int64_t s, int c, double&) const { return r[s * ld + c]; }
  VL_D void out(int64_t, int, double, double&) const {}
};
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
  VL_D void prefetch(int64_t s) const {
    prefetch_l2(r + s * ld);
    prefetch_l2(v + s * ld);
  }
};
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

// ---- sandwich form, product modes 1 / 2 (no B h pass) ------------------------
__global__ void omega_kernel(int64_t n, const double* __restrict__ Dinv, const double* __restrict__ dinv,
                             double* __restrict__ om) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    om[i] = Dinv[i] * dinv[i];
}
// folded weights of the fused backward product: val2[e] = valT[e] om[tidx[e]]
__global__ void fold_kernel(int64_t nnz, const double* __restrict__ valT, const int32_t* __restrict__ tidx,
                            const double* __restrict__ om, double* __restrict__ val2) {
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < nnz; e += (int64_t)gridDim.x * blockDim.x)
    val2[e] = valT[e] * __ldg(om + tidx[e]);
}
// backward rhs: r_{l+1} = r - alpha (W h + q) (not stored: E stores it next
// iteration), ||r_{l+1}||^2
struct BwdRhsDef {
  const double* r;
  const double* h;
  const double* q;
  const double* W;
  const double* alpha;
  int ld;
  VL_D double rhs(int64_t s, int c, double& acc) const {
    const int64_t o = s * ld + c;
    const double rn = fma(-alpha[c], fma(W[s], h[o], q[o]), r[o]);  // alpha = 0 for frozen columns
    acc += rn * rn;
    return rn;
  }
  VL_D void out(int64_t, int, double, double&) const {}
};
// mode 1: the same solve also emits p = B^T (om o y) and stores r_{l+1}
// (at the end of the row, off the dependency chain)
struct BwdRhsDefP : BwdRhsDef {
  static constexpr bool kPsum = true;
  const double* om;
  double* pout;
  double* rout;
  VL_D void keep_rhs(int64_t s, int c, double rn) const { rout[s * ld + c] = rn; }
  VL_D void fin_row(int64_t s, int c, double x, double rn, double ps) const {
    const int64_t o = s * ld + c;
    rout[o] = rn;
    pout[o] = fma(__ldg(om + s), x, ps);
  }
};
// forward: z = B^-1 (y / d); acc += r_{l+1} . z
struct FwdDotDef {
  const double* y;
  const double* dinv;
  const double* r;
  const double* h;
  const double* q;
  const double* W;
  const double* alpha;
  int ld;
  VL_D double rhs(int64_t s, int c, double&) const { return y[s * ld + c] * dinv[s]; }
  VL_D void out(int64_t s, int c, double x, double& acc) const {
    const int64_t o = s * ld + c;
    acc += fma(-alpha[c], fma(W[s], h[o], q[o]), r[o]) * x;
  }
};
// mode 2: p = B^T (om o y) as a product pass on a side stream, concurrent
// with the forward solve (a small grid that fits beside the solve's CTAs)
struct LoadOm {
  const double* y;
  const double* om;
  VL_D void operator()(int64_t j, int, double* out) const { out[0] = __ldg(om + j) * __ldg(y + j); }
};
struct PBody1 {
  BView B;
  const double* y;
  const double* om;
  double* p;
  template <int G, int NU, int U, int NR>
  VL_D void run(int64_t s, bool valid, int gl, int t, double (&)[NR][NU * U]) const {
    double a[1] = {0.0};
    gather_Bt<1, 1, 1>(B, s, valid, gl, t, LoadOm{y, om}, a);
    if (valid) p[s] = fma(__ldg(om + s), __ldg(y + s), a[0]);
  }
};
constexpr int kSideThreads = 128;
template <class Body>
__global__ void __launch_bounds__(kSideThreads, 8) side_rows1_kernel(int64_t n, Body body,
                                                                     const int* __restrict__ gate) {
  if (gate != nullptr && *((volatile const int*)gate) == 0) return;
  const int wib = threadIdx.x >> 5, wpb = blockDim.x >> 5;
  int64_t chunk = (n + gridDim.x - 1) / gridDim.x;
  chunk = (chunk + 31) / 32 * 32;
  const int64_t r0 = (int64_t)blockIdx.x * chunk;
  const int64_t r1 = r0 + chunk < n ? r0 + chunk : n;
  double acc[1][1] = {{0.0}};
  for (int64_t s0 = r0 + (int64_t)wib * 32; s0 < r1; s0 += (int64_t)wpb * 32) {
    const int64_t s = s0 + (threadIdx.x & 31);
    body.template run<1, 1, 1, 1>(s, s < r1, 0, 1, acc);
  }
}
// E: [UPDR: r = r - alpha (W h + q)] and u += alpha h (deferred from the
// last backward solve); h = z + beta h; q = p + beta q; acc += h . (W h + q)
template <bool UPDR>
struct EBody {
  const double* z;
  const double* p;
  double* h;
  double* q;
  double* r;
  double* u;
  const double* W;
  const double* alpha;
  const double* beta;
  int ld;
  template <int G, int NU, int U, int NR>
  VL_D void run(int64_t s, bool valid, int gl, int t, double (&acc)[NR][NU * U]) const {
    if (!valid) return;
    constexpr int NC = NU * U;
    double hs[NC], qs[NC], zs[NC], ps[NC], us[NC], rs[NC];
    load_row<G, NU, U>(h, ld, s, gl, t, hs);
    load_row<G, NU, U>(q, ld, s, gl, t, qs);
    if constexpr (UPDR) load_row<G, NU, U>(r, ld, s, gl, t, rs);
    load_row<G, NU, U>(u, ld, s, gl, t, us);
    load_row<G, NU, U>(z, ld, s, gl, t, zs);
    load_row<G, NU, U>(p, ld, s, gl, t, ps);
    const double ws = W[s];
#pragma unroll
    for (int i = 0; i < NC; ++i) {
      const int c = vl::Cols<G, NU, U>::col(gl, i);
      const bool on = c < t;
      const double al = on ? alpha[c] : 0.0, be = on ? beta[c] : 0.0;
      if constexpr (UPDR) rs[i] = fma(-al, fma(ws, hs[i], qs[i]), rs[i]);
      us[i] = fma(al, hs[i], us[i]);
      hs[i] = zs[i] + be * hs[i];
      qs[i] = ps[i] + be * qs[i];
      acc[0][i] += hs[i] * fma(ws, hs[i], qs[i]);
    }
    if constexpr (UPDR) store_row<G, NU, U>(r, ld, s, gl, t, rs);
    store_row<G, NU, U>(u, ld, s, gl, t, us);
    store_row<G, NU, U>(h, ld, s, gl, t, hs);
    store_row<G, NU, U>(q, ld, s, gl, t, qs);
  }
};
struct UFlushBody {  // u += alpha h
  const double* h;
  double* u;
  const double* alpha;
  int ld;
  template <int G, int NU, int U, int NR>
  VL_D void run(int64_t s, bool valid, int gl, int t, double (&)[NR][NU * U]) const {
    if (!valid) return;
    constexpr int NC = NU * U;
    double hs[NC], us[NC];
    load_row<G, NU, U>(h, ld, s, gl, t, hs);
    load_row<G, NU, U>(u, ld, s, gl, t, us);
#pragma unroll
    for (int i = 0; i < NC; ++i) {
      const int c = vl::Cols<G, NU, U>::col(gl, i);
      us[i] = fma(c < t ? alpha[c] : 0.0, hs[i], us[i]);
    }
    store_row<G, NU, U>(u, ld, s, gl, t, us);
  }
};
}  // namespace

void pcg_vadu(Ctx& C, const SysVadu& S, int t, int ld, const double* b, double* u, double tol, int max_iter,
              bool capture, PcgResult* out) {
  const Factor& F = *S.F;
  const Pattern& P = *F.pat;
  const int64_t n = P.n;
  if (!(tol > 0)) fail(kEConfig, "tol must be > 0");
  if (max_iter < 0) fail(kEConfig, "max_iter must be >= 0");
  const size_t vb = sizeof(double) * (size_t)n * ld;
  DevBuf r, z, w, v, tmp, h0;
  r.alloc(vb); z.alloc(vb); w.alloc(vb); v.alloc(vb); tmp.alloc(vb); h0.alloc(vb);
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
  DepsEll dfw = deps_fwd(F);
  DepsCsr dbw{P.tptr.as<int32_t>(), P.tidx.as<int32_t>(), F.valT.as<double>()};
  double* hb[1] = {h0.as<double>()};

  const bool diagp = S.pkind == 1;  // diagonal preconditioner: product form, elementwise P^-1
  const int pmode = diagp ? -1 : (t == 1 ? C.pmode1 : C.pmodeT);  // 3: single RHS only
  DevBuf om, val2;
  if (pmode >= 1) {  // om = D^-1 / d
    const int g = std::max(1, std::min(4 * C.num_sms, (int)((n + 255) / 256)));
    om.alloc(sizeof(double) * (size_t)n);
    omega_kernel<<<g, 256, 0, C.stream>>>(n, S.Dinv, S.dinv, om.as<double>());
    VL_LAUNCH_CHECK();
    if (pmode == 1 && t > 1) {
      const int64_t nnzT = P.nnz_off;
      val2.alloc(sizeof(double) * (size_t)std::max<int64_t>(nnzT, 1));
      fold_kernel<<<8 * C.num_sms, 256, 0, C.stream>>>(nnzT, F.valT.as<double>(), P.tidx.as<int32_t>(),
                                                       om.as<double>(), val2.as<double>());
      VL_LAUNCH_CHECK();
    }
    if (pmode == 2 && C.side == nullptr) {
      VL_CUDA(cudaStreamCreateWithFlags(&C.side, cudaStreamNonBlocking));
      VL_CUDA(cudaEventCreateWithFlags(&C.ev_fork, cudaEventDisableTiming));
      VL_CUDA(cudaEventCreateWithFlags(&C.ev_join, cudaEventDisableTiming));
    }
  }
  DepsCsrW2 dbw2{P.tptr.as<int32_t>(), P.tidx.as<int32_t>(), F.valT.as<double>(), val2.as<double>()};
  dispatch_cols(t, ld, [&](auto g, auto nu, auto uu) {
    constexpr int G = decltype(g)::value, NU = decltype(nu)::value, U = decltype(uu)::value;
    constexpr bool DEFER = (G == 1 && NU == 1 && U == 1);  // mode 0, single RHS: r/u updates deferred
    const char* tg_h = t == 1 ? "cg1_hupd" : "cgT_hupd";
    const char* tg_bw = t == 1 ? "cg1_trsv_Bt" : "cgT_trsv_Bt";
    const char* tg_fw = t == 1 ? "cg1_trsv_B" : "cgT_trsv_B";
    const char* tg_b = t == 1 ? "cg1_spmm_B" : "cgT_spmm_B";
    const char* tg_bt = t == 1 ? "cg1_spmm_Bt" : "cgT_spmm_Bt";
    const double vbytes = 8.0 * (double)n * t;
    double* R = r.as<double>();
    double* Y = w.as<double>();    // y = B^-T r
    double* Z = z.as<double>();
    double* Q = v.as<double>();    // v (modes -1, 0) / q (modes 1, 2)
    double* Pp = tmp.as<double>(); // tmp (modes -1, 0) / p (modes 1, 2)
    double* Hh = hb[0];
    const double* Om = om.as<double>();
    ProfScope ps_init(C, t == 1 ? "cg1_init" : "cgT_init", 0.0);
    launch_rows<G, NU, U, 1, 0>(C, n, t, InitBody{b, R, u, Hh, ld}, InitFin{K, tol});
    // p = B^T (om o y) on the side stream, concurrent with the forward solve
    auto side_fork = [&]() {
      VL_CUDA(cudaEventRecord(C.ev_fork, C.stream));
      VL_CUDA(cudaStreamWaitEvent(C.side, C.ev_fork, 0));
      ProfScope ps(C, tg_bt, bapply_bytes(P, 1, 2));
      cudaEvent_t ev = (C.prof.on && C.prof.tag) ? prof_begin(C, C.side) : nullptr;
      C.prof.launches++;
      side_rows1_kernel<<<C.num_sms, kSideThreads, 0, C.side>>>(n, PBody1{B, Y, Om, Pp}, gate);
      VL_LAUNCH_CHECK();
      if (ev) prof_end(C, ev, C.side);
      VL_CUDA(cudaEventRecord(C.ev_join, C.side));
    };
    auto side_join = [&]() { VL_CUDA(cudaStreamWaitEvent(C.stream, C.ev_join, 0)); };
    auto fwd_dot = [&]() { return FwdDotDef{Y, S.dinv, R, Hh, Q, S.W, K.alpha, ld}; };
    auto fwd_dot1 = [&]() { return RhsScaleDot<false>{Y, S.dinv, R, nullptr, nullptr, ld}; };
    if (diagp) {
      launch_rows<G, NU, U, 1, 0>(C, n, t, DiagInitBody{R, S.dinv, Z, ld}, RzInitFin{K}, gate);
    } else if (pmode == 0 || pmode == 3) {
      if (pmode == 3) VL_CUDA(cudaMemsetAsync(Pp, 0, vb, C.stream));  // D^-1 B h_{-1} = 0
      launch_trsv<G, NU, U, 0>(C, F, false, t, ld, dbw, Y, RhsPlainActive{R, ld}, Fin0<0>{}, gate);
      launch_trsv<G, NU, U, 1>(C, F, true, t, ld, dfw, Z, RhsScaleDot<false>{Y, S.dinv, R, nullptr, nullptr, ld},
                               RzInitFin{K}, gate);
    } else {
      VL_CUDA(cudaMemsetAsync(Q, 0, vb, C.stream));  // q_{-1} = 0 (h_{-1} = 0 from InitBody)
      const BwdRhsDef bb{R, Hh, Q, S.W, K.alpha, ld};
      if (pmode == 1) {
        if constexpr (DEFER)
          launch_trsv<G, NU, U, 0>(C, F, false, t, ld, dbw, Y, BwdRhsDefP{bb, Om, Pp, R}, Fin0<0>{}, gate);
        else
          launch_trsv<G, NU, U, 0>(C, F, false, t, ld, dbw2, Y, BwdRhsDefP{bb, Om, Pp, R}, Fin0<0>{}, gate);
        launch_trsv<G, NU, U, 1>(C, F, true, t, ld, dfw, Z, fwd_dot1(), RzInitFin{K}, gate);
      } else {
        launch_trsv<G, NU, U, 0>(C, F, false, t, ld, dbw, Y, bb, Fin0<0>{}, gate);
        if constexpr (DEFER) side_fork();
        launch_trsv<G, NU, U, 1>(C, F, true, t, ld, dfw, Z, fwd_dot(), RzInitFin{K}, gate);
        side_join();
      }
    }
    int status[3] = {0, 0, 0};
    int l = 0;
    int chunk = 4;
    while (l < max_iter) {
      const int lim = std::min(max_iter, l + chunk);
      for (; l < lim; ++l) {
        if (pmode == 1 || pmode == 2) {
          {
            ProfScope ps(C, tg_h, (pmode == 1 ? 8.0 : 10.0) * vbytes + 8.0 * n);
            if (pmode == 1)
              launch_rows<G, NU, U, 1, 0>(C, n, t, EBody<false>{Z, Pp, Hh, Q, R, u, S.W, K.alpha, K.beta, ld},
                                          K2Fin{K, l, cap}, gate);
            else
              launch_rows<G, NU, U, 1, 0>(C, n, t, EBody<true>{Z, Pp, Hh, Q, R, u, S.W, K.alpha, K.beta, ld},
                                          K2Fin{K, l, cap}, gate);
          }
          const BwdRhsDef bb{R, Hh, Q, S.W, K.alpha, ld};
          if (pmode == 1) {
            // B^-T solve + fused B^T(om o y): B pattern/values + r, h, q, W in; y, p out
            ProfScope ps(C, tg_bw, bapply_bytes(P, t, 2) + 4.0 * vbytes + (t > 1 ? 8.0 * P.nnz_off : 0.0));
            if constexpr (DEFER)
              launch_trsv<G, NU, U, 1>(C, F, false, t, ld, dbw, Y, BwdRhsDefP{bb, Om, Pp, R}, K3Fin{K, l}, gate);
            else
              launch_trsv<G, NU, U, 1>(C, F, false, t, ld, dbw2, Y, BwdRhsDefP{bb, Om, Pp, R}, K3Fin{K, l}, gate);
          } else {
            ProfScope ps(C, tg_bw, bapply_bytes(P, t, 1) + 2.0 * vbytes);
            launch_trsv<G, NU, U, 1>(C, F, false, t, ld, dbw, Y, bb, K3Fin{K, l}, gate);
          }
          if (pmode == 2) {
            if constexpr (DEFER) side_fork();
          }
          if (pmode == 1) {
            ProfScope ps(C, tg_fw, bapply_bytes(P, t, 1) + vbytes);
            launch_trsv<G, NU, U, 1>(C, F, true, t, ld, dfw, Z, fwd_dot1(), K4Fin{K, l, cap}, gate);
          } else {
            ProfScope ps(C, tg_fw, bapply_bytes(P, t, 2) + 3.0 * vbytes);
            launch_trsv<G, NU, U, 1>(C, F, true, t, ld, dfw, Z, fwd_dot(), K4Fin{K, l, cap}, gate);
          }
          if (pmode == 2) side_join();
          continue;
        }
        double* hn = Hh;
        if constexpr (DEFER) {
          if (pmode == 3) {
            {
              ProfScope ps(C, tg_h, 8.0 * 12 * n);
              launch_rows<1, 1, 1, 0, 0>(C, n, 1, DeferGBody{Z, Y, Om, hn, Pp, R, u, Q, K.alpha, K.beta},
                                         Fin0<0>{}, gate);
            }
            {
              ProfScope ps(C, tg_bt, bapply_bytes(P, t, 1));
              launch_rows<G, NU, U, 1, 0>(C, n, t, K2Body{B, hn, Pp, Q, S.W, ld}, K2Fin{K, l, cap}, gate);
            }
            {
              ProfScope ps(C, tg_bw, bapply_bytes(P, t, 0));
              launch_trsv<G, NU, U, 1>(C, F, false, t, ld, dbw, Y, K3Rhs{R, Q, K.alpha, ld}, K3Fin{K, l}, gate);
            }
            {
              ProfScope ps(C, tg_fw, bapply_bytes(P, t, 1));
              launch_trsv<G, NU, U, 1>(C, F, true, t, ld, dfw, Z, RhsScaleDot<DEFER>{Y, S.dinv, R, Q, K.alpha, ld},
                                       K4Fin{K, l, cap}, gate);
            }
            continue;
          }
        }
        {
          ProfScope ps(C, tg_h, 24.0 * n * t);
          if (DEFER || diagp)
            launch_rows<G, NU, U, 0, 0>(C, n, t, DeferBody<true>{Z, hn, R, u, Q, K.alpha, K.beta, ld}, Fin0<0>{},
                                        gate);
          else
            launch_rows<G, NU, U, 0, 0>(C, n, t, HUpdBody{Z, hn, K.beta, ld}, Fin0<0>{}, gate);
        }
        {
          ProfScope ps(C, tg_b, bapply_bytes(P, t, 1));
          launch_rows<G, NU, U, 0, 0>(C, n, t, K1Body{B, hn, Pp, S.Dinv, ld}, Fin0<0>{}, gate);
        }
        {
          ProfScope ps(C, tg_bt, bapply_bytes(P, t, 1));
          launch_rows<G, NU, U, 1, 0>(C, n, t, K2Body{B, hn, Pp, Q, S.W, ld}, K2Fin{K, l, cap}, gate);
        }
        if (diagp) {
          launch_rows<G, NU, U, 1, 0>(C, n, t, DiagStepBody<false>{R, Q, K.alpha, nullptr, nullptr, ld},
                                      K3Fin{K, l}, gate);
          launch_rows<G, NU, U, 1, 0>(C, n, t, DiagStepBody<true>{R, Q, K.alpha, S.dinv, Z, ld}, K4Fin{K, l, cap},
                                      gate);
          continue;
        }
        {
          ProfScope ps(C, tg_bw, bapply_bytes(P, t, 0));
          if constexpr (DEFER)
            launch_trsv<G, NU, U, 1>(C, F, false, t, ld, dbw, Y, K3Rhs{R, Q, K.alpha, ld}, K3Fin{K, l}, gate);
          else
            launch_trsv<G, NU, U, 1>(C, F, false, t, ld, dbw, Y, K3RhsFused{R, u, Q, hn, K.alpha, ld}, K3Fin{K, l},
                                     gate);
        }
        {
          ProfScope ps(C, tg_fw, bapply_bytes(P, t, 1));
          launch_trsv<G, NU, U, 1>(C, F, true, t, ld, dfw, Z, RhsScaleDot<DEFER>{Y, S.dinv, R, Q, K.alpha, ld},
                                   K4Fin{K, l, cap}, gate);
        }
      }
      VL_CUDA(cudaMemcpyAsync(status, K.status, sizeof(status), cudaMemcpyDeviceToHost, C.stream));
      VL_CUDA(cudaStreamSynchronize(C.stream));
      if (status[1] != 0 || status[0] == 0) break;
      chunk = std::min(chunk * 2, 16);
    }
    // flush the last deferred update (alpha = 0 when nothing is pending)
    if (pmode == 1 || pmode == 2)
      launch_rows<G, NU, U, 0, 0>(C, n, t, UFlushBody{Hh, u, K.alpha, ld}, Fin0<0>{});
    else if (DEFER || diagp)
      launch_rows<G, NU, U, 0, 0>(C, n, t, DeferBody<false>{nullptr, Hh, R, u, Q, K.alpha, nullptr, ld}, Fin0<0>{});
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
