// Laplace objective on the device (laplace.py, likelihoods.py).
#include <cmath>
#include <cstring>

#include "bodies.cuh"
#include "laplace.h"
#include "launch.cuh"
#include "lrac.h"
#include "ops.h"

namespace vl {

// ---------------------------------------------------------------------------
// Likelihood functors (likelihoods.py:62-174), elementwise in mu.
// ---------------------------------------------------------------------------
struct Lik {
  int fam;
  double a;       // gamma shape
  double aloga;   // a log a - lgamma(a)
  VL_D static double logaddexp0(double mu) {  // numpy npy_logaddexp(0, mu)
    if (mu == 0.0) return 0.6931471805599453;
    const double tmp = -mu;
    if (tmp > 0) return log1p(exp(mu));
    if (tmp <= 0) return mu + log1p(exp(-mu));
    return tmp;
  }
  VL_D static double expit(double x) {
    if (x < 0) {
      const double z = exp(x);
      return z / (1.0 + z);
    }
    return 1.0 / (1.0 + exp(-x));
  }
  VL_D static double log_ndtr(double x) {
    const double t = x * 0.70710678118654752440;
    if (x < -1.0) return log(erfcx(-t) / 2.0) - t * t;
    return log1p(-erfc(t) / 2.0);
  }
  VL_D double logdens(double y, double mu) const {
    if (fam == 0) return y * mu - logaddexp0(mu);
    if (fam == 1) return log_ndtr((2.0 * y - 1.0) * mu);
    if (fam == 3) return y * mu - exp(mu) - lgamma(y + 1.0);
    return aloga + (a - 1.0) * log(y) - a * mu - a * y * exp(-mu);
  }
  // returns log p and writes d1, d2, d3
  VL_D double derivs(double y, double mu, double& d1, double& d2, double& d3) const {
    if (fam == 0) {
      const double p = expit(mu);
      const double w = p * (1.0 - p);
      d1 = y - p;
      d2 = -w;
      d3 = -w * (1.0 - 2.0 * p);
    } else if (fam == 1) {
      const double z = 2.0 * y - 1.0;
      const double u = z * mu;
      const double g = exp(-0.5 * u * u - 0.91893853320467274178 - log_ndtr(u));
      d1 = z * g;
      d2 = -g * (u + g);
      d3 = z * g * ((u + g) * (u + g) + g * (u + g) - 1.0);
    } else if (fam == 3) {  // Poisson, log link (the prediction config's family; test-registered in the reference)
      const double e = exp(mu);
      d1 = y - e;
      d2 = -e;
      d3 = -e;
    } else {
      const double w = a * y * exp(-mu);
      d1 = -a + w;
      d2 = -w;
      d3 = w;
    }
    return logdens(y, mu);
  }
};

static Lik make_lik(const LikSpec& L) {
  Lik k;
  k.fam = L.family;
  k.a = L.shape;
  k.aloga = (L.family == 2) ? L.shape * std::log(L.shape) - std::lgamma(L.shape) : 0.0;
  if (L.family < 0 || L.family > 3) fail(kEConfig, "unknown likelihood family");
  if (L.family == 2 && !(L.shape > 0)) fail(kEConfig, "gamma shape must be > 0");
  return k;
}

namespace {

// ---- Newton bodies (t = 1) ---------------------------------------------------
// b <- b + step*delta (if delta), derivatives at mu = F + b, W = max(-d2,0),
// rhs = W b + d1.  sums: [log p, ||rhs||^2, max |d1|]
struct DerivsBody {
  Lik L;
  const double* y;
  const double* Fv;
  double* b;
  const double* delta;
  double step;
  double* d1;
  double* W;
  double* d3;
  double* rhs;
  template <int G, int NU, int U, int NR>
  VL_D void run(int64_t s, bool valid, int, int, double (&acc)[NR][NU * U]) const {
    if (!valid) return;
    double bs = b[s];
    if (delta != nullptr) {
      bs = bs + step * delta[s];
      b[s] = bs;
    }
    double a1, a2, a3;
    const double lp = L.derivs(y[s], Fv[s] + bs, a1, a2, a3);
    const double w = fmax(-a2, 0.0);
    d1[s] = a1;
    W[s] = w;
    d3[s] = a3;
    const double r = w * bs + a1;
    rhs[s] = r;
    acc[0][0] += lp;
    acc[1][0] += r * r;
    acc[2][0] = fmax(acc[2][0], fabs(a1));
  }
};

// trial point bt = b + step*delta: sums [log p(bt), bt^T Q bt = sum (B bt)^2 / D]
struct TrialBody {
  Lik L;
  BView B;
  const double* y;
  const double* Fv;
  const double* b;
  const double* delta;
  double step;
  const double* Dinv;
  template <int G, int NU, int U, int NR>
  VL_D void run(int64_t s, bool valid, int gl, int t, double (&acc)[NR][NU * U]) const {
    auto load = [&](int64_t j, int, double* out) { out[0] = b[j] + step * delta[j]; };
    double a[1] = {0.0};
    gather_B<1, 1, 1>(B, B.val, s, valid, gl, 1, load, a);
    if (!valid) return;
    const double bs = b[s] + step * delta[s];
    const double Bb = bs + a[0];
    acc[0][0] += L.logdens(y[s], Fv[s] + bs);
    acc[1][0] += Bb * Bb * Dinv[s];
  }
};

struct DiffBody {  // delta = x - b
  const double* x;
  const double* b;
  double* delta;
  template <int G, int NU, int U, int NR>
  VL_D void run(int64_t s, bool valid, int, int, double (&)[NR][NU * U]) const {
    if (valid) delta[s] = x[s] - b[s];
  }
};

struct ScaleBBody {  // tmp = Dinv o (B b)
  BView B;
  const double* b;
  const double* Dinv;
  double* tmp;
  template <int G, int NU, int U, int NR>
  VL_D void run(int64_t s, bool valid, int gl, int t, double (&)[NR][NU * U]) const {
    double a[1] = {0.0};
    gather_B<1, 1, 1>(B, B.val, s, valid, gl, 1, LoadU<1>{b, 1}, a);
    if (valid) tmp[s] = Dinv[s] * (b[s] + a[0]);
  }
};

struct GradNormBody {  // max |d1 - B^T tmp|
  BView B;
  const double* tmp;
  const double* d1;
  template <int G, int NU, int U, int NR>
  VL_D void run(int64_t s, bool valid, int gl, int t, double (&acc)[NR][NU * U]) const {
    double a[1] = {0.0};
    gather_Bt<1, 1, 1>(B, s, valid, gl, 1, LoadU<1>{tmp, 1}, a);
    if (valid) acc[0][0] = fmax(acc[0][0], fabs(d1[s] - (tmp[s] + a[0])));
  }
};

struct DiagsBody {
  const double* D;
  const double* W;
  double* Dinv;
  double* dinv;
  template <int G, int NU, int U, int NR>
  VL_D void run(int64_t s, bool valid, int, int, double (&)[NR][NU * U]) const {
    if (!valid) return;
    const double di = 1.0 / D[s];
    Dinv[s] = di;
    dinv[s] = 1.0 / (W[s] + di);
  }
};

template <int NR>
struct CopySums {
  double* dst;
  VL_D void operator()(const double* sums, int t) const {
    for (int i = threadIdx.x; i < NR * t; i += blockDim.x) dst[i] = sums[i];
  }
};

}  // namespace

static void read_sums(Ctx& C, const double* dev, double* host, int cnt) {
  VL_CUDA(cudaMemcpyAsync(host, dev, sizeof(double) * cnt, cudaMemcpyDeviceToHost, C.stream));
  VL_CUDA(cudaStreamSynchronize(C.stream));
}

namespace {
// 1/d of the eq6 preconditioner variants (preconditioners.py:338-387):
// 0 vadu / 1 l1: d = W + 1/D ; 2 lva: d = 1/D ; 3 diag: d = W + diag(B^T D^-1 B) ; 4 identity: d = 1
struct PrecDinvBody {
  int variant;
  BView B;
  const double* D;
  const double* W;
  double* dinv;
  template <int G, int NU, int U, int NR>
  VL_D void run(int64_t s, bool valid, int, int, double (&)[NR][NU * U]) const {
    if (!valid) return;
    double v;
    if (variant <= 1) {
      v = 1.0 / (W[s] + 1.0 / D[s]);
    } else if (variant == 2) {
      v = D[s];
    } else if (variant == 3) {
      // column s of B: the unit diagonal (row s) and the children rows
      double q = 1.0 / D[s];
      for (int32_t e = B.tptr[s]; e < B.tptr[s + 1]; ++e) {
        const double b = B.valT[e];
        q += b * b / D[B.tidx[e]];
      }
      v = 1.0 / (W[s] + q);
    } else {
      v = 1.0;
    }
    dinv[s] = v;
  }
};
struct SumLogBody {
  const double* x;
  template <int G, int NU, int U, int NR>
  VL_D void run(int64_t s, bool valid, int, int, double (&acc)[NR][NU * U]) const {
    if (valid) acc[0][0] += log(x[s]);
  }
};
}  // namespace

void precond_dinv(Ctx& C, const Factor& F, int variant, const double* W, double* dinv) {
  if (variant < 0 || variant > 4) fail(kEConfig, "unknown eq6 preconditioner variant");
  launch_rows<1, 1, 1, 0, 0>(C, F.pat->n, 1, PrecDinvBody{variant, bview(F, false), F.D.as<double>(), W, dinv},
                             Fin0<0>{});
}

double sum_log(Ctx& C, int64_t n, const double* x) {
  double* sums = C.dev_scalars.as<double>();
  launch_rows<1, 1, 1, 1, 0>(C, n, 1, SumLogBody{x}, CopySums<1>{sums});
  double h;
  VL_CUDA(cudaMemcpyAsync(&h, sums, sizeof(double), cudaMemcpyDeviceToHost, C.stream));
  VL_CUDA(cudaStreamSynchronize(C.stream));
  return h;
}

void vadu_diags(Ctx& C, const Factor& F, const double* W, double* Dinv, double* dinv) {
  launch_rows<1, 1, 1, 0, 0>(C, F.pat->n, 1, DiagsBody{F.D.as<double>(), W, Dinv, dinv}, Fin0<0>{});
}

namespace {
struct CountNonPosBody {  // #{W <= 0} (LRAC / eq7 require W > 0)
  const double* W;
  template <int G, int NU, int U, int NR>
  VL_D void run(int64_t s, bool valid, int, int, double (&acc)[NR][NU * U]) const {
    if (valid && !(W[s] > 0.0)) acc[0][0] += 1.0;
  }
};
}  // namespace

namespace {
struct EinvBody {
  int kind;
  const double* W;
  const double* dst;
  double* out;
  template <int G, int NU, int U, int NR>
  VL_D void run(int64_t s, bool valid, int, int, double (&)[NR][NU * U]) const {
    if (valid) out[s] = kind == 1 ? 1.0 / W[s] : 1.0 / (dst[s] + 1.0 / W[s]);
  }
};
}  // namespace

void lowrank_einv(Ctx& C, int64_t n, int kind, const double* W, const double* diag_st, double* einv) {
  if (kind != 1 && kind != 2) fail(kEConfig, "unknown low-rank preconditioner kind");
  if (kind == 2 && diag_st == nullptr) fail(kEConfig, "l2 needs diag(SigmaTilde)");
  launch_rows<1, 1, 1, 0, 0>(C, n, 1, EinvBody{kind, W, diag_st, einv}, Fin0<0>{});
}

double count_nonpos(Ctx& C, int64_t n, const double* W) {
  double* sums = C.dev_scalars.as<double>();
  launch_rows<1, 1, 1, 1, 0>(C, n, 1, CountNonPosBody{W}, CopySums<1>{sums});
  double g;
  read_sums(C, sums, &g, 1);
  return g;
}

void newton_mode(Ctx& C, const Factor& F, const LikSpec& LS, const NewtonCfg& cfg, const double* y, const double* Fv,
                 double* b, double* W, double* d1, double* d3, NewtonOut* out, const LracFactor* lrac) {
  const Pattern& P = *F.pat;
  const int64_t n = P.n;
  const Lik L = make_lik(LS);
  const size_t vb = sizeof(double) * (size_t)n;
  DevBuf rhs, bnew, delta, Dinv, dinv, tmp;
  rhs.alloc(vb); bnew.alloc(vb); delta.alloc(vb); Dinv.alloc(vb); dinv.alloc(vb); tmp.alloc(vb);
  double* sums = C.dev_scalars.as<double>();
  double h[8];
  BView B = bview(F, false);
  ProfScope ps(C, "newton_misc", 0.0);
  VL_CUDA(cudaMemsetAsync(b, 0, vb, C.stream));
  auto derivs = [&](const double* dlt, double step) {
    launch_rows<1, 1, 1, 3, 4>(C, n, 1, DerivsBody{L, y, Fv, b, dlt, step, d1, W, d3, rhs.as<double>()},
                               CopySums<3>{sums});
    read_sums(C, sums, h, 3);
  };
  auto grad_norm = [&]() {
    launch_rows<1, 1, 1, 0, 0>(C, n, 1, ScaleBBody{B, b, Dinv.as<double>(), tmp.as<double>()}, Fin0<0>{});
    launch_rows<1, 1, 1, 1, 1>(C, n, 1, GradNormBody{B, tmp.as<double>(), d1}, CopySums<1>{sums});
    double g;
    read_sums(C, sums, &g, 1);
    return g;
  };
  // Dinv = 1/D is fixed for this factor; d depends on W (recomputed per step)
  derivs(nullptr, 0.0);
  vadu_diags(C, F, W, Dinv.as<double>(), dinv.as<double>());
  double logp = h[0], rn2 = h[1];
  double quad = 0.0;
  double obj = -logp;
  double gnorm = h[2];
  bool converged = false;
  int iters = 0;
  double safety = 1.0;
  SysVadu S{&F, W, Dinv.as<double>(), dinv.as<double>(), precond_pkind(cfg.precond)};
  out->cg_iters.clear();
  int it;
  for (it = 1; it <= cfg.max_iter; ++it) {
    iters = it;
    const double rn = std::sqrt(rn2);
    double tol = cfg.mode_cg_tol;
    if (rn > 0.0) tol = std::min(tol, std::max(safety * 0.25 * gnorm / rn, 1e-14));
    vadu_diags(C, F, W, Dinv.as<double>(), dinv.as<double>());
    if (cfg.precond > 1) precond_dinv(C, F, cfg.precond, W, dinv.as<double>());
    PcgResult pr;
    if (lrac == nullptr && cfg.wb_kind != 2) {
      pcg_vadu(C, S, 1, 1, rhs.as<double>(), bnew.as<double>(), tol, cfg.cg_max_iter, false, &pr);
    } else {
      const bool nonpos = count_nonpos(C, n, W) > 0;
      if (cfg.wb_kind == 1) {
        if (nonpos) fail(kEFactorization, "low-rank preconditioner diagonal part must be positive and finite");
      } else if (nonpos) {
        fail(kECapability,
             "this preconditioner works on SigmaTilde + W^{-1} and needs W > 0 everywhere (eq7 split; log W "
             "undefined); switch to an eq6 preconditioner such as vadu");
      }
      LracPrec Pr;
      if (cfg.wb_kind == 0) {
        lrac_prepare(C, F, *lrac, W, Pr);
      } else {
        lowrank_einv(C, n, cfg.wb_kind, W, cfg.diag_st, tmp.as<double>());
        lowrank_prepare(C, F, cfg.wb_kind == 2 ? nullptr : lrac, W, tmp.as<double>(), cfg.wb_kind == 1 ? 1 : 0, Pr);
      }
      lrac_solve_system(C, Pr, 1, rhs.as<double>(), bnew.as<double>(), tol, cfg.cg_max_iter, &pr);
    }
    out->cg_iters.push_back(pr.iters[0]);
    launch_rows<1, 1, 1, 0, 0>(C, n, 1, DiffBody{bnew.as<double>(), b, delta.as<double>()}, Fin0<0>{});
    double step = 1.0, obj_try = 0.0, quad_try = 0.0;
    bool accepted = false;
    for (int k = 0; k < 11; ++k) {
      launch_rows<1, 1, 1, 2, 0>(C, n, 1, TrialBody{L, B, y, Fv, b, delta.as<double>(), step, Dinv.as<double>()},
                                 CopySums<2>{sums});
      read_sums(C, sums, h, 2);
      quad_try = h[1];
      obj_try = -h[0] + 0.5 * quad_try;
      if (obj_try <= obj + 1e-12 * (1.0 + std::fabs(obj))) {
        accepted = true;
        break;
      }
      step *= 0.5;
    }
    if (!accepted) break;
    const double obj_change = obj - obj_try;
    obj = obj_try;
    quad = quad_try;
    derivs(delta.as<double>(), step);
    logp = h[0];
    rn2 = h[1];
    const double gprev = gnorm;
    gnorm = grad_norm();
    if (gnorm > 0.5 * gprev) safety = std::max(0.2 * safety, 1e-10);
    if (std::getenv("VL_DEBUG_NEWTON"))
      fprintf(stderr, "[newton] it=%d cg_tol=%.3e cg_its=%d step=%.4g obj=%.12g dobj=%.3e gnorm=%.3e\n", it, tol,
              pr.iters[0], step, obj, obj_change, gnorm);
    if (gnorm < cfg.grad_tol && obj_change < cfg.obj_tol * (1.0 + std::fabs(obj))) {
      converged = true;
      break;
    }
  }
  if (it > cfg.max_iter) iters = cfg.max_iter;
  out->logp = logp;
  out->quad = quad;
  out->objective = obj;
  out->iters = iters;
  out->grad_norm = gnorm;
  out->converged = converged ? 1 : 0;
  if (!converged) {
    const double g = grad_norm();
    out->grad_norm = g;
    if (g >= cfg.grad_tol) {
      char buf[200];
      snprintf(buf, sizeof(buf),
               "Newton mode finding did not converge in %d iterations (gradient sup-norm %.2e)", iters, g);
      fail(kEConvergence, buf);
    }
    out->converged = 1;
  }
}

// ---------------------------------------------------------------------------
// Probes
// ---------------------------------------------------------------------------
namespace {

struct SqrtDBody {  // sd = sqrt(W + 1/D)
  const double* D;
  const double* W;
  double* sd;
  template <int G, int NU, int U, int NR>
  VL_D void run(int64_t s, bool valid, int, int, double (&)[NR][NU * U]) const {
    if (valid) sd[s] = sqrt(W[s] + 1.0 / D[s]);
  }
};

struct ProbeZBody {  // Z = B^T (sd o G)
  BView B;
  const double* G;
  const double* sd;
  double* Z;
  int ld;
  template <int G_, int NU, int U, int NR>
  VL_D void run(int64_t s, bool valid, int gl, int t, double (&)[NR][NU * U]) const {
    auto load = [&](int64_t j, int c, double* out) {
      load_unit<U>(G + j * ld + c, out);
      const double f = sd[j];
#pragma unroll
      for (int i = 0; i < U; ++i) out[i] *= f;
    };
    double a[NU * U];
    zero(a);
    gather_Bt<G_, NU, U>(B, s, valid, gl, t, load, a);
    if (!valid) return;
    double g[NU * U];
    load_row<G_, NU, U>(G, ld, s, gl, t, g);
    const double f = sd[s];
#pragma unroll
    for (int i = 0; i < NU * U; ++i) a[i] += f * g[i];
    store_row<G_, NU, U>(Z, ld, s, gl, t, a);
  }
};

struct PsolveRhs {  // V = B^-1 (G / sd);  acc += Z . V
  const double* G;
  const double* sd;
  const double* Z;
  int ld;
  VL_D double rhs(int64_t s, int c, double&) const { return G[s * ld + c] / sd[s]; }
  VL_D void out(int64_t s, int c, double x, double& acc) const { acc += Z[s * ld + c] * x; }
};

struct FactorSumsBody {
  const double* D;
  const double* W;
  const double* dDs;
  const double* dDr;
  template <int G, int NU, int U, int NR>
  VL_D void run(int64_t s, bool valid, int, int, double (&acc)[NR][NU * U]) const {
    if (!valid) return;
    const double Ds = D[s], w = W[s];
    acc[0][0] += log(Ds);
    acc[1][0] += log(w + 1.0 / Ds);
    if (dDs != nullptr) {
      acc[2][0] += dDs[s] / Ds;
      acc[3][0] += dDr[s] / Ds;
      const double den = Ds * (Ds * w + 1.0);
      acc[4][0] += -(dDs[s] / den);
      acc[5][0] += -(dDr[s] / den);
    }
  }
};

}  // namespace

namespace {
struct SqrtInvBody {  // sd = 1/sqrt(dinv) = sqrt(d)
  const double* dinv;
  double* sd;
  template <int G, int NU, int U, int NR>
  VL_D void run(int64_t s, bool valid, int, int, double (&)[NR][NU * U]) const {
    if (valid) sd[s] = 1.0 / sqrt(dinv[s]);
  }
};
// diagonal P: Z = sqrt(d) o G, V = P^-1 Z = Z / d, w_c = z_c . v_c
struct ProbeDiagBody {
  const double* G;
  const double* sd;
  double* Z;
  double* V;
  int ld;
  template <int G_, int NU, int U, int NR>
  VL_D void run(int64_t s, bool valid, int gl, int t, double (&acc)[NR][NU * U]) const {
    if (!valid) return;
    double g[NU * U], z[NU * U], v[NU * U];
    load_row<G_, NU, U>(G, ld, s, gl, t, g);
    const double f = sd[s];
#pragma unroll
    for (int i = 0; i < NU * U; ++i) {
      z[i] = f * g[i];
      v[i] = z[i] / (f * f);
      acc[0][i] += z[i] * v[i];
    }
    store_row<G_, NU, U>(Z, ld, s, gl, t, z);
    store_row<G_, NU, U>(V, ld, s, gl, t, v);
  }
};
}  // namespace

void probes_eq6(Ctx& C, const Factor& F, const double* dinv, int pkind, int t, int ld, const double* G, double* Z,
                double* V, double* w_host) {
  const Pattern& P = *F.pat;
  const int64_t n = P.n;
  DevBuf sd;
  sd.alloc(sizeof(double) * n);
  launch_rows<1, 1, 1, 0, 0>(C, n, 1, SqrtInvBody{dinv, sd.as<double>()}, Fin0<0>{});
  double* sums = C.dev_scalars.as<double>();
  if (t > 256) fail(kECapacity, "too many probe columns per call");
  if (pkind == 1) {
    dispatch_cols(t, ld, [&](auto g, auto nu, auto uu) {
      constexpr int G_ = decltype(g)::value, NU = decltype(nu)::value, U = decltype(uu)::value;
      ProfScope ps(C, "probe_Z", 0.0);
      launch_rows<G_, NU, U, 1, 0>(C, n, t, ProbeDiagBody{G, sd.as<double>(), Z, V, ld}, CopySums<1>{sums});
    });
    read_sums(C, sums, w_host, t);
    return;
  }
  BView B = bview(F, false);
  DepsEll dfw = deps_fwd(F);
  dispatch_cols(t, ld, [&](auto g, auto nu, auto uu) {
    constexpr int G_ = decltype(g)::value, NU = decltype(nu)::value, U = decltype(uu)::value;
    {
      ProfScope ps(C, "probe_Z", bapply_bytes(P, t, 1));
      launch_rows<G_, NU, U, 0, 0>(C, n, t, ProbeZBody{B, G, sd.as<double>(), Z, ld}, Fin0<0>{});
    }
    ProfScope ps(C, "probe_V", bapply_bytes(P, t, 1) + 8.0 * n * t);
    launch_trsv<G_, NU, U, 1>(C, F, true, t, ld, dfw, V, PsolveRhs{G, sd.as<double>(), Z, ld}, CopySums<1>{sums});
  });
  read_sums(C, sums, w_host, t);
}

namespace {
// forward solve of P^-1 z = B^-1 (dinv o B^-T z) with the SLQ weight z_c . v_c fused
struct RhsDinvDotZ {
  const double* y;
  const double* dinv;
  const double* Z;
  int ld;
  VL_D double rhs(int64_t s, int c, double&) const { return y[s * ld + c] * dinv[s]; }
  VL_D void out(int64_t s, int c, double x, double& acc) const { acc += Z[s * ld + c] * x; }
};
// diagonal P: V = dinv o Z, w_c = z_c . v_c
struct GivenDiagBody {
  const double* Z;
  const double* dinv;
  double* V;
  int ld;
  template <int G_, int NU, int U, int NR>
  VL_D void run(int64_t s, bool valid, int gl, int t, double (&acc)[NR][NU * U]) const {
    if (!valid) return;
    double z[NU * U], v[NU * U];
    load_row<G_, NU, U>(Z, ld, s, gl, t, z);
    const double f = dinv[s];
#pragma unroll
    for (int i = 0; i < NU * U; ++i) {
      v[i] = f * z[i];
      if (vl::Cols<G_, NU, U>::col(gl, i) < t) acc[0][i] += z[i] * v[i];
    }
    store_row<G_, NU, U>(V, ld, s, gl, t, v);
  }
};

VL_D uint64_t splitmix64(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

// Rademacher probes: entry (factor row i, column c) = sign bit of
// splitmix64(seed * golden + i * t_glob + c0 + c) -> -1 / +1; written in storage order
__global__ void rademacher_kernel(int64_t n, int t, int ld, int t_glob, int c0, uint64_t seed,
                                  const int32_t* __restrict__ fidx, double* __restrict__ Z) {
  const int64_t tot = n * (int64_t)t;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < tot; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t s = e / t;
    const int c = (int)(e % t);
    const uint64_t key = seed * 0x9E3779B97F4A7C15ull + (uint64_t)fidx[s] * (uint64_t)t_glob + (uint64_t)(c0 + c);
    Z[s * ld + c] = (splitmix64(key) >> 63) ? -1.0 : 1.0;
  }
}
}  // namespace

void rademacher_probes(Ctx& C, const Pattern& P, int t, int t_glob, int c0, uint64_t seed, double* Z) {
  const int64_t tot = P.n * (int64_t)t;
  const int blocks = (int)std::max<int64_t>(1, std::min<int64_t>((tot + 255) / 256, 8LL * C.num_sms));
  rademacher_kernel<<<blocks, 256, 0, C.stream>>>(P.n, t, t, t_glob, c0, seed, P.fidx.as<int32_t>(), Z);
  VL_LAUNCH_CHECK();
}

// Caller-supplied probes Z (laplace.py:340 ProbeSet injection): V = P^-1 Z for the eq6
// sandwich / diagonal preconditioners, w_c = z_c . v_c (iterative.py:268-271)
void probes_given(Ctx& C, const Factor& F, const double* dinv, int pkind, int t, int ld, const double* Z, double* V,
                  double* w_host) {
  const Pattern& P = *F.pat;
  const int64_t n = P.n;
  double* sums = C.dev_scalars.as<double>();
  if (t > 256) fail(kECapacity, "too many probe columns per call");
  if (pkind == 1) {
    dispatch_cols(t, ld, [&](auto g, auto nu, auto uu) {
      constexpr int G_ = decltype(g)::value, NU = decltype(nu)::value, U = decltype(uu)::value;
      launch_rows<G_, NU, U, 1, 0>(C, n, t, GivenDiagBody{Z, dinv, V, ld}, CopySums<1>{sums});
    });
    read_sums(C, sums, w_host, t);
    return;
  }
  DevBuf Y;
  Y.alloc(sizeof(double) * (size_t)n * ld);
  DepsEll dfw = deps_fwd(F);
  DepsCsr dbw{P.tptr.as<int32_t>(), P.tidx.as<int32_t>(), F.valT.as<double>()};
  dispatch_cols(t, ld, [&](auto g, auto nu, auto uu) {
    constexpr int G_ = decltype(g)::value, NU = decltype(nu)::value, U = decltype(uu)::value;
    ProfScope ps(C, "probe_given", 2.0 * bapply_bytes(P, t, 1));
    launch_trsv<G_, NU, U, 0>(C, F, false, t, ld, dbw, Y.as<double>(), TrsvPlain{Z, ld}, Fin0<0>{});
    launch_trsv<G_, NU, U, 1>(C, F, true, t, ld, dfw, V, RhsDinvDotZ{Y.as<double>(), dinv, Z, ld}, CopySums<1>{sums});
  });
  read_sums(C, sums, w_host, t);
}

void probes_vadu(Ctx& C, const Factor& F, const double* W, int t, int ld, const double* G, double* Z, double* V,
                 double* w_host) {
  const Pattern& P = *F.pat;
  const int64_t n = P.n;
  DevBuf sd;
  sd.alloc(sizeof(double) * n);
  launch_rows<1, 1, 1, 0, 0>(C, n, 1, SqrtDBody{F.D.as<double>(), W, sd.as<double>()}, Fin0<0>{});
  BView B = bview(F, false);
  DepsEll dfw = deps_fwd(F);
  double* sums = C.dev_scalars.as<double>();
  if (t > 256) fail(kECapacity, "too many probe columns per call");
  dispatch_cols(t, ld, [&](auto g, auto nu, auto uu) {
    constexpr int G_ = decltype(g)::value, NU = decltype(nu)::value, U = decltype(uu)::value;
    {
      ProfScope ps(C, "probe_Z", bapply_bytes(P, t, 1));
      launch_rows<G_, NU, U, 0, 0>(C, n, t, ProbeZBody{B, G, sd.as<double>(), Z, ld}, Fin0<0>{});
    }
    ProfScope ps(C, "probe_V", bapply_bytes(P, t, 1) + 8.0 * n * t);
    launch_trsv<G_, NU, U, 1>(C, F, true, t, ld, dfw, V,
                              PsolveRhs{G, sd.as<double>(), Z, ld}, CopySums<1>{sums});
  });
  read_sums(C, sums, w_host, t);
}

void factor_sums(Ctx& C, const Factor& F, const double* W, double* out_host) {
  double* sums = C.dev_scalars.as<double>();
  if (F.has_grad) {
    launch_rows<1, 1, 1, 6, 0>(C, F.pat->n, 1,
                               FactorSumsBody{F.D.as<double>(), W, F.dD_sig.as<double>(), F.dD_rho.as<double>()},
                               CopySums<6>{sums});
    read_sums(C, sums, out_host, 6);
  } else {
    launch_rows<1, 1, 1, 2, 0>(C, F.pat->n, 1, FactorSumsBody{F.D.as<double>(), W, nullptr, nullptr},
                               CopySums<2>{sums});
    read_sums(C, sums, out_host, 2);
    for (int i = 2; i < 6; ++i) out_host[i] = 0.0;
  }
}

// ---------------------------------------------------------------------------
// Gradient passes
// ---------------------------------------------------------------------------
namespace {

template <int G>
VL_D double gsum(double v) {
#pragma unroll
  for (int o = 1; o < G; o <<= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Fused: BU, BV, dBU, dBV per row -> per-row control-variate weight and s,
// per-column STE partial sums.
template <bool XI>
struct GradProbeBody {
  BView B;
  const double* dval;
  const double* U_;
  const double* V_;
  const double* D;
  const double* dDs;
  const double* dDr;
  const double* W;
  const double* d3;
  const double* md3x;
  double* s_out;
  int ld;
  int plain;  // preconditioners without a control variate (laplace.py:433-436): c = 0
  template <int G, int NU, int U, int NR>
  VL_D void run(int64_t s, bool valid, int gl, int t, double (&acc)[NR][NU * U]) const {
    constexpr int NC = NU * U;
    double BU[NC], BV[NC], dBU[NC], dBV[NC];
    zero(BU); zero(BV); zero(dBU); zero(dBV);
    const int cs = valid ? B.cnt[s] : 0;
    const int64_t base = (valid ? s : 0) * B.m;
    for (int e = 0; e < cs; ++e) {
      const int32_t j = B.nbr[base + e];
      const double w = B.val[base + e];
      const double dw = dval[base + e];
#pragma unroll
      for (int k = 0; k < NU; ++k) {
        const int c = U * (gl + G * k);
        if (c < t) {
          double uu[U], vv[U];
          load_unit<U>(U_ + (int64_t)j * ld + c, uu);
          load_unit<U>(V_ + (int64_t)j * ld + c, vv);
#pragma unroll
          for (int i = 0; i < U; ++i) {
            BU[U * k + i] += w * uu[i];
            BV[U * k + i] += w * vv[i];
            dBU[U * k + i] += dw * uu[i];
            dBV[U * k + i] += dw * vv[i];
          }
        }
      }
    }
    double us[NC], vs[NC];
    load_row<G, NU, U>(U_, ld, valid ? s : 0, gl, valid ? t : 0, us);
    load_row<G, NU, U>(V_, ld, valid ? s : 0, gl, valid ? t : 0, vs);
    double H[NC], R[NC];
    double sh = 0.0, sr = 0.0;
#pragma unroll
    for (int i = 0; i < NC; ++i) {
      const int c = vl::Cols<G, NU, U>::col(gl, i);
      BU[i] += us[i];
      BV[i] += vs[i];
      const bool on = valid && c < t;
      H[i] = on ? us[i] * vs[i] : 0.0;
      R[i] = on ? BV[i] * BV[i] : 0.0;
      sh += H[i];
      sr += R[i];
    }
    sh = gsum<G>(sh);
    sr = gsum<G>(sr);
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
    svr = gsum<G>(svr);
    scv = gsum<G>(scv);
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
    sm = gsum<G>(sm);
    if (!valid) return;
    const double Ds = D[s], Dinv = 1.0 / Ds, ws = W[s];
    if (gl == 0) {
      const double exact = cw / (ws + Dinv);
      s_out[s] = 0.5 * ((-d3[s]) * (exact + sm / t));
    }
    const double qs = dDs[s] * Dinv * Dinv;
    const double qr = dDr[s] * Dinv * Dinv;
    const double mx = XI ? md3x[s] : 0.0;
#pragma unroll
    for (int i = 0; i < NC; ++i) {
      const int c = vl::Cols<G, NU, U>::col(gl, i);
      if (c >= t) continue;
      acc[0][i] += -(BU[i] * qs * BV[i]);
      acc[1][i] += -(qs * BV[i] * BV[i]);
      acc[2][i] += (dBU[i] * BV[i] + BU[i] * dBV[i]) * Dinv - BU[i] * qr * BV[i];
      acc[3][i] += 2.0 * dBV[i] * BV[i] * Dinv - qr * BV[i] * BV[i] + 2.0 * ws * dBV[i] * BV[i];
      if constexpr (XI) {
        acc[4][i] += mx * us[i] * vs[i];
        acc[5][i] += mx * BV[i] * BV[i];
      }
    }
  }
};

// Probe-sharded variant (multi-GPU): the per-row control-variate statistics
// need all t probes, so they are split into allreduce-able row sums.
//   MODE 1: rowA = [sum_c H, sum_c R] (local columns) + STE column partials
//   MODE 2: rowB = [sum_c (H - hbar)(R - rbar), sum_c (R - rbar)^2] with the
//           global means hbar = rowA/t_glob (rowA already allreduced)
template <int MODE, bool XI>
struct GradSplitBody {
  BView B;
  const double* dval;
  const double* U_;
  const double* V_;
  const double* D;
  const double* dDs;
  const double* dDr;
  const double* W;
  const double* md3x;
  double* rowA;
  double* rowB;
  int tg;
  int ld;
  template <int G, int NU, int U, int NR>
  VL_D void run(int64_t s, bool valid, int gl, int t, double (&acc)[NR][NU * U]) const {
    constexpr int NC = NU * U;
    double BU[NC], BV[NC], dBU[NC], dBV[NC];
    zero(BU); zero(BV); zero(dBU); zero(dBV);
    const int cs = valid ? B.cnt[s] : 0;
    const int64_t base = (valid ? s : 0) * B.m;
    for (int e = 0; e < cs; ++e) {
      const int32_t j = B.nbr[base + e];
      const double w = B.val[base + e];
      const double dw = (MODE == 1) ? dval[base + e] : 0.0;
#pragma unroll
      for (int k = 0; k < NU; ++k) {
        const int c = U * (gl + G * k);
        if (c < t) {
          double uu[U], vv[U];
          load_unit<U>(V_ + (int64_t)j * ld + c, vv);
          if (MODE == 1) load_unit<U>(U_ + (int64_t)j * ld + c, uu);
#pragma unroll
          for (int i = 0; i < U; ++i) {
            BV[U * k + i] += w * vv[i];
            if (MODE == 1) {
              BU[U * k + i] += w * uu[i];
              dBU[U * k + i] += dw * uu[i];
              dBV[U * k + i] += dw * vv[i];
            }
          }
        }
      }
    }
    double us[NC], vs[NC];
    load_row<G, NU, U>(U_, ld, valid ? s : 0, gl, valid ? t : 0, us);
    load_row<G, NU, U>(V_, ld, valid ? s : 0, gl, valid ? t : 0, vs);
    double a = 0.0, b = 0.0;
    double hm = 0.0, rm = 0.0;
    if (MODE == 2 && valid) {
      hm = rowA[2 * s] / tg;
      rm = rowA[2 * s + 1] / tg;
    }
#pragma unroll
    for (int i = 0; i < NC; ++i) {
      const int c = vl::Cols<G, NU, U>::col(gl, i);
      BU[i] += us[i];
      BV[i] += vs[i];
      if (valid && c < t) {
        const double H = us[i] * vs[i], R = BV[i] * BV[i];
        if (MODE == 1) {
          a += H;
          b += R;
        } else {
          a += (H - hm) * (R - rm);
          b += (R - rm) * (R - rm);
        }
      }
    }
    a = gsum<G>(a);
    b = gsum<G>(b);
    if (!valid) return;
    if (gl == 0) {
      double* dst = (MODE == 1) ? rowA : rowB;
      dst[2 * s] = a;
      dst[2 * s + 1] = b;
    }
    if (MODE != 1) return;
    const double Dinv = 1.0 / D[s], ws = W[s];
    const double qs = dDs[s] * Dinv * Dinv;
    const double qr = dDr[s] * Dinv * Dinv;
    const double mx = XI ? md3x[s] : 0.0;
#pragma unroll
    for (int i = 0; i < NC; ++i) {
      const int c = vl::Cols<G, NU, U>::col(gl, i);
      if (c >= t) continue;
      acc[0][i] += -(BU[i] * qs * BV[i]);
      acc[1][i] += -(qs * BV[i] * BV[i]);
      acc[2][i] += (dBU[i] * BV[i] + BU[i] * dBV[i]) * Dinv - BU[i] * qr * BV[i];
      acc[3][i] += 2.0 * dBV[i] * BV[i] * Dinv - qr * BV[i] * BV[i] + 2.0 * ws * dBV[i] * BV[i];
      if constexpr (XI) {
        acc[4][i] += mx * us[i] * vs[i];
        acc[5][i] += mx * BV[i] * BV[i];
      }
    }
  }
};

// MODE 3: s = 0.5 md3 (c/(W + 1/D) + (sumH - c sumR)/t), c = cov/var (ddof 1)
struct GradSplitFinishBody {
  const double* rowA;
  const double* rowB;
  const double* D;
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
    const double exact = cw / (W[s] + 1.0 / D[s]);
    s_out[s] = 0.5 * ((-d3[s]) * (exact + (rowA[2 * s] - cw * rowA[2 * s + 1]) / tg));
  }
};

struct ScalarTermsBody {
  BView B;
  const double* dval;
  const double* b;
  const double* tv;
  const double* D;
  const double* dDs;
  const double* dDr;
  template <int G, int NU, int U, int NR>
  VL_D void run(int64_t s, bool valid, int, int, double (&acc)[NR][NU * U]) const {
    if (!valid) return;
    double Bb = b[s], Bt = tv[s], dBb = 0.0, dBt = 0.0;
    const int cs = B.cnt[s];
    const int64_t base = s * B.m;
    for (int e = 0; e < cs; ++e) {
      const int32_t j = B.nbr[base + e];
      const double w = B.val[base + e], dw = dval[base + e];
      const double bj = b[j], tj = tv[j];
      Bb += w * bj;
      Bt += w * tj;
      dBb += dw * bj;
      dBt += dw * tj;
    }
    const double Dinv = 1.0 / D[s];
    const double qs = dDs[s] * Dinv * Dinv, qr = dDr[s] * Dinv * Dinv;
    acc[0][0] += -(qs * Bb * Bb);
    acc[1][0] += -(Bt * qs * Bb);
    acc[2][0] += 2.0 * dBb * Bb * Dinv - qr * Bb * Bb;
    acc[3][0] += (dBt * Bb + Bt * dBb) * Dinv - Bt * qr * Bb;
  }
};

struct DFBody {
  const double* d1;
  const double* sv;
  const double* W;
  const double* tv;
  const double* X;
  int ld;
  template <int G, int NU, int U, int NR>
  VL_D void run(int64_t s, bool valid, int gl, int t, double (&acc)[NR][NU * U]) const {
    if (!valid) return;
    const double dF = -d1[s] + sv[s] - W[s] * tv[s];
    double x[NU * U];
    load_row<G, NU, U>(X, ld, s, gl, t, x);
#pragma unroll
    for (int i = 0; i < NU * U; ++i) acc[0][i] += x[i] * dF;
  }
};

struct GammaXiBody {
  const double* y;
  const double* Fv;
  const double* b;
  const double* W;
  const double* D;
  const double* tv;
  double* md3x;
  template <int G, int NU, int U, int NR>
  VL_D void run(int64_t s, bool valid, int, int, double (&acc)[NR][NU * U]) const {
    if (!valid) return;
    const double mu = Fv[s] + b[s];
    const double e = y[s] * exp(-mu);
    md3x[s] = e;
    acc[0][0] += log(y[s]) - mu - e;
    acc[1][0] += tv[s] * (-1.0 + e);
    acc[2][0] += e / (W[s] + 1.0 / D[s]);
  }
};

}  // namespace

void grad_probe_pass(Ctx& C, const Factor& F, const double* W, const double* d3, const double* U, const double* V,
                     int t, int ld, double* s_out, double* cols_host, const double* xi_md3, double* xi_cols_host,
                     int plain) {
  if (!F.has_grad) fail(kEConfig, "factor was built without gradient");
  const Pattern& P = *F.pat;
  BView B = bview(F, false);
  double* sums = C.dev_scalars.as<double>();
  if (6 * t > 8192) fail(kECapacity, "too many probe columns per call");
  // bytes: B and dB values + indices once, U and V read once (gathers), s written
  ProfScope ps(C, "grad_pass", 20.0 * ((double)P.nnz_off) + 4.0 * (P.n + 1) + 16.0 * P.n * t + 40.0 * P.n);
  dispatch_cols(t, ld, [&](auto g, auto nu, auto uu) {
    constexpr int G = decltype(g)::value, NU = decltype(nu)::value, U_ = decltype(uu)::value;
    if (xi_md3 == nullptr) {
      launch_rows<G, NU, U_, 4, 0>(C, P.n, t,
                                   GradProbeBody<false>{B, F.dval.as<double>(), U, V, F.D.as<double>(),
                                                        F.dD_sig.as<double>(), F.dD_rho.as<double>(), W, d3, nullptr,
                                                        s_out, ld, plain},
                                   CopySums<4>{sums});
    } else {
      launch_rows<G, NU, U_, 6, 0>(C, P.n, t,
                                   GradProbeBody<true>{B, F.dval.as<double>(), U, V, F.D.as<double>(),
                                                       F.dD_sig.as<double>(), F.dD_rho.as<double>(), W, d3, xi_md3,
                                                       s_out, ld, plain},
                                   CopySums<6>{sums});
    }
  });
  read_sums(C, sums, cols_host, 4 * t);
  if (xi_md3 != nullptr) read_sums(C, sums + 4 * t, xi_cols_host, 2 * t);
}

void grad_probe_pass_split(Ctx& C, const Factor& F, int mode, const double* W, const double* d3, const double* U,
                           const double* V, int t, int ld, int t_glob, double* rowA, double* rowB, double* s_out,
                           double* cols_host, const double* xi_md3, double* xi_cols_host, int plain) {
  if (!F.has_grad) fail(kEConfig, "factor was built without gradient");
  const Pattern& P = *F.pat;
  BView B = bview(F, false);
  double* sums = C.dev_scalars.as<double>();
  ProfScope ps(C, "grad_pass_split", 0.0);
  if (mode == 3) {
    launch_rows<1, 1, 1, 0, 0>(C, P.n, 1,
                               GradSplitFinishBody{rowA, rowB, F.D.as<double>(), W, d3, s_out, t_glob, plain},
                               Fin0<0>{});
    return;
  }
  if (t < 1 || 6 * t > 8192) fail(kECapacity, "invalid probe shard width");
  dispatch_cols(t, ld, [&](auto g, auto nu, auto uu) {
    constexpr int G = decltype(g)::value, NU = decltype(nu)::value, U_ = decltype(uu)::value;
    auto common = [&](auto body_tag) {};
    (void)common;
    if (mode == 1) {
      if (xi_md3 == nullptr) {
        launch_rows<G, NU, U_, 4, 0>(C, P.n, t,
                                     GradSplitBody<1, false>{B, F.dval.as<double>(), U, V, F.D.as<double>(),
                                                             F.dD_sig.as<double>(), F.dD_rho.as<double>(), W,
                                                             nullptr, rowA, rowB, t_glob, ld},
                                     CopySums<4>{sums});
      } else {
        launch_rows<G, NU, U_, 6, 0>(C, P.n, t,
                                     GradSplitBody<1, true>{B, F.dval.as<double>(), U, V, F.D.as<double>(),
                                                            F.dD_sig.as<double>(), F.dD_rho.as<double>(), W, xi_md3,
                                                            rowA, rowB, t_glob, ld},
                                     CopySums<6>{sums});
      }
    } else if (mode == 2) {
      launch_rows<G, NU, U_, 0, 0>(C, P.n, t,
                                   GradSplitBody<2, false>{B, F.dval.as<double>(), U, V, F.D.as<double>(),
                                                           F.dD_sig.as<double>(), F.dD_rho.as<double>(), W, nullptr,
                                                           rowA, rowB, t_glob, ld},
                                   Fin0<0>{});
    } else {
      fail(kEConfig, "unknown split mode");
    }
  });
  if (mode == 1) {
    read_sums(C, sums, cols_host, 4 * t);
    if (xi_md3 != nullptr) read_sums(C, sums + 4 * t, xi_cols_host, 2 * t);
  }
}

void grad_scalar_terms(Ctx& C, const Factor& F, const double* b, const double* tvec, double* out_host) {
  if (!F.has_grad) fail(kEConfig, "factor was built without gradient");
  double* sums = C.dev_scalars.as<double>();
  launch_rows<1, 1, 1, 4, 0>(C, F.pat->n, 1,
                             ScalarTermsBody{bview(F, false), F.dval.as<double>(), b, tvec, F.D.as<double>(),
                                             F.dD_sig.as<double>(), F.dD_rho.as<double>()},
                             CopySums<4>{sums});
  read_sums(C, sums, out_host, 4);
}

void grad_dF(Ctx& C, int64_t n, const double* d1, const double* s, const double* W, const double* tvec,
             const double* X, int p, double* dbeta_host) {
  if (p <= 0) return;
  double* sums = C.dev_scalars.as<double>();
  if (p > 128) fail(kECapacity, "too many fixed-effect columns");
  dispatch_cols(p, p, [&](auto g, auto nu, auto uu) {
    constexpr int G = decltype(g)::value, NU = decltype(nu)::value, U = decltype(uu)::value;
    launch_rows<G, NU, U, 1, 0>(C, n, p, DFBody{d1, s, W, tvec, X, p}, CopySums<1>{sums});
  });
  read_sums(C, sums, dbeta_host, p);
}

void gamma_xi_terms(Ctx& C, const Factor& F, const double* y, const double* Fv, const double* b, const double* W,
                    const double* tvec, double* md3x_out, double* out_host) {
  double* sums = C.dev_scalars.as<double>();
  launch_rows<1, 1, 1, 3, 0>(C, F.pat->n, 1, GammaXiBody{y, Fv, b, W, F.D.as<double>(), tvec, md3x_out},
                             CopySums<3>{sums});
  read_sums(C, sums, out_host, 3);
}

}  // namespace vl
