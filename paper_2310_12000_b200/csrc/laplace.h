// Laplace objective on the device: likelihood functors, damped Newton mode
// finding, probe generation, gradient passes.
#pragma once

#include <vector>

#include "context.h"
#include "pcg.h"

namespace vl {

struct LikSpec {
  int family;    // 0 bernoulli-logit, 1 bernoulli-probit, 2 gamma
  double shape;  // gamma shape (xi)
};

struct NewtonCfg {
  double mode_cg_tol;  // min(cg_tol, 1e-4)
  int cg_max_iter;
  int max_iter;
  double grad_tol;
  double obj_tol;
  int precond = 0;  // eq6 variant (precond_dinv); ignored with lrac
  // low-rank-plus-diagonal preconditioners (lrac != nullptr or wb_kind == 2):
  // 0 lrac (eq7, e = 1/W), 1 pchol-precision / rowsel (eq6, e = W), 2 l2 (eq7, k = 0,
  // e = diag(SigmaTilde) + 1/W with diag_st = diag(SigmaTilde))
  int wb_kind = 0;
  const double* diag_st = nullptr;
};

struct NewtonOut {
  double logp = 0, quad = 0, objective = 0, grad_norm = 0;
  int iters = 0;
  int converged = 0;
  std::vector<int> cg_iters;
};

// Damped Newton for b* (laplace.py:204-287).  Device vectors (storage order,
// length n): y, F in; b, W, d1, d3 out.  Throws kEConvergence (state valid).
struct LracFactor;
// lrac != nullptr selects the LRAC preconditioner with the eq7 system
// (laplace.py:118-127 CapabilityError when some W <= 0).
void newton_mode(Ctx& C, const Factor& F, const LikSpec& L, const NewtonCfg& cfg, const double* y,
                 const double* Fv, double* b, double* W, double* d1, double* d3, NewtonOut* out,
                 const LracFactor* lrac = nullptr);

// 1/e of the low-rank-plus-diagonal variants: kind 1: 1/W ; kind 2: 1/(diag_st + 1/W)
void lowrank_einv(Ctx& C, int64_t n, int kind, const double* W, const double* diag_st, double* einv);

// number of entries with W <= 0 (eq7 / LRAC capability check)
double count_nonpos(Ctx& C, int64_t n, const double* W);

// 1/D and 1/(W + 1/D) (VADU diagonal)
void vadu_diags(Ctx& C, const Factor& F, const double* W, double* Dinv, double* dinv);

// eq6 preconditioner variants (preconditioners.py:338-387):
//   0 vadu, 1 l1   P = B^T diag(W + 1/D) B          (sandwich)
//   2 lva          P = B^T diag(1/D) B              (sandwich)
//   3 diag         P = diag(W + diag(B^T D^-1 B))   (diagonal)
//   4 identity     P = I                            (diagonal)
// dinv = 1/d of the sandwich / diagonal; pkind 0 sandwich, 1 diagonal.
void precond_dinv(Ctx& C, const Factor& F, int variant, const double* W, double* dinv);
inline int precond_pkind(int variant) { return variant <= 2 ? 0 : 1; }
double sum_log(Ctx& C, int64_t n, const double* x);
// Z ~ N(0, P) from base normals G, V = P^-1 Z, w_c = z_c . v_c for either kind
// Rademacher probe block (factor-order counter hash, storage-order output), columns c0..c0+t of t_glob
void rademacher_probes(Ctx& C, const Pattern& P, int t, int t_glob, int c0, uint64_t seed, double* Z);
// V = P^-1 Z and w_c = z_c . v_c for caller-supplied probes
void probes_given(Ctx& C, const Factor& F, const double* dinv, int pkind, int t, int ld, const double* Z, double* V,
                  double* w_host);
void probes_eq6(Ctx& C, const Factor& F, const double* dinv, int pkind, int t, int ld, const double* G, double* Z,
                double* V, double* w_host);

// Z = B^T (sqrt(d) o G), V = B^-1 (G / sqrt(d)) = P^-1 Z, w_c = z_c . v_c
// (preconditioners.py:121-122, iterative.py:268-271).  G, Z, V: n x ld.
void probes_vadu(Ctx& C, const Factor& F, const double* W, int t, int ld, const double* G, double* Z, double* V,
                 double* w_host);

// sums over rows: [sum log D, sum log d, sum dD_s/D, sum dD_r/D,
//                  -sum dD_s/(D(DW+1)), -sum dD_r/(D(DW+1))]
void factor_sums(Ctx& C, const Factor& F, const double* W, double* out_host);

// Fused gradient probe pass (laplace.py:389-436 VADU branch and the STE
// h/r terms of laplace.py:493-541 + iterative.py:280-304):
//   s = 0.5 * dlogdet/dmu (n, device),
//   cols (host, 4 x t): h_sigma2, r_sigma2, h_rho, r_rho per probe
//   plus (if xi_md3 != null) 2 x t: h_xi, r_xi with md3x = xi_md3.
void grad_probe_pass(Ctx& C, const Factor& F, const double* W, const double* d3, const double* U, const double* V,
                     int t, int ld, double* s_out, double* cols_host, const double* xi_md3, double* xi_cols_host,
                     int plain = 0);

// Probe-sharded split of grad_probe_pass (modes 1, 2, 3; see laplace.cu).
// rowA/rowB: n x 2 device; between modes the caller allreduces them.
void grad_probe_pass_split(Ctx& C, const Factor& F, int mode, const double* W, const double* d3, const double* U,
                           const double* V, int t, int ld, int t_glob, double* rowA, double* rowB, double* s_out,
                           double* cols_host, const double* xi_md3, double* xi_cols_host, int plain = 0);

// Scalar gradient terms with b and tvec (host out, 4 values):
// [quad_sigma2(b), tvec.dQ_sigma2 b, quad_rho(b), tvec.dQ_rho b]
void grad_scalar_terms(Ctx& C, const Factor& F, const double* b, const double* tvec, double* out_host);

// dF = -d1 + s - W o tvec ;  dbeta = X^T dF  (X: n x p storage order);
// extra (xi): sum(tvec o d2xi) where d2xi = -1 + y e^{-mu} (gamma) if gamma
void grad_dF(Ctx& C, int64_t n, const double* d1, const double* s, const double* W, const double* tvec,
             const double* X, int p, double* dbeta_host);

// Gamma xi terms: [sum(log y - mu - y e^{-mu}), sum(tvec (-1 + y e^{-mu})), sum(md3x / (W + 1/D))]
// and md3x = y e^{-mu} written to md3x_out (n).
void gamma_xi_terms(Ctx& C, const Factor& F, const double* y, const double* Fv, const double* b, const double* W,
                    const double* tvec, double* md3x_out, double* out_host);

}  // namespace vl
