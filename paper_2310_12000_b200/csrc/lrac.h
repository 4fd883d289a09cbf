// LRAC preconditioner (preconditioners.py:167-214, 288-320; laplace.py:118-153)
// and the eq7 system  A = SigmaTilde + W^-1  (laplace.py:156-182).
#pragma once

#include <vector>

#include "context.h"
#include "pcg.h"

namespace vl {

// Rank-k pivoted Cholesky of the exact covariance, kept with the factor
// (theta-only, laplace.py:128-136).  L: n x k row-major, storage order.
struct LracFactor {
  int k = 0, keff = 0;
  DevBuf L;                 // n x k
  std::vector<int32_t> piv_f;  // pivots, factor order
  DevBuf piv_s;             // pivots, storage order
};

// Low-rank-plus-diagonal preconditioner P = L L^T + diag(e)
// (LowRankPlusDiagonalPreconditioner, preconditioners.py:161-214) for one W:
// W here is 1/e (the Woodbury diagonal): lrac e = 1/W, pchol-precision and
// rowsel e = W, l2 (k = 0) e = diag(SigmaTilde) + 1/W.  Wop is the system's W
// (operator), eq6 selects the system form W + Q (else SigmaTilde + 1/W).
// M = I + L^T diag(1/e) L = Lm Lm^T.
struct LracPrec {
  const Factor* F = nullptr;
  const LracFactor* LF = nullptr;
  const double* W = nullptr;    // 1/e
  const double* Wop = nullptr;  // operator W
  int eq6 = 0;
  DevBuf Lm;                // k x k column-major lower Cholesky factor of M
  DevBuf Lmi;               // Lm^-1 (k x k, column-major, lower)
  DevBuf Minv;              // M^-1 = Lm^-T Lm^-1 (k x k, column-major, symmetric)
  DevBuf own;               // owned 1/e buffer when computed here
  LracFactor empty;         // k = 0 factor for the diagonal-only (l2) form
  double logdetM = 0.0;
  double sumlogW = 0.0;     // sum log(1/e)
};

void lrac_pchol(Ctx& C, const Factor& F, LracFactor& LF, int k, double tol);
void lrac_prepare(Ctx& C, const Factor& F, const LracFactor& LF, const double* W, LracPrec& P);
// general form: LF may be null (k = 0); einv = 1/e (null -> Wop, the lrac case)
void lowrank_prepare(Ctx& C, const Factor& F, const LracFactor* LF, const double* Wop, const double* einv, int eq6,
                     LracPrec& P);
// pivoted Cholesky of the precision B^T D^-1 B (PrecisionAccessor, preconditioners.py:228-246)
void pchol_precision(Ctx& C, const Factor& F, LracFactor& LF, int k, double tol);
// rowsel factor U = B_S^T D_S^-1/2 over the k rows of largest sum_j B_ij^2 / D_i (preconditioners.py:323-335, 372-379)
void rowsel_factor(Ctx& C, const Factor& F, LracFactor& LF, int k);
// diag(SigmaTilde) (vecchia.py:198-212) by batched B^-T solves of identity columns
void diag_sigma_tilde(Ctx& C, const Factor& F, double* out);
// z = P^-1 r for t columns (n x t)
void lrac_apply_inv(Ctx& C, const LracPrec& P, int t, const double* r, double* z);
// PCG on (SigmaTilde + W^-1) U = Bm  (iterative.py:104-178 per column)
void pcg_lrac(Ctx& C, const LracPrec& P, int t, const double* b, double* u, double tol, int max_iter, bool capture,
              PcgResult* out);
// y = SigmaTilde x = B^-1 (D o B^-T x)  (vecchia.py:185-192), t columns
void apply_sigma_tilde(Ctx& C, const Factor& F, int t, const double* x, double* y, double* scratch);
// u = (W + SigmaTilde^-1)^-1 rhs via the eq7 form (laplace.py:176-179)
void lrac_solve_system(Ctx& C, const LracPrec& P, int t, const double* rhs, double* u, double tol, int max_iter,
                       PcgResult* out);

void lrac_free_handles();
// LRAC gradient pieces (laplace.py:369-436, 493-576 eq7 with the LRAC preconditioner):
// s (n, device) = 0.5 dlogdet/dmu; host: hcols/rcols (2 x t: sigma2, rho), dPt (2);
// with md3x (gamma): xicols (2 x t: h_xi, r_xi), xis = [sum G2 m3, sum m3 / W].
void lrac_grad(Ctx& C, const LracPrec& Pr, int t, const double* U, const double* V, const double* d3,
               const double* md3x, double* s_out, double* hcols, double* rcols, double* dPt, double* xicols,
               double* xis, int plain = 0);
// probe-sharded lrac_grad: mode 1 local row sums + per-column outputs, 2 centred sums, 3 s
void lrac_grad_split(Ctx& C, const LracPrec& Pr, int mode, int t, int t_glob, const double* U, const double* V,
                     const double* d3, const double* md3x, double* rowA, double* rowB, double* s_out, double* hcols,
                     double* rcols, double* dPt, double* xicols, double* xis, int plain);
double lrac_sumlogW(Ctx& C, int64_t n, const double* W);
void lrac_probes(Ctx& C, const LracPrec& Pr, int t, const double* Gn, const double* Gk, double* Z, double* V,
                 double* w_host);

}  // namespace vl
