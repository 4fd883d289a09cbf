// Preconditioned CG on the Laplace system with many right-hand sides.
#pragma once

#include <vector>

#include "context.h"

namespace vl {

// VADU / eq6 system:  A = diag(W) + B^T D^-1 B,  P^-1 = B^-1 diag(1/d) B^-T, d = W + 1/D
struct SysVadu {
  const Factor* F;
  const double* W;     // n
  const double* Dinv;  // n   1/D
  const double* dinv;  // n   1/d of the preconditioner (vadu: 1/(W + 1/D))
  int pkind = 0;       // 0: P = B^T diag(d) B (K3/K4 triangular solves); 1: P = diag(d)
};

struct PcgResult {
  std::vector<int> iters;       // per column
  std::vector<int> converged;   // per column
  std::vector<double> res;      // final residual norms
  std::vector<double> alpha;    // [iters_max x t] history (row l = iteration l)
  std::vector<double> beta;     // [iters_max x t]
  int max_iters = 0;
};

// Solve A U = Bm (n x t, leading dimension ld) column by column to
// ||r_c|| < tol ||b_c||; U written to `u` (n x ld).  Mirrors
// iterative.py:104-178 per column (same stopping rule, breakdown checks and
// Lanczos coefficient capture).
void pcg_vadu(Ctx& C, const SysVadu& S, int t, int ld, const double* b, double* u, double tol, int max_iter,
              bool capture, PcgResult* out);

}  // namespace vl
