// Dense fp64 linear algebra of the low-rank (LRAC / Woodbury) paths, hand
// written for sm_100a: a tiled column-major GEMM with optional split-K, a
// diagonal weight along the contraction dimension (C = A diag(w) B) and a
// lower-triangle-only mode (SYRK), plus a blocked lower-triangular inverse
// built on it.  Triangular solves of the Woodbury core and the _lrac_dL chain
// (laplace.py:369-386) are applied as products with explicit triangular
// inverses.  Column-major conventions follow BLAS so call sites read like
// the BLAS calls they replace.
#pragma once

#include "context.h"

namespace vl {

struct Gemm {
  bool ta = false, tb = false;  // op(A) = A^T / op(B) = B^T
  int m = 0, n = 0, k = 0;      // C (m x n) = alpha op(A) (m x k) [diag(kw)] op(B) (k x n) + beta C
  double alpha = 1.0, beta = 0.0;
  const double* A = nullptr;
  int lda = 0;
  const double* B = nullptr;
  int ldb = 0;
  double* C = nullptr;
  int ldc = 0;
  const double* kw = nullptr;   // optional weights along k (length k)
  bool lower = false;           // write only C(i, j) with i >= j (m == n)
};

void dgemm(Ctx& C, const Gemm& g);

// Linv (k x k, column-major, lower) = L^-1 for lower-triangular L; the
// strictly upper parts of Linv are zeroed.
void dtrtri_lower(Ctx& C, int k, const double* L, int ldl, double* Linv, int ldi);

}  // namespace vl
