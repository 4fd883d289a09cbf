// Row bodies shared by the kernels: gathers over the rows of B (ELL, storage
// order) and over the children CSR of B^T.
#pragma once

#include "common.cuh"

namespace vl {

// Read-only view of B's structure + values.
struct BView {
  const int32_t* nbr;   // n*m
  const int32_t* cnt;   // n
  const double* val;    // n*m   off-diagonal values of B (row i: -A_i)
  const int32_t* tptr;  // n+1   children CSR (B^T rows)
  const int32_t* tidx;
  const double* valT;
  int m;
};

// acc[k] += sum_e B[s, j_e] * load(j_e, c)   (off-diagonal part only)
template <int G, int NC, class Load>
VL_D void gather_B(const BView& B, int64_t s, int gl, int t, const Load& load, double (&acc)[NC]) {
  const int cs = B.cnt[s];
  const int32_t* nb = B.nbr + s * B.m;
  const double* vv = B.val + s * B.m;
  for (int e = 0; e < cs; ++e) {
    const int32_t j = nb[e];
    const double w = vv[e];
#pragma unroll
    for (int k = 0; k < NC; ++k) {
      int c = gl + G * k;
      if (c < t) acc[k] += w * load(j, c);
    }
  }
}

// acc[k] += sum_{children i of s} B[i, s] * load(i, c)
template <int G, int NC, class Load>
VL_D void gather_Bt(const BView& B, int64_t s, int gl, int t, const Load& load, double (&acc)[NC]) {
  const int e0 = B.tptr[s], e1 = B.tptr[s + 1];
  for (int e = e0; e < e1; ++e) {
    const int32_t i = B.tidx[e];
    const double w = B.valT[e];
#pragma unroll
    for (int k = 0; k < NC; ++k) {
      int c = gl + G * k;
      if (c < t) acc[k] += w * load(i, c);
    }
  }
}

struct LoadVec {
  const double* x;
  int t;
  VL_D double operator()(int64_t j, int c) const { return x[j * t + c]; }
};

// ---- plain products ---------------------------------------------------------
struct BodyBx {  // y = B x
  BView B;
  const double* x;
  double* y;
  template <int G, int NC, int NR>
  VL_D void run(int64_t s, bool valid, int gl, int t, double (&)[NR][NC]) const {
    if (!valid) return;
    double a[NC];
#pragma unroll
    for (int k = 0; k < NC; ++k) a[k] = 0.0;
    gather_B<G, NC>(B, s, gl, t, LoadVec{x, t}, a);
#pragma unroll
    for (int k = 0; k < NC; ++k) {
      int c = gl + G * k;
      if (c < t) y[s * t + c] = x[s * t + c] + a[k];
    }
  }
};

struct BodyBtx {  // y = B^T x
  BView B;
  const double* x;
  double* y;
  template <int G, int NC, int NR>
  VL_D void run(int64_t s, bool valid, int gl, int t, double (&)[NR][NC]) const {
    if (!valid) return;
    double a[NC];
#pragma unroll
    for (int k = 0; k < NC; ++k) a[k] = 0.0;
    gather_Bt<G, NC>(B, s, gl, t, LoadVec{x, t}, a);
#pragma unroll
    for (int k = 0; k < NC; ++k) {
      int c = gl + G * k;
      if (c < t) y[s * t + c] = x[s * t + c] + a[k];
    }
  }
};

// dB x with dB sharing B's pattern (no diagonal)
struct BodyDBx {
  BView dB;
  const double* x;
  double* y;
  template <int G, int NC, int NR>
  VL_D void run(int64_t s, bool valid, int gl, int t, double (&)[NR][NC]) const {
    if (!valid) return;
    double a[NC];
#pragma unroll
    for (int k = 0; k < NC; ++k) a[k] = 0.0;
    gather_B<G, NC>(dB, s, gl, t, LoadVec{x, t}, a);
#pragma unroll
    for (int k = 0; k < NC; ++k) {
      int c = gl + G * k;
      if (c < t) y[s * t + c] = a[k];
    }
  }
};

// ---- plain triangular solves -------------------------------------------------
struct TrsvPlain {
  const double* b;
  int t;
  VL_D double rhs(int64_t s, int c, double&) const { return b[s * t + c]; }
  VL_D void out(int64_t, int, double, double&) const {}
};

}  // namespace vl
