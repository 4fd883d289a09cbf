// Row bodies shared by the kernels: gathers over the rows of B (ELL, storage
// order) and over the children CSR of B^T, with 16-byte column units and a
// 4-way unrolled entry loop (4 x NU independent gathers in flight per lane;
// index/weight loads are uniform across the G lanes of a group -> L1
// broadcast).
#pragma once

#include "common.cuh"
#include "rows.cuh"

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
  int64_t nnzT;         // entries of the children CSR
};

// Strided vector view: x[row * ld + col]
struct VecView {
  const double* x;
  int ld;
};

// acc[i] += sum_e w_e * X[j_e, col(i)] over entries [0, cs) given by idx/wt.
template <int G, int NU, int U, class Idx, class Wt, class Load>
VL_D void gather(int cs, int gl, int t, const Idx& idx, const Wt& wt, const Load& load, double (&acc)[NU * U]) {
  int e = 0;
  for (; e + 4 <= cs; e += 4) {
    int32_t j[4];
    double w[4];
    double v[4][NU * U];
#pragma unroll
    for (int q = 0; q < 4; ++q) { j[q] = idx(e + q); w[q] = wt(e + q); }
#pragma unroll
    for (int q = 0; q < 4; ++q)
#pragma unroll
      for (int k = 0; k < NU; ++k) {
        const int c = U * (gl + G * k);
        if (c < t) load(j[q], c, &v[q][U * k]);
        else
#pragma unroll
          for (int i = 0; i < U; ++i) v[q][U * k + i] = 0.0;
      }
#pragma unroll
    for (int q = 0; q < 4; ++q)
#pragma unroll
      for (int i = 0; i < NU * U; ++i) acc[i] += w[q] * v[q][i];
  }
  for (; e < cs; ++e) {
    const int32_t j = idx(e);
    const double w = wt(e);
#pragma unroll
    for (int k = 0; k < NU; ++k) {
      const int c = U * (gl + G * k);
      if (c < t) {
        double v[U];
        load(j, c, v);
#pragma unroll
        for (int i = 0; i < U; ++i) acc[U * k + i] += w * v[i];
      }
    }
  }
}

// unit loader from a strided vector (read-only path)
template <int U>
struct LoadU {
  const double* x;
  int ld;
  VL_D void operator()(int64_t j, int c, double* out) const { load_unit<U>(x + j * ld + c, out); }
};

// Single-column (t == 1) gathers of rows_kernel: the warp's lanes own 32
// CONSECUTIVE storage rows, whose entries are contiguous in the ELL / CSR
// arrays.  The warp streams that entry range in 256-entry windows with
// coalesced index/value loads (lane = entry) and independent x gathers, parks
// (w, x) pairs in shared memory, and each lane then folds its own row's
// entries in entry order with the same fma chain as gather() -> identical
// results, ~1/3 of the memory transactions of lane-per-row loads.
constexpr int kStreamWin = 256;
#ifndef VL_STREAM_ELL
#define VL_STREAM_ELL 0
#endif
#ifndef VL_STREAM_PROD
#define VL_STREAM_PROD 1
#endif
#ifndef VL_STREAM_PF
#define VL_STREAM_PF 8   // windows ahead (measured on the t = 1 product: 0.114 -> 0.106 ms; 20: 0.110)
#endif
template <class Idx, class Wt, class Load>
VL_D void stream_rows1(int64_t E0, int64_t E1, int64_t b, int64_t e, const Idx& idx, const Wt& wt, const Load& load,
                       double& acc, const int32_t* pf_i = nullptr, const double* pf_w = nullptr, int64_t pf_end = 0) {
  __shared__ double s_w[kRowsThreads / 32][kStreamWin];
  __shared__ double s_x[kRowsThreads / 32][kStreamWin];
  const int lane = threadIdx.x & 31;
  double* sw = s_w[threadIdx.x >> 5];
  double* sx = s_x[threadIdx.x >> 5];
  constexpr int K = kStreamWin / 32;
  for (int64_t w0 = E0; w0 < E1; w0 += kStreamWin) {
    int32_t j[K];
    double wv[K], xv[K];
#if VL_STREAM_PF
    // the window VL_STREAM_PF ahead: its 8 index lines and 16 value lines into L2
    // (entries past E1 belong to the next rows of the stream, read by the next warp)
    const int64_t nw = w0 + (int64_t)VL_STREAM_PF * kStreamWin;
    if (pf_i != nullptr && nw + kStreamWin <= pf_end) {
      if (lane < 8) asm volatile("prefetch.global.L2 [%0];" ::"l"(pf_i + nw + lane * 32));
      else if (lane < 24) asm volatile("prefetch.global.L2 [%0];" ::"l"(pf_w + nw + (lane - 8) * 16));
    }
#endif
#pragma unroll
    for (int k = 0; k < K; ++k) {
      const int64_t g = w0 + k * 32 + lane;
      const bool on = g < E1;
      j[k] = on ? idx(g) : 0;
      wv[k] = on ? wt(g) : 0.0;
    }
#pragma unroll
    for (int k = 0; k < K; ++k) {
      if (w0 + k * 32 + lane < E1) load(j[k], 0, &xv[k]);
      else xv[k] = 0.0;
    }
#if VL_STREAM_PROD
    // products formed in parallel (8 per lane), the lane's fold is one shared
    // load + add per entry of its row (the longest row of the window sets the
    // warp's fold time)
#pragma unroll
    for (int k = 0; k < K; ++k) sw[k * 32 + lane] = wv[k] * xv[k];
    __syncwarp();
    const int64_t lo = b > w0 ? b : w0;
    const int64_t hi = e < w0 + kStreamWin ? e : w0 + kStreamWin;
    for (int64_t q = lo; q < hi; ++q) acc += sw[q - w0];
    __syncwarp();
#else
#pragma unroll
    for (int k = 0; k < K; ++k) {
      sw[k * 32 + lane] = wv[k];
      sx[k * 32 + lane] = xv[k];
    }
    __syncwarp();
    const int64_t lo = b > w0 ? b : w0;
    const int64_t hi = e < w0 + kStreamWin ? e : w0 + kStreamWin;
    for (int64_t q = lo; q < hi; ++q) acc = fma(sw[q - w0], sx[q - w0], acc);
    __syncwarp();
#endif
  }
}

// acc += (off-diagonal of B row s) . X      (B row: ELL, in reference order)
template <int G, int NU, int U, class Load>
VL_D void gather_B(const BView& B, const double* vals, int64_t s, bool valid, int gl, int t, const Load& load,
                   double (&acc)[NU * U]) {
  const int cs = valid ? B.cnt[s] : 0;
  // (fixed-width ELL rows stream fine from L1 lane-per-row; measured faster than stream_rows1)
  if constexpr (G == 1 && NU == 1 && U == 1 && VL_STREAM_ELL) {
    const unsigned vm = __ballot_sync(0xffffffffu, valid);  // valid lanes: a prefix of 32 consecutive rows
    if (vm == 0u) return;
    const int64_t s0 = __shfl_sync(0xffffffffu, s, 0);
    const int64_t m = B.m;
    stream_rows1(
        s0 * m, (s0 + __popc(vm)) * m, valid ? s * m : 0, valid ? s * m + cs : 0,
        [&](int64_t g) { return B.nbr[g]; }, [&](int64_t g) { return vals[g]; }, load, acc[0]);
    return;
  }
  const int32_t* nb = B.nbr + (valid ? s : 0) * B.m;
  const double* vv = vals + (valid ? s : 0) * B.m;
  gather<G, NU, U>(
      cs, gl, t, [&](int e) { return nb[e]; }, [&](int e) { return vv[e]; }, load, acc);
}

// xs + (off-diagonal of B row s) . x for ONE column, accumulated with
// error-free transformations (Ogita-Rump-Oishi Dot2: TwoProduct via fma +
// TwoSum).  B x cancels heavily when x is smooth (O(1) terms, O(sqrt(D))
// result); divided by D (down to ~1e-10 at n = 1e6, rho = 0.02) the plain
// fp64 rounding becomes a 1e-6..1e-5 noise floor in the Newton gradient.
template <class Load>
VL_D double gather_B_dot2(const BView& B, const double* vals, int64_t s, double xs, const Load& load) {
  const int cs = B.cnt[s];
  const int32_t* nb = B.nbr + s * B.m;
  const double* vv = vals + s * B.m;
  double sum = xs, comp = 0.0;
  int e = 0;
  auto add = [&](double w, double x) {
    const double p = w * x;
    const double pe = fma(w, x, -p);
    const double t = sum + p;
    const double bb = t - sum;
    const double se = (sum - (t - bb)) + (p - bb);
    sum = t;
    comp += pe + se;
  };
  for (; e + 4 <= cs; e += 4) {
    const int32_t j0 = nb[e], j1 = nb[e + 1], j2 = nb[e + 2], j3 = nb[e + 3];
    const double w0 = vv[e], w1 = vv[e + 1], w2 = vv[e + 2], w3 = vv[e + 3];
    double x0, x1, x2, x3;
    load(j0, 0, &x0);
    load(j1, 0, &x1);
    load(j2, 0, &x2);
    load(j3, 0, &x3);
    add(w0, x0);
    add(w1, x1);
    add(w2, x2);
    add(w3, x3);
  }
  for (; e < cs; ++e) {
    double x;
    load(nb[e], 0, &x);
    add(vv[e], x);
  }
  return sum + comp;
}

// acc += (column s of B's off-diagonal) . X   (children CSR)
template <int G, int NU, int U, class Load>
VL_D void gather_Bt(const BView& B, int64_t s, bool valid, int gl, int t, const Load& load, double (&acc)[NU * U]) {
  const int e0 = valid ? B.tptr[s] : 0;
  const int cs = valid ? B.tptr[s + 1] - e0 : 0;
  if constexpr (G == 1 && NU == 1 && U == 1) {
    const unsigned vm = __ballot_sync(0xffffffffu, valid);
    if (vm == 0u) return;
    const int nv = __popc(vm);
    const int64_t E0 = __shfl_sync(0xffffffffu, e0, 0);
    const int64_t E1 = __shfl_sync(0xffffffffu, e0 + cs, nv - 1);
    stream_rows1(
        E0, E1, e0, (int64_t)e0 + cs, [&](int64_t g) { return B.tidx[g]; }, [&](int64_t g) { return B.valT[g]; },
        load, acc[0], B.tidx, B.valT, B.nnzT);
    return;
  }
  const int32_t* ti = B.tidx + e0;
  const double* tv = B.valT + e0;
  gather<G, NU, U>(
      cs, gl, t, [&](int e) { return ti[e]; }, [&](int e) { return tv[e]; }, load, acc);
}

template <int NC>
VL_D void zero(double (&a)[NC]) {
#pragma unroll
  for (int k = 0; k < NC; ++k) a[k] = 0.0;
}

// store the lane's columns of row s
template <int G, int NU, int U>
VL_D void store_row(double* y, int ld, int64_t s, int gl, int t, const double (&a)[NU * U]) {
#pragma unroll
  for (int k = 0; k < NU; ++k) {
    const int c = U * (gl + G * k);
    if (c < t) {
      if constexpr (U == 2) *reinterpret_cast<double2*>(y + s * ld + c) = make_double2(a[2 * k], a[2 * k + 1]);
      else y[s * ld + c] = a[k];
    }
  }
}

template <int G, int NU, int U>
VL_D void load_row(const double* x, int ld, int64_t s, int gl, int t, double (&a)[NU * U]) {
#pragma unroll
  for (int k = 0; k < NU; ++k) {
    const int c = U * (gl + G * k);
    if (c < t) load_unit<U>(x + s * ld + c, &a[U * k]);
    else
#pragma unroll
      for (int i = 0; i < U; ++i) a[U * k + i] = 0.0;
  }
}

// ---- plain products ---------------------------------------------------------
struct BodyBx {  // y = B x  (op 0) or y = dB x (op 2: no unit diagonal)
  BView B;
  const double* vals;
  const double* x;
  double* y;
  int ld;
  int unit_diag;
  template <int G, int NU, int U, int NR>
  VL_D void run(int64_t s, bool valid, int gl, int t, double (&)[NR][NU * U]) const {
    double a[NU * U];
    zero(a);
    gather_B<G, NU, U>(B, vals, s, valid, gl, t, LoadU<U>{x, ld}, a);
    if (!valid) return;
    if (unit_diag) {
      double xs[NU * U];
      load_row<G, NU, U>(x, ld, s, gl, t, xs);
#pragma unroll
      for (int i = 0; i < NU * U; ++i) a[i] += xs[i];
    }
    store_row<G, NU, U>(y, ld, s, gl, t, a);
  }
};

struct BodyBtx {  // y = B^T x
  BView B;
  const double* x;
  double* y;
  int ld;
  template <int G, int NU, int U, int NR>
  VL_D void run(int64_t s, bool valid, int gl, int t, double (&)[NR][NU * U]) const {
    double a[NU * U];
    zero(a);
    gather_Bt<G, NU, U>(B, s, valid, gl, t, LoadU<U>{x, ld}, a);
    if (!valid) return;
    double xs[NU * U];
    load_row<G, NU, U>(x, ld, s, gl, t, xs);
#pragma unroll
    for (int i = 0; i < NU * U; ++i) a[i] += xs[i];
    store_row<G, NU, U>(y, ld, s, gl, t, a);
  }
};

// ---- plain triangular solves -------------------------------------------------
struct TrsvPlain {
  const double* b;
  int ld;
  VL_D double rhs(int64_t s, int c, double&) const { return b[s * ld + c]; }
  VL_D void out(int64_t, int, double, double&) const {}
  VL_D void prefetch(int64_t s) const { asm volatile("prefetch.global.L2 [%0];" ::"l"(b + s * ld)); }
};

}  // namespace vl
