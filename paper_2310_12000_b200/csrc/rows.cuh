// Row-parallel kernel frameworks over the n x ld row-major (storage order)
// vectors of the Vecchia path.
//
// Column mapping.  A row is owned by a group of G lanes.  Columns are moved
// in units of U doubles (U = 2 -> 16-byte vector loads when ld is even);
// lane gl of a group owns units u = gl + G*k (k < NU), i.e. columns
// c = U*u + i (i < U).  Per-lane column arrays have NC = NU*U entries and
// entry a[U*k + i] is column U*(gl + G*k) + i.
//
//  * rows_kernel : no dependencies (products with B, B^T, dB, elementwise
//                  passes).
//  * trsv_kernel : dependency-driven (sync-free) triangular solve.  Rows are
//                  visited in level order; a row polls the VALUES of the rows
//                  it reads (x is pre-filled with a NaN sentinel), warp-
//                  converged, so there is no per-row flag, fence or
//                  per-level barrier.  Launched cooperatively (all CTAs
//                  co-resident) with a static level-order assignment, which
//                  makes the spin deadlock-free.
//
// Both end with a DETERMINISTIC column reduction (NR quantities per column):
// fixed-order warp -> block -> grid (last-block) sums, no float atomics.
#pragma once

#include <cuda_runtime.h>

#include <type_traits>
#include <utility>

#include "common.cuh"

namespace vl {

constexpr int kRowsThreads = 256;

// ---- column-unit helpers ---------------------------------------------------
template <int G, int NU, int U>
struct Cols {
  static constexpr int NC = NU * U;
  VL_D static int col(int gl, int i) { return U * (gl + G * (i / U)) + (i % U); }
};

template <int U>
VL_D void load_unit(const double* p, double* out) {
  if constexpr (U == 2) {
    double2 v = __ldg(reinterpret_cast<const double2*>(p));
    out[0] = v.x;
    out[1] = v.y;
  } else {
    out[0] = __ldg(p);
  }
}

// L2-coherent polling load of one unit (bypasses L1).
template <int U>
VL_D void ld_cg_unit(const double* p, double* out) {
  if constexpr (U == 2) {
    double a, b;
    asm volatile("ld.global.cg.v2.f64 {%0, %1}, [%2];" : "=d"(a), "=d"(b) : "l"(p));
    out[0] = a;
    out[1] = b;
  } else {
    double a;
    // (ld.relaxed.gpu / ld.cv / ld.volatile measured identical on B200)
    asm volatile("ld.global.cg.f64 %0, [%1];" : "=d"(a) : "l"(p));
    out[0] = a;
  }
}

// Optional fused product of the backward solve (Body::kPsum): alongside
// y = B^-T rhs the rows also emit p = B^T (om o y), i.e.
//   p_s = om_s y_s + sum_{e in deps(s)} w_e om_dep(e) y_dep(e),
// from the same dependency gathers (om = body.om, a per-row weight).  Such a
// body's rhs() is pure; the row's epilogue calls
//   body.fin_row(s, c, x, rhs, psum)   (stores p = om_s x + psum and,
//                                       optionally, the rhs value itself)
// after x_s is published, and the head path calls body.keep_rhs(s, c, rhs).
#ifndef VL_PS_NOGATHER
#define VL_OMLOAD(p) __ldg(p)
#else  // diagnostic: fused product without the om gathers (wrong values)
#define VL_OMLOAD(p) 1.0
#endif
template <class T, class = void>
struct PsumOf : std::false_type {};
template <class T>
struct PsumOf<T, std::void_t<decltype(T::kPsum)>> : std::bool_constant<T::kPsum> {};

template <int NR>
struct Fin0 {
  VL_D void operator()(const double* /*sums*/, int /*t*/) const {}
};

// acc[r][i] for columns Cols::col(gl, i).  MAXMASK bit r set -> max-reduce.
template <int G, int NU, int U, int NR, int MAXMASK>
VL_D void block_reduce_cols(double (&acc)[NR > 0 ? NR : 1][NU * U], int t, double* out, double* sh) {
  if constexpr (NR == 0) return;
  constexpr int NC = NU * U;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
#pragma unroll
  for (int r = 0; r < NR; ++r)
#pragma unroll
    for (int i = 0; i < NC; ++i)
#pragma unroll
      for (int o = G; o < 32; o <<= 1) {
        double other = __shfl_xor_sync(0xffffffffu, acc[r][i], o);
        acc[r][i] = ((MAXMASK >> r) & 1) ? fmax(acc[r][i], other) : acc[r][i] + other;
      }
  // lane gl (< G) of warp w writes its NC entries
  if (lane < G) {
#pragma unroll
    for (int r = 0; r < NR; ++r)
#pragma unroll
      for (int i = 0; i < NC; ++i) sh[((warp * NR + r) * NC + i) * G + lane] = acc[r][i];
  }
  __syncthreads();
  for (int idx = threadIdx.x; idx < NR * t; idx += blockDim.x) {
    const int r = idx / t, c = idx - r * t;
    const int u = c / U, ii = c % U;
    const int gl = u % G, k = u / G;
    const int i = U * k + ii;
    double s = 0.0;
    for (int w = 0; w < nwarps; ++w) {
      double v = sh[((w * NR + r) * NC + i) * G + gl];
      s = ((MAXMASK >> r) & 1) ? fmax(s, v) : s + v;
    }
    out[idx] = s;
  }
}

// Grid-level finalisation by the last CTA to finish (fixed block order).
// `total_slots` partial slots may be filled by several stream-ordered
// launches (the solve segments); the CTA drawing the last ticket reduces all.
template <int NR, int MAXMASK, class Fin>
VL_D void grid_finalize(const double* partials, unsigned* counter, int t, const Fin& fin, double* sh,
                        int total_slots = -1) {
  if constexpr (NR == 0) return;
  const int nb = total_slots > 0 ? total_slots : (int)gridDim.x;
  __threadfence();
  __syncthreads();
  __shared__ unsigned s_ticket;
  if (threadIdx.x == 0) s_ticket = atomicAdd(counter, 1u);
  __syncthreads();
  if (s_ticket != (unsigned)nb - 1) return;
  __threadfence();
  // one warp per output: lane l folds slots l, l+32, ... in order, then a
  // fixed xor tree -> deterministic, and ~nb/32 independent loads per lane
  // instead of one thread walking nb dependent-latency loads
  const int lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  for (int idx = threadIdx.x >> 5; idx < NR * t; idx += nw) {
    const int r = idx / t;
    const bool mx = (MAXMASK >> r) & 1;
    double s = 0.0;
    int b = lane;
    for (; b + 96 < nb; b += 128) {
      const double v0 = __ldcg(partials + (size_t)b * NR * t + idx);
      const double v1 = __ldcg(partials + (size_t)(b + 32) * NR * t + idx);
      const double v2 = __ldcg(partials + (size_t)(b + 64) * NR * t + idx);
      const double v3 = __ldcg(partials + (size_t)(b + 96) * NR * t + idx);
      s = mx ? fmax(fmax(fmax(fmax(s, v0), v1), v2), v3) : (((s + v0) + v1) + v2) + v3;
    }
    for (; b < nb; b += 32) {
      const double v = __ldcg(partials + (size_t)b * NR * t + idx);
      s = mx ? fmax(s, v) : s + v;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double other = __shfl_xor_sync(0xffffffffu, s, o);
      s = mx ? fmax(s, other) : s + other;
    }
    if (lane == 0) sh[idx] = s;
  }
  __syncthreads();
  fin(sh, t);
  __syncthreads();
  if (threadIdx.x == 0) *counter = 0u;  // ready for the next launch using this slot
}

template <int G, int NU, int U, int NR>
constexpr size_t red_smem_bytes(int threads, int t) {
  size_t a = (size_t)(threads / 32) * (NR > 0 ? NR : 1) * NU * U * G * sizeof(double);
  size_t b = (size_t)(NR > 0 ? NR : 1) * t * sizeof(double);
  return a > b ? a : b;
}

// ---------------------------------------------------------------------------
// Body concept for rows_kernel:
//   template <int G, int NU, int U, int NR>
//   VL_D void run(int64_t s, bool valid, int gl, int t, double (&acc)[NR][NU*U]) const;
// run() is called by every lane of the warp (valid == false for tail rows)
// so bodies may use warp shuffles.
// ---------------------------------------------------------------------------
// Row run [r0, r1) of CTA b of `grid`: contiguous equal-row chunks (multiple
// of GPW), or, with a weight pointer wptr (n + 1, nondecreasing; the children
// CSR pointer of a B^T pass), equal shares of the weight wptr[s] + s so rows
// with hundreds of children (the first points of a random order) do not pile
// up in one CTA.
template <int GPW>
VL_D void row_run(int64_t n, const int32_t* __restrict__ wptr, int64_t b, int64_t grid, int64_t& r0, int64_t& r1,
                  int wpb = 1) {
  if (wptr != nullptr) {
    const int64_t W = (int64_t)wptr[n] + n;
    auto first_row = [&](int64_t target) {  // smallest s with wptr[s] + s >= target
      int64_t lo = 0, hi = n;
      while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if ((int64_t)wptr[mid] + mid < target) lo = mid + 1;
        else hi = mid;
      }
      return lo;
    };
    // run boundaries on multiples of GPW (warp-aligned rows for the t = 1 streaming gathers)
    r0 = first_row(W * b / grid) / GPW * GPW;
    r1 = b + 1 == grid ? n : first_row(W * (b + 1) / grid) / GPW * GPW;
  } else {
    // a multiple of one row group per warp of the CTA: every warp gets the
    // same number of groups (no idle warps at the closing block reduction)
    const int64_t unit = (int64_t)GPW * wpb;
    int64_t chunk = (n + grid - 1) / grid;
    chunk = (chunk + unit - 1) / unit * unit;
    r0 = b * chunk;
    r1 = r0 + chunk < n ? r0 + chunk : n;
    if (r0 > n) r0 = n;
  }
}

template <int G, int NU, int U, int NR, int MAXMASK, class Body, class Fin>
__global__ void __launch_bounds__(kRowsThreads) rows_kernel(int64_t n, int t, Body body, Fin fin,
                                                            double* __restrict__ partials,
                                                            unsigned* __restrict__ counter,
                                                            const int* __restrict__ gate,
                                                            const int32_t* __restrict__ wptr = nullptr) {
  if (gate != nullptr && *((volatile const int*)gate) == 0) return;
  extern __shared__ double rsh[];
  constexpr int GPW = 32 / G;
  constexpr int NRR = NR > 0 ? NR : 1;
  const int lane = threadIdx.x & 31;
  const int gl = lane % G;
  const int gi = lane / G;
  // Block-contiguous row chunks: each CTA sweeps a compact run of storage rows
  // (a spatial patch in Hilbert order), so neighbour rows gathered by
  // adjacent rows are reused from L1 instead of re-fetched from L2.
  const int wib = threadIdx.x >> 5, wpb = blockDim.x >> 5;
  int64_t r0, r1;
  row_run<GPW>(n, wptr, blockIdx.x, gridDim.x, r0, r1, wpb);
  double acc[NRR][NU * U];
#pragma unroll
  for (int r = 0; r < NRR; ++r)
#pragma unroll
    for (int i = 0; i < NU * U; ++i) acc[r][i] = 0.0;
  for (int64_t s0 = r0 + (int64_t)wib * GPW; s0 < r1; s0 += (int64_t)wpb * GPW) {
    const int64_t s = s0 + gi;
    body.template run<G, NU, U, NRR>(s, s < r1, gl, t, acc);
  }
  if constexpr (NR > 0) {
    block_reduce_cols<G, NU, U, NR, MAXMASK>(acc, t, partials + (size_t)blockIdx.x * NR * t, rsh);
    grid_finalize<NR, MAXMASK>(partials, counter, t, fin, rsh);
  }
}

// SM-local variant for gather bodies over spatially ordered rows (t > 1):
// ONE CTA of kLocalThreads per SM sweeps one contiguous run of storage rows
// (a spatial patch) with its warps interleaved row by row, so the whole SM
// works on one narrow window of rows at a time and the neighbour rows its
// gathers touch are L1 hits (the window's rows were just read or are read by
// the neighbouring warps).  With 8 independent CTAs per SM each SM juggles 8
// windows whose union overflows L1 (and, across the chip, L2): measured on
// the kNN factor at t = 64, X was re-read 2x (B x) to 10x (B^T x) from HBM.
// Used for the plain products (vl_spmm): B X at t = 16 0.30 -> 0.22 ms; the
// reducing probe / gradient passes measured slower with it (their reduction
// scratch at 1024 threads eats the L1 carve-out) and keep rows_kernel.
constexpr int kLocalThreads = 1024;
template <int G, int NU, int U, int NR, int MAXMASK, class Body, class Fin>
__global__ void __launch_bounds__(kLocalThreads, 1) rows_local_kernel(int64_t n, int t, Body body, Fin fin,
                                                                      double* __restrict__ partials,
                                                                      unsigned* __restrict__ counter,
                                                                      const int* __restrict__ gate,
                                                                      const int32_t* __restrict__ wptr) {
  if (gate != nullptr && *((volatile const int*)gate) == 0) return;
  extern __shared__ double rsh[];
  constexpr int GPW = 32 / G;
  constexpr int NRR = NR > 0 ? NR : 1;
  const int lane = threadIdx.x & 31;
  const int gl = lane % G;
  const int gi = lane / G;
  const int wib = threadIdx.x >> 5, wpb = blockDim.x >> 5;
  int64_t r0, r1;
  row_run<GPW>(n, wptr, blockIdx.x, gridDim.x, r0, r1, wpb);
  double acc[NRR][NU * U];
#pragma unroll
  for (int r = 0; r < NRR; ++r)
#pragma unroll
    for (int i = 0; i < NU * U; ++i) acc[r][i] = 0.0;
  for (int64_t s0 = r0 + (int64_t)wib * GPW; s0 < r1; s0 += (int64_t)wpb * GPW) {
    const int64_t s = s0 + gi;
    body.template run<G, NU, U, NRR>(s, s < r1, gl, t, acc);
  }
  if constexpr (NR > 0) {
    block_reduce_cols<G, NU, U, NR, MAXMASK>(acc, t, partials + (size_t)blockIdx.x * NR * t, rsh);
    grid_finalize<NR, MAXMASK>(partials, counter, t, fin, rsh);
  }
}

// ---------------------------------------------------------------------------
// Dependency-driven triangular solve (value-as-flag).
//   x_s = rhs(s,c) - sum_{e in deps(s)} w_e * x_{dep(e)}
// `order` lists storage rows in level order, each level padded with -1 to a
// multiple of 32, so the rows of one warp-iteration are always independent.
// Body concept:
//   VL_D double rhs(int64_t s, int c, double& racc) const;
//   VL_D void   out(int64_t s, int c, double x, double& racc) const;
// ---------------------------------------------------------------------------
constexpr unsigned long long kSentinel = 0xFFFFFFFFFFFFFFFFull;

VL_D bool is_sentinel(double v) { return (unsigned long long)__double_as_longlong(v) == kSentinel; }
VL_D double sanitize(double v) { return is_sentinel(v) ? __longlong_as_double(0x7ff8000000000000ll) : v; }

struct DepsEll {
  const int32_t* nbr;
  const int32_t* cnt;
  const double* val;
  int m;
  VL_D int count(int64_t s) const { return cnt[s]; }
  VL_D int64_t base(int64_t s) const { return s * m; }
  VL_D int32_t idx(int64_t b) const { return nbr[b]; }
  VL_D double w(int64_t b) const { return val[b]; }
  VL_D const void* iaddr(int64_t b) const { return nbr + b; }
  VL_D const void* vaddr(int64_t b) const { return val + b; }
};
struct DepsCsr {
  const int32_t* ptr;
  const int32_t* ind;
  const double* val;
  VL_D int count(int64_t s) const { return ptr[s + 1] - ptr[s]; }
  VL_D int64_t base(int64_t s) const { return ptr[s]; }
  VL_D int32_t idx(int64_t b) const { return ind[b]; }
  VL_D double w(int64_t b) const { return val[b]; }
  VL_D const void* iaddr(int64_t b) const { return ind + b; }
  VL_D const void* vaddr(int64_t b) const { return val + b; }
};
// children CSR + per-entry folded weights val2[e] = val[e] * om[ind[e]] of a
// fused backward product (streamed with the values instead of gathered)
struct DepsCsrW2 {
  const int32_t* ptr;
  const int32_t* ind;
  const double* val;
  const double* val2;
  VL_D int count(int64_t s) const { return ptr[s + 1] - ptr[s]; }
  VL_D int64_t base(int64_t s) const { return ptr[s]; }
  VL_D int32_t idx(int64_t b) const { return ind[b]; }
  VL_D double w(int64_t b) const { return val[b]; }
  VL_D double w2(int64_t b) const { return val2[b]; }
  VL_D const void* iaddr(int64_t b) const { return ind + b; }
  VL_D const void* vaddr(int64_t b) const { return val + b; }
};
// Column-unit solves over the children CSR (B^T: heavy-tailed dependency
// counts) take 8-entry gather batches at 3 CTAs/SM; over the ELL (B, <= m
// entries) 4-entry batches at 4 CTAs/SM (measured at t = 16 / 50 / 64).
template <class Deps>
constexpr bool csr_deps() {
  return !std::is_same<Deps, DepsEll>::value;
}
template <class T, class = void>
struct HasW2 : std::false_type {};
template <class T>
struct HasW2<T, std::void_t<decltype(std::declval<T>().w2(0))>> : std::true_type {};

// One solve row per group: rhs, dependency gather (optionally polling the
// sentinel), epilogue and store.  Called by every lane of the warp.
#ifndef VL_LANEMETA
#define VL_LANEMETA 1
#endif
template <int G, int NU, int U, bool POLL, class Deps, class Body>
VL_D void trsv_row(int64_t p, int64_t pend_, int t, int ld, const int32_t* __restrict__ order, const Deps& deps,
                   double* __restrict__ x, const Body& body, unsigned smax, long long* __restrict__ tstamp, int gl,
                   double (&acc0)[NU * U]) {
  constexpr int NC = NU * U;
#ifndef VL_BATCH2
#define VL_BATCH2 4
#endif
#ifndef VL_BATCH2C
#define VL_BATCH2C 8
#endif
  constexpr int BATCH = (NC == 1) ? 32 : (NC == 2 ? (csr_deps<Deps>() ? VL_BATCH2C : VL_BATCH2) : 8);
  using CL = Cols<G, NU, U>;
  constexpr bool PS = PsumOf<Body>::value;
  const int32_t so = (p < pend_) ? order[p] : -1;
  const bool valid = so >= 0;
  const int64_t s = valid ? so : 0;
  double xs[NC], ps[NC], rh[NC];
  auto take_rhs = [&]() {
#pragma unroll
    for (int i = 0; i < NC; ++i) {
      const int c = CL::col(gl, i);
      xs[i] = (valid && c < t) ? body.rhs(s, c, acc0[i]) : 0.0;
      rh[i] = xs[i];
    }
  };
#pragma unroll
  for (int i = 0; i < NC; ++i) ps[i] = 0.0;
#ifndef VL_RHS_LATE
  take_rhs();  // (taking it after the first gathers measured slower at t = 50)
#endif
  const int cs = valid ? deps.count(s) : 0;
  const int64_t b0 = valid ? deps.base(s) : 0;
  const int cmax = (int)__reduce_max_sync(0xffffffffu, (unsigned)cs);
  // Lane-parallel metadata (VL_LANEMETA): the G lanes of a row load G
  // consecutive (index, weight) entries in one coalesced round and the batches
  // take them by shuffle, so a batch's gathers do not wait behind a dependent
  // index load (one metadata round trip per G entries instead of per batch).
  constexpr bool LM = VL_LANEMETA && G >= BATCH && (G % BATCH) == 0;
  int32_t jl = 0;
  double wl = 0.0, ol = 0.0;
  for (int e0 = 0; e0 < cmax; e0 += BATCH) {
    int32_t j[BATCH];
    double w[BATCH], o[BATCH];
    double v[BATCH][NC];
    if constexpr (LM) {
      if (e0 % G == 0) {
        const int e = e0 + gl;
        const bool on = e < cs;
        jl = on ? deps.idx(b0 + e) : 0;
        wl = on ? deps.w(b0 + e) : 0.0;
        if constexpr (PS) {
          if constexpr (HasW2<Deps>::value) ol = on ? deps.w2(b0 + e) : 0.0;
          else ol = on ? wl * VL_OMLOAD(body.om + jl) : 0.0;
        }
      }
#pragma unroll
      for (int q = 0; q < BATCH; ++q) {
        const int src = (e0 + q) % G;
        j[q] = __shfl_sync(0xffffffffu, jl, src, G);
        w[q] = __shfl_sync(0xffffffffu, wl, src, G);
        if constexpr (PS) o[q] = __shfl_sync(0xffffffffu, ol, src, G);
      }
    } else {
#pragma unroll
      for (int q = 0; q < BATCH; ++q) {
        const bool on = e0 + q < cs;
        j[q] = on ? deps.idx(b0 + e0 + q) : 0;
        w[q] = on ? deps.w(b0 + e0 + q) : 0.0;
      }
      if constexpr (PS) {
#pragma unroll
        for (int q = 0; q < BATCH; ++q) {
          const bool on = e0 + q < cs;
          if constexpr (HasW2<Deps>::value) o[q] = on ? deps.w2(b0 + e0 + q) : 0.0;
          else o[q] = on ? w[q] * VL_OMLOAD(body.om + j[q]) : 0.0;
        }
      }
    }
#pragma unroll
    for (int q = 0; q < BATCH; ++q)
#pragma unroll
      for (int k = 0; k < NU; ++k) {
        const int c = U * (gl + G * k);
        if (e0 + q < cs && c < t) {
          ld_cg_unit<U>(x + (int64_t)j[q] * ld + c, &v[q][U * k]);
        } else {
#pragma unroll
          for (int i = 0; i < U; ++i) v[q][U * k + i] = 0.0;
        }
      }
#ifdef VL_RHS_LATE
    if (e0 == 0) take_rhs();
#endif
    if constexpr (POLL) {
      // warp-converged polling: the whole warp re-polls its pending entries together
      unsigned ns = 8;
      for (;;) {
        bool pend = false;
#pragma unroll
        for (int q = 0; q < BATCH; ++q)
#pragma unroll
          for (int i = 0; i < NC; ++i) pend |= is_sentinel(v[q][i]);
        if (!__any_sync(0xffffffffu, pend)) break;
        if (smax) {
          __nanosleep(ns);
          ns = ns < smax ? ns * 2 : smax;
        }
#pragma unroll
        for (int q = 0; q < BATCH; ++q)
#pragma unroll
          for (int k = 0; k < NU; ++k) {
            bool pk = false;
#pragma unroll
            for (int i = 0; i < U; ++i) pk |= is_sentinel(v[q][U * k + i]);
            if (pk) ld_cg_unit<U>(x + (int64_t)j[q] * ld + U * (gl + G * k), &v[q][U * k]);
          }
      }
    }
#pragma unroll
    for (int q = 0; q < BATCH; ++q)
#pragma unroll
      for (int i = 0; i < NC; ++i) {
        xs[i] -= w[q] * v[q][i];
        if constexpr (PS) ps[i] += o[q] * v[q][i];
      }
  }
#ifdef VL_RHS_LATE
  if (cmax == 0) take_rhs();
#endif
  if (valid) {
#pragma unroll
    for (int k = 0; k < NU; ++k) {
      const int c = U * (gl + G * k);
      if (c < t) {
        double* dst = x + s * ld + c;
        if constexpr (U == 2) {
          __stcg(reinterpret_cast<double2*>(dst), make_double2(sanitize(xs[2 * k]), sanitize(xs[2 * k + 1])));
        } else {
          __stcg(dst, sanitize(xs[k]));
        }
      }
    }
    // epilogue after the store: its loads are off the dependency chain
#pragma unroll
    for (int i = 0; i < NC; ++i) {
      const int c = CL::col(gl, i);
      if (c < t) body.out(s, c, xs[i], acc0[i]);
    }
    if constexpr (PS) {
#pragma unroll
      for (int i = 0; i < NC; ++i) {
        const int c = CL::col(gl, i);
        if (c < t) body.fin_row(s, c, xs[i], rh[i], ps[i]);
      }
    }
    if (tstamp != nullptr && gl == 0) {
      long long g;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g));
      tstamp[s] = g;
    }
  }
}

// Single-column row per lane with per-lane early completion: every lane runs
// the same converged loop (one batch of 32 dependencies at a time), but a lane
// stores its row as soon as ITS dependencies are in, instead of waiting for
// the slowest row of the warp.  Without this, a row of level l+1 effectively
// waits for the slowest of ~32 x deg rows of level l (a per-level barrier with
// tail latency); with it, each row waits only for its own dependencies.
// xs -= sum_q w[q] v[q] over one batch.  VL_TREE_SUM = 0: the entries in order
// (one dependent fma chain of B); 1: four interleaved partial sums folded
// pairwise (chain of B/4 + 2), a fixed order as well.
// xs -= sum_q w[q] v[q] over one batch: the entries in order (one dependent
// fma chain of B), or, with TREE, four interleaved partial sums folded
// pairwise (chain of B/4 + 2; a fixed order as well).  Measured on the t = 1
// PCG: forward solve 0.371 -> 0.354 ms; the backward solve (fused product
// children CSR, two batches per item) 0.402 -> 0.431 ms, so it keeps the chain.
#ifndef VL_TREE_SUM
#define VL_TREE_SUM 1
#endif
template <int B, bool TREE>
VL_D void fold_batch(const double (&w)[B], const double (&v)[B], double& xs) {
  if constexpr (TREE && VL_TREE_SUM) {
    double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
#pragma unroll
    for (int q = 0; q < B; q += 4) {
      a0 = fma(w[q], v[q], a0);
      a1 = fma(w[q + 1], v[q + 1], a1);
      a2 = fma(w[q + 2], v[q + 2], a2);
      a3 = fma(w[q + 3], v[q + 3], a3);
    }
    xs -= (a0 + a1) + (a2 + a3);
  } else {
#pragma unroll
    for (int q = 0; q < B; ++q) xs -= w[q] * v[q];
  }
}

#ifndef VL_POLL_ONE
#define VL_POLL_ONE 0
#endif
template <class Deps, class Body>
VL_D void trsv_row1(int64_t p, int64_t pend_, const int32_t* __restrict__ order, const Deps& deps,
                    double* __restrict__ x, const Body& body, unsigned smax, long long* __restrict__ tstamp,
                    double& acc0) {
  constexpr int B = 32;
  const int32_t so = (p < pend_) ? order[p] : -1;
  const bool valid = so >= 0;
  const int64_t s = valid ? so : 0;
  constexpr bool PS = PsumOf<Body>::value;
  double xs = 0.0, rh = 0.0;  // rhs taken after the first gathers are issued
  double ps = 0.0;
  int plast = -1;  // first entry of the row's last batch (still in registers at the end)
  const int cs = valid ? deps.count(s) : 0;
  const int64_t b0 = valid ? deps.base(s) : 0;
#ifdef VL_TS_EXT
  long long rounds = 0;
  if (tstamp != nullptr && valid) {
    long long g;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g));
    tstamp[VL_TS_EXT + s] = g;
  }
#endif
  int e0 = 0;
  int32_t j[B];
  double w[B], v[B];
#pragma unroll
  for (int q = 0; q < B; ++q) {
    const bool on = q < cs;
    j[q] = on ? deps.idx(b0 + q) : 0;
    w[q] = on ? deps.w(b0 + q) : 0.0;
  }
#pragma unroll
  for (int q = 0; q < B; ++q) {
    if (q < cs) ld_cg_unit<1>(x + (int64_t)j[q], &v[q]);
    else v[q] = 0.0;
  }
  if (valid) xs = rh = body.rhs(s, 0, acc0);
  bool done = !valid;
  unsigned ns = 8;
  int pq = -1;
  for (;;) {
    if (!done) {
      bool pend = false;
#pragma unroll
      for (int q = 0; q < B; ++q) pend |= is_sentinel(v[q]);
#ifdef VL_TS_EXT
      ++rounds;
      if (!pend && tstamp != nullptr) {
        long long g;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g));
        tstamp[2LL * VL_TS_EXT + s] = g;
        tstamp[3LL * VL_TS_EXT + s] = rounds;
      }
#endif
      if (!pend) {
        fold_batch<B, !csr_deps<Deps>()>(w, v, xs);
        const int eb = e0;
        e0 += B;
        if (e0 >= cs) {
          __stcg(x + s, sanitize(xs));
          body.out(s, 0, xs, acc0);
          if constexpr (PS) plast = eb;
          if (tstamp != nullptr) {
            long long g;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g));
            tstamp[s] = g;
          }
          done = true;
        } else {
          if constexpr (PS) {
#pragma unroll
            for (int q = 0; q < B; ++q)
              if (eb + q < cs) ps += (w[q] * VL_OMLOAD(body.om + j[q])) * v[q];
          }
#pragma unroll
          for (int q = 0; q < B; ++q) {
            const bool on = e0 + q < cs;
            j[q] = on ? deps.idx(b0 + e0 + q) : 0;
            w[q] = on ? deps.w(b0 + e0 + q) : 0.0;
          }
#pragma unroll
          for (int q = 0; q < B; ++q) {
            if (e0 + q < cs) ld_cg_unit<1>(x + (int64_t)j[q], &v[q]);
            else v[q] = 0.0;
          }
          pq = -1;
        }
      }
    }
    if (__all_sync(0xffffffffu, done)) break;
    if (smax) {
      __nanosleep(ns);
      ns = ns < smax ? ns * 2 : smax;
    }
    if (!done) {
#if VL_POLL_ONE
      // Re-poll only one pending dependency (pq) while it is pending; once it
      // has arrived, re-poll every still-pending one in a single round.  Keeps
      // the L2 request rate of thousands of waiting warps low.
      bool pq_pending = false;
#pragma unroll
      for (int q = 0; q < B; ++q)
        if (q == pq && is_sentinel(v[q])) pq_pending = true;
      if (pq_pending) {
#pragma unroll
        for (int q = 0; q < B; ++q)
          if (q == pq) ld_cg_unit<1>(x + (int64_t)j[q], &v[q]);
      } else {
        int nq = -1;
#pragma unroll
        for (int q = 0; q < B; ++q)
          if (is_sentinel(v[q])) {
            ld_cg_unit<1>(x + (int64_t)j[q], &v[q]);
            nq = nq < 0 ? q : nq;
          }
        pq = nq;
      }
#else
#pragma unroll
      for (int q = 0; q < B; ++q)
        if (is_sentinel(v[q])) ld_cg_unit<1>(x + (int64_t)j[q], &v[q]);
#endif
    }
  }
  if constexpr (PS) {
    // fused B^T(om o y) of the row: once per item, after the warp's poll loop,
    // so the om gathers never stall lanes that are still waiting
    if (valid && plast >= 0) {
#pragma unroll
      for (int q = 0; q < B; ++q)
        if (plast + q < cs) ps += (w[q] * VL_OMLOAD(body.om + j[q])) * v[q];
    }
    if (valid) body.fin_row(s, 0, xs, rh, ps);
  }
}

// Coalesced dependency slab of the light single-RHS items (Pattern::Slabs).
struct Slab {
  const uint32_t* off;
  const uint32_t* w;
  const int32_t* idx;
  const double* val;
  // VL_FRONT: running count of completed single-RHS items (all launches of the context) and
  // the count at this launch's start; a waiting item backs off by its distance to the count
  unsigned* front = nullptr;
  unsigned fbase = 0;
};
#ifndef VL_FRONT
#define VL_FRONT 0
#endif
#ifndef VL_GATHER_CA
#define VL_GATHER_CA 1   // measured: B^-1 0.351 -> 0.344 ms, B^-T 0.401 -> 0.392 ms, bit-identical
#endif
#ifndef VL_FRONT_D0
#define VL_FRONT_D0 96      // items ahead of the completed count that poll at full rate
#endif
#ifndef VL_FRONT_NS
#define VL_FRONT_NS 4       // back-off per item of distance beyond D0 (ns)
#endif
#ifndef VL_FRONT_MAX
#define VL_FRONT_MAX 1500   // back-off cap (ns)
#endif

// trsv_row1 over the item's slab: the 32 lanes read entry e of their rows as
// one 128-byte (index) and one 256-byte (value) transaction, instead of 32
// scattered row segments; padded entries have idx -1 / value 0.  Same
// per-lane early completion and the same summation order as trsv_row1.
template <class Body, bool TREE>
VL_D void trsv_row1s(int64_t p, int64_t pend_, const int32_t* __restrict__ order, uint32_t off, int wk,
                     const Slab& sl, int lane, double* __restrict__ x, const Body& body, unsigned smax,
                     long long* __restrict__ tstamp, double& acc0, int32_t so_in = -2, unsigned my = 0u) {
  constexpr int B = 32;
  const int32_t so = so_in != -2 ? so_in : ((p < pend_) ? order[p] : -1);
  const bool valid = so >= 0;
  const int64_t s = valid ? so : 0;
  constexpr bool PS = PsumOf<Body>::value;
  double xs = 0.0, rh = 0.0;  // rhs taken after the first gathers are issued
  double ps = 0.0;
  int plast = -1;  // first entry of the row's last batch (still in registers at the end)
#ifdef VL_TS_EXT
  long long rounds = 0;
  if (tstamp != nullptr && valid) {
    long long g;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g));
    tstamp[VL_TS_EXT + s] = g;
  }
#endif
  const int32_t* ip = sl.idx + (int64_t)off * 32 + lane;
  const double* vp = sl.val + (int64_t)off * 32 + lane;
  int e0 = 0;
  int32_t j[B];
  double w[B], v[B];
#pragma unroll
  for (int q = 0; q < B; ++q) {
    const bool on = q < wk;
    j[q] = on ? __ldg(ip + q * 32) : -1;
    w[q] = on ? __ldg(vp + q * 32) : 0.0;
  }
#ifdef VL_TS_EXT
  if (tstamp != nullptr && valid && j[0] >= -1) {  // slab entries arrived
    long long g;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g));
    tstamp[4LL * VL_TS_EXT + s] = g;
  }
#endif
  // First gather round.  VL_GATHER_CA: through L1 (ld.global.ca).  x entries are written once
  // (sentinel -> value), so a cached VALUE is final; a cached sentinel only costs one round of
  // the L2-coherent polls below.  L1 is invalidated at every launch boundary.
#pragma unroll
  for (int q = 0; q < B; ++q) {
#if VL_GATHER_CA
    if (j[q] >= 0) asm volatile("ld.global.ca.f64 %0, [%1];" : "=d"(v[q]) : "l"(x + (int64_t)j[q]));
#else
    if (j[q] >= 0) ld_cg_unit<1>(x + (int64_t)j[q], &v[q]);
#endif
    else v[q] = 0.0;
  }
  if (valid) xs = rh = body.rhs(s, 0, acc0);
  bool done = !valid;
  unsigned ns = 8;
#if VL_FRONT
  unsigned fcount = my, fnext = 0u;  // first round: distance unknown -> regular back-off
#endif
  for (;;) {
    if (!done) {
      bool pend = false;
#pragma unroll
      for (int q = 0; q < B; ++q) pend |= is_sentinel(v[q]);
#ifdef VL_TS_EXT
      ++rounds;
      if (!pend && tstamp != nullptr) {
        long long g;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g));
        tstamp[2LL * VL_TS_EXT + s] = g;
        tstamp[3LL * VL_TS_EXT + s] = rounds;
      }
#endif
      if (!pend) {
        fold_batch<B, TREE>(w, v, xs);
        const int eb = e0;
        e0 += B;
        if (e0 >= wk) {
          __stcg(x + s, sanitize(xs));
          body.out(s, 0, xs, acc0);
          if constexpr (PS) plast = eb;
          if (tstamp != nullptr) {
            long long g;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g));
            tstamp[s] = g;
          }
          done = true;
        } else {
          if constexpr (PS) {
#pragma unroll
            for (int q = 0; q < B; ++q)
              if (j[q] >= 0) ps += (w[q] * VL_OMLOAD(body.om + j[q])) * v[q];
          }
#pragma unroll
          for (int q = 0; q < B; ++q) {
            const bool on = e0 + q < wk;
            j[q] = on ? __ldg(ip + (e0 + q) * 32) : -1;
            w[q] = on ? __ldg(vp + (e0 + q) * 32) : 0.0;
          }
#pragma unroll
          for (int q = 0; q < B; ++q) {
            if (j[q] >= 0) ld_cg_unit<1>(x + (int64_t)j[q], &v[q]);
            else v[q] = 0.0;
          }
        }
      }
    }
    if (__all_sync(0xffffffffu, done)) break;
#if VL_FRONT
    if (sl.front != nullptr) {
      // distance of this item to the completed count as read in the previous round
      const int dist = (int)(my - fcount);
      if (dist > VL_FRONT_D0) {
        const int bo = (dist - VL_FRONT_D0) * VL_FRONT_NS;
        __nanosleep(bo < VL_FRONT_MAX ? bo : VL_FRONT_MAX);
      } else if (smax) {
        __nanosleep(ns);
        ns = ns < smax ? ns * 2 : smax;
      }
      unsigned f = 0u;
      if (lane == 0) asm volatile("ld.global.cg.u32 %0, [%1];" : "=r"(f) : "l"(sl.front));
      fnext = f;
    } else
#endif
    if (smax) {
      __nanosleep(ns);
      ns = ns < smax ? ns * 2 : smax;
    }
    if (!done) {
#pragma unroll
      for (int q = 0; q < B; ++q)
        if (is_sentinel(v[q])) ld_cg_unit<1>(x + (int64_t)j[q], &v[q]);
    }
#if VL_FRONT
    if (sl.front != nullptr) fcount = __shfl_sync(0xffffffffu, fnext, 0);
#endif
  }
  if constexpr (PS) {
    // fused B^T(om o y) of the row: once per item, after the warp's poll loop,
    // so the om gathers never stall lanes that are still waiting
    if (valid && plast >= 0) {
#pragma unroll
      for (int q = 0; q < B; ++q)
        if (j[q] >= 0) ps += (w[q] * VL_OMLOAD(body.om + j[q])) * v[q];
    }
    if (valid) body.fin_row(s, 0, xs, rh, ps);
  }
}

struct TrsvLaunch {
  int64_t p0, p1;          // position range (thick) ; unused by thin
  int L0, L1;              // level range (thin)
  const int32_t* lptr;     // device level pointer (thin)
  int slot_base, total_slots;
};

// Thick segment: grid-wide sync-free over positions [p0, p1).
#ifndef VL_PS_MINB
#define VL_PS_MINB 4
#endif
#ifndef VL_MINB_ELL
#define VL_MINB_ELL 4
#endif
#ifndef VL_MINB_CSR
#define VL_MINB_CSR 3
#endif
template <int U, class Body, class Deps>
constexpr int trsv_min_blocks() {
  return U == 2 ? (csr_deps<Deps>() ? VL_MINB_CSR : (PsumOf<Body>::value ? VL_PS_MINB : VL_MINB_ELL)) : 1;
}
template <int G, int NU, int U, int NR, class Deps, class Body, class Fin>
__global__ void __launch_bounds__(kRowsThreads, (trsv_min_blocks<U, Body, Deps>())) trsv_kernel(TrsvLaunch L, int t, int ld,
                                                            const int32_t* __restrict__ order, Deps deps,
                                                            double* __restrict__ x, Body body, Fin fin,
                                                            double* __restrict__ partials,
                                                            unsigned* __restrict__ counter,
                                                            const int* __restrict__ gate, unsigned smax,
                                                            long long* __restrict__ tstamp) {
  if (gate != nullptr && *((volatile const int*)gate) == 0) return;
  extern __shared__ double rsh[];
  constexpr int GPW = 32 / G;
  constexpr int NC = NU * U;
  constexpr int NRR = NR > 0 ? NR : 1;
  const int lane = threadIdx.x & 31;
  const int gl = lane % G;
  const int gi = lane / G;
  const int64_t gwarp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  double acc[NRR][NC];
#pragma unroll
  for (int r = 0; r < NRR; ++r)
#pragma unroll
    for (int i = 0; i < NC; ++i) acc[r][i] = 0.0;
  for (int64_t pbase = L.p0 + gwarp * GPW; pbase < L.p1; pbase += nwarps * GPW)
    trsv_row<G, NU, U, true>(pbase + gi, L.p1, t, ld, order, deps, x, body, smax, tstamp, gl, acc[0]);
  if constexpr (NR > 0) {
    block_reduce_cols<G, NU, U, NR, 0>(acc, t, partials + (size_t)(L.slot_base + blockIdx.x) * NR * t, rsh);
    grid_finalize<NR, 0>(partials, counter, t, fin, rsh, L.total_slots);
  }
}

// Single right-hand side: work items in level order.  A light item is a
// 32-row chunk of one level (thread per row); a heavy item (bit 31 set) is
// one row solved warp-per-row with the lanes over its dependencies (rows of
// thin levels / rows with many children), then a shuffle reduction.
constexpr uint32_t kHeavyBit = 0x80000000u;
#ifndef VL_CARRY
#define VL_CARRY 0
#endif
template <class T, class = void>
struct HasPrefetch : std::false_type {};
template <class T>
struct HasPrefetch<T, std::void_t<decltype(std::declval<const T&>().prefetch(0))>> : std::true_type {};
VL_D void prefetch_l2(const void* p) { asm volatile("prefetch.global.L2 [%0];" ::"l"(p)); }
#ifndef VL_PREFETCH
#define VL_PREFETCH 1
#endif
#ifndef VL_HPREFETCH
#define VL_HPREFETCH 0
#endif

#ifndef VL_HPOLL_THR
#define VL_HPOLL_THR 0
#endif
#ifndef VL_HPOLL_NS
#define VL_HPOLL_NS 100
#endif
template <int NR, class Deps, class Body, class Fin>
__global__ void __launch_bounds__(kRowsThreads) trsv1_kernel(int64_t nitems, int64_t npos,
                                                             const uint32_t* __restrict__ items,
                                                             const int32_t* __restrict__ order, Deps deps,
                                                             double* __restrict__ x, Body body, Fin fin,
                                                             double* __restrict__ partials,
                                                             unsigned* __restrict__ counter,
                                                             const int* __restrict__ gate, unsigned smax,
                                                             long long* __restrict__ tstamp, int slot_base,
                                                             int total_slots, Slab sl) {
  if (gate != nullptr && *((volatile const int*)gate) == 0) {
#if VL_FRONT
    if (sl.front != nullptr && blockIdx.x == 0 && threadIdx.x == 0) atomicAdd(sl.front, (unsigned)nitems);
#endif
    return;
  }
  extern __shared__ double rsh[];
  constexpr int NRR = NR > 0 ? NR : 1;
  constexpr int HB = 8;  // deps per lane per heavy round (256 per warp)
  const int lane = threadIdx.x & 31;
  const int64_t gwarp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  double acc[NRR][1];
#pragma unroll
  for (int r = 0; r < NRR; ++r) acc[r][0] = 0.0;
  // Two-deep item pipeline: while item i is processed, the descriptors of
  // item i + 2W are in flight and the structure of item i + W (its order
  // entries and slab lines) is prefetched into L2, so a warp reaching its next
  // item finds the dependent-load chain mostly in L2 instead of HBM.
  // light item: d = first position, (o, w) = slab columns; heavy item:
  // d = row | kHeavyBit, o = base of its dependencies, w = their count
  auto desc = [&](int64_t i, uint32_t& d, uint32_t& o, uint32_t& w) {
    if (i < nitems) {
      d = __ldg(items + i);
      o = __ldg(sl.off + i);
      w = __ldg(sl.w + i);
    } else {
      d = kHeavyBit; o = 0u; w = 0u;
    }
  };
  uint32_t c_d, c_o, c_w, n_d, n_o, n_w;
  desc(gwarp, c_d, c_o, c_w);
  desc(gwarp + nwarps, n_d, n_o, n_w);
#if VL_CARRY
  // the lane's row of the current / next light item, loaded one item ahead
  // (takes the order -> row load off the item's dependent-load chain), and the
  // next item's right-hand-side lines prefetched into L2 through the body hook
  auto row_of = [&](uint32_t d) -> int32_t {
    if (d & kHeavyBit) return -1;
    const int64_t p = (int64_t)d + lane;
    return p < npos ? __ldg(order + p) : -1;
  };
  int32_t c_s = row_of(c_d), n_s = row_of(n_d);
#endif
  for (int64_t it = gwarp; it < nitems; it += nwarps) {
    const uint32_t item = c_d;
    const uint32_t off = c_o, wk = c_w;
#if VL_CARRY
    const int32_t so = c_s;
    if constexpr (HasPrefetch<Body>::value) {
      if (it + nwarps < nitems && n_s >= 0) body.prefetch(n_s);
    }
#endif
    if (VL_HPREFETCH && it + nwarps < nitems && (n_d & kHeavyBit)) {
      // next heavy item: its first round of dependency indices / values
      const int64_t nb = n_o;
      const int ne = (int)min(n_w, (uint32_t)(32 * HB));
      if (lane * 32 < ne) asm volatile("prefetch.global.L2 [%0];" ::"l"(deps.iaddr(nb + lane * 32)));
      if (lane * 16 < ne) asm volatile("prefetch.global.L2 [%0];" ::"l"(deps.vaddr(nb + lane * 16)));
    }
    if (VL_PREFETCH && sl.idx != nullptr && it + nwarps < nitems && !(n_d & kHeavyBit)) {
#if !VL_CARRY
      asm volatile("prefetch.global.L2 [%0];" ::"l"(order + n_d + lane));
#endif
      for (uint32_t l = lane; l < 3 * n_w; l += 32) {
        const char* a = l < n_w ? reinterpret_cast<const char*>(sl.idx + ((int64_t)n_o + l) * 32)
                                : reinterpret_cast<const char*>(sl.val + (int64_t)n_o * 32) + (int64_t)(l - n_w) * 128;
        asm volatile("prefetch.global.L2 [%0];" ::"l"(a));
      }
    }
    c_d = n_d; c_o = n_o; c_w = n_w;
    desc(it + 2 * nwarps, n_d, n_o, n_w);
#if VL_CARRY
    c_s = n_s;
    n_s = row_of(n_d);
#endif
    if (!(item & kHeavyBit)) {
      if (sl.idx != nullptr)
#if VL_CARRY
        trsv_row1s<Body, !csr_deps<Deps>()>((int64_t)item + lane, npos, order, off, (int)wk, sl, lane, x, body, smax,
                                            tstamp, acc[0][0], so, sl.fbase + (unsigned)it);
#else
        trsv_row1s<Body, !csr_deps<Deps>()>((int64_t)item + lane, npos, order, off, (int)wk, sl, lane, x, body, smax,
                                            tstamp, acc[0][0], -2, sl.fbase + (unsigned)it);
#endif
      else
        trsv_row1((int64_t)item + lane, npos, order, deps, x, body, smax, tstamp, acc[0][0]);
#if VL_FRONT
      if (sl.front != nullptr && lane == 0) asm volatile("red.global.add.u32 [%0], 1;" ::"l"(sl.front) : "memory");
#endif
      continue;
    }
    const int64_t s = (int64_t)(item & ~kHeavyBit);
    const int cs = (int)wk;
    const int64_t b0 = (int64_t)off;
    constexpr bool PS = PsumOf<Body>::value;
    double part = 0.0, part2 = 0.0, rv = 0.0;
    for (int e0 = 0; e0 < cs; e0 += 32 * HB) {
      int32_t j[HB];
      double w[HB], v[HB], o[HB];
#pragma unroll
      for (int q = 0; q < HB; ++q) {
        const int e = e0 + q * 32 + lane;
        const bool on = e < cs;
        j[q] = on ? deps.idx(b0 + e) : 0;
        w[q] = on ? deps.w(b0 + e) : 0.0;
        if (on) ld_cg_unit<1>(x + (int64_t)j[q], &v[q]);
        else v[q] = 0.0;
        if constexpr (PS) o[q] = on ? w[q] * VL_OMLOAD(body.om + j[q]) : 0.0;
      }
      if (e0 == 0 && lane == 0) rv = body.rhs(s, 0, acc[0][0]);
      unsigned ns = 8;
      for (;;) {
        bool pend = false;
#pragma unroll
        for (int q = 0; q < HB; ++q) pend |= is_sentinel(v[q]);
#if VL_HPOLL_THR > 0
        // a row still missing many dependencies is far from the front: back off, so its polls
        // do not load the L2 path of the rows one hop from completion
        const unsigned pm = __ballot_sync(0xffffffffu, pend);
        if (!pm) break;
        if (__popc(pm) > VL_HPOLL_THR) __nanosleep(VL_HPOLL_NS);
        else if (smax) {
          __nanosleep(ns);
          ns = ns < smax ? ns * 2 : smax;
        }
#else
        if (!__any_sync(0xffffffffu, pend)) break;
        if (smax) {
          __nanosleep(ns);
          ns = ns < smax ? ns * 2 : smax;
        }
#endif
#pragma unroll
        for (int q = 0; q < HB; ++q)
          if (is_sentinel(v[q])) ld_cg_unit<1>(x + (int64_t)j[q], &v[q]);
      }
#pragma unroll
      for (int q = 0; q < HB; ++q) {
        part += w[q] * v[q];
        if constexpr (PS) part2 += o[q] * v[q];
      }
    }
    if (cs == 0 && lane == 0) rv = body.rhs(s, 0, acc[0][0]);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
    if constexpr (PS) {
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) part2 += __shfl_xor_sync(0xffffffffu, part2, o);
    }
    if (lane == 0) {
      const double xs = rv - part;
      __stcg(x + s, sanitize(xs));
      body.out(s, 0, xs, acc[0][0]);
      if constexpr (PS) body.fin_row(s, 0, xs, rv, part2);
      if (tstamp != nullptr) {
        long long g;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g));
        tstamp[s] = g;
      }
#if VL_FRONT
      if (sl.front != nullptr) asm volatile("red.global.add.u32 [%0], 1;" ::"l"(sl.front) : "memory");
#endif
    }
  }
  if constexpr (NR > 0) {
    block_reduce_cols<1, 1, 1, NR, 0>(acc, 1, partials + (size_t)(slot_base + blockIdx.x) * NR, rsh);
    grid_finalize<NR, 0>(partials, counter, 1, fin, rsh, total_slots);
  }
}

constexpr int kThinThreads = 1024;

// Thin segment: ONE CTA walks levels [L0, L1) with a barrier per level (no
// polling: every dependency is in an earlier level or an earlier segment).
template <int G, int NU, int U, int NR, class Deps, class Body, class Fin>
__global__ void __launch_bounds__(kThinThreads) trsv_thin_kernel(TrsvLaunch L, int t, int ld,
                                                                 const int32_t* __restrict__ order, Deps deps,
                                                                 double* __restrict__ x, Body body, Fin fin,
                                                                 double* __restrict__ partials,
                                                                 unsigned* __restrict__ counter,
                                                                 const int* __restrict__ gate,
                                                                 long long* __restrict__ tstamp) {
  if (gate != nullptr && *((volatile const int*)gate) == 0) return;
  extern __shared__ double rsh[];
  constexpr int GPW = 32 / G;
  constexpr int NC = NU * U;
  constexpr int NRR = NR > 0 ? NR : 1;
  const int lane = threadIdx.x & 31;
  const int gl = lane % G;
  const int gi = lane / G;
  const int warp = threadIdx.x >> 5;
  const int nwarps = blockDim.x >> 5;
  double acc[NRR][NC];
#pragma unroll
  for (int r = 0; r < NRR; ++r)
#pragma unroll
    for (int i = 0; i < NC; ++i) acc[r][i] = 0.0;
  for (int lv = L.L0; lv < L.L1; ++lv) {
    const int64_t q0 = L.lptr[lv], q1 = L.lptr[lv + 1];
    for (int64_t pbase = q0 + (int64_t)warp * GPW; pbase < q1; pbase += (int64_t)nwarps * GPW)
      trsv_row<G, NU, U, false>(pbase + gi, q1, t, ld, order, deps, x, body, 0u, tstamp, gl, acc[0]);
    __syncthreads();
  }
  if constexpr (NR > 0) {
    block_reduce_cols<G, NU, U, NR, 0>(acc, t, partials + (size_t)L.slot_base * NR * t, rsh);
    grid_finalize<NR, 0>(partials, counter, t, fin, rsh, L.total_slots);
  }
}

}  // namespace vl
