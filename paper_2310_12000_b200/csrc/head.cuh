// Dense head block of the triangular solves.
//
// The rows of the first head_L forward levels (H of them, in level order)
// form a closed unit-lower-triangular block B_HH; no row outside has a child
// inside it.  X = B_HH^-1 is formed densely once per factor (column-major,
// lower triangular) and replaces head_L dependency hops in every solve:
//   forward  (B^-1):  x_H = X (rhs_H)                     then the rest
//   backward (B^-T):  the rest first, then x_H = X^T (rhs_H - B_RH^T x_R)
// The solve's fused rhs/out bodies run on the head rows exactly as on the
// others, and its column reductions use the same partial-slot space.
#pragma once

#include "rows.cuh"

namespace vl {

// one warp per column c: x = B_HH^-1 e_c by forward substitution in head
// order (lanes over the row's dependencies), x kept in shared memory.
__global__ void __launch_bounds__(128) head_inverse_kernel(int H, int m, const int32_t* __restrict__ head_rows,
                                                           const int32_t* __restrict__ head_nbr,
                                                           const int32_t* __restrict__ cnt,
                                                           const double* __restrict__ val, double* __restrict__ X);

// rhs (+ backward external gather) of the head rows -> Y (H x t, ld t)
template <int G, int NU, int U, int NR, bool EXT, class Body, class Fin>
__global__ void __launch_bounds__(kRowsThreads) head_rhs_kernel(int H, int t, int ld,
                                                                const int32_t* __restrict__ head_rows,
                                                                const int32_t* __restrict__ head_pos,
                                                                const int32_t* __restrict__ tptr,
                                                                const int32_t* __restrict__ tidx,
                                                                const double* __restrict__ valT,
                                                                const double* __restrict__ x, double* __restrict__ Y,
                                                                Body body, Fin fin, double* __restrict__ partials,
                                                                unsigned* __restrict__ counter, int slot_base,
                                                                int total_slots, const int* __restrict__ gate) {
  if (gate != nullptr && *((volatile const int*)gate) == 0) return;
  extern __shared__ double rsh[];
  constexpr int GPW = 32 / G;
  constexpr int NC = NU * U;
  constexpr int NRR = NR > 0 ? NR : 1;
  using CL = Cols<G, NU, U>;
  const int lane = threadIdx.x & 31, gl = lane % G, gi = lane / G;
  const int64_t gwarp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  double acc[NRR][NC];
#pragma unroll
  for (int r = 0; r < NRR; ++r)
#pragma unroll
    for (int i = 0; i < NC; ++i) acc[r][i] = 0.0;
  if constexpr (EXT && G == 1 && NU == 1 && U == 1) {
    // single column: one warp per head row, lanes over its children
    for (int64_t h = gwarp; h < H; h += nwarps) {
      const int64_t s = head_rows[h];
      const int e0 = tptr[s], e1 = tptr[s + 1];
      // 4 entries per lane in flight; the head mask and x load both depend only
      // on the child index (x of a head child is read but not used) -- the
      // same per-lane entry order as a plain strided loop
      double part = 0.0;
      for (int eb = e0 + lane; eb < e1; eb += 128) {
        int32_t ch[4];
        double w[4], xv[4];
        int hp[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int e = eb + 32 * q;
          ch[q] = e < e1 ? tidx[e] : 0;
          w[q] = e < e1 ? valT[e] : 0.0;
        }
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          hp[q] = head_pos[ch[q]];
          xv[q] = __ldcg(x + (int64_t)ch[q] * ld);
        }
#pragma unroll
        for (int q = 0; q < 4; ++q)
          if (eb + 32 * q < e1 && hp[q] < 0) part += w[q] * xv[q];
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
      if (lane == 0) {
        const double rv = body.rhs(s, 0, acc[0][0]);
        if constexpr (PsumOf<Body>::value) body.keep_rhs(s, 0, rv);
        Y[h] = rv - part;
      }
    }
  } else
  for (int64_t h0 = gwarp * GPW; h0 < H; h0 += nwarps * GPW) {
    const int64_t h = h0 + gi;
    if (h >= H) continue;
    const int64_t s = head_rows[h];
    double ys[NC];
#pragma unroll
    for (int i = 0; i < NC; ++i) {
      const int c = CL::col(gl, i);
      ys[i] = c < t ? body.rhs(s, c, acc[0][i]) : 0.0;
      if constexpr (PsumOf<Body>::value)
        if (c < t) body.keep_rhs(s, c, ys[i]);
    }
    if (EXT) {
      // children outside the head (head children are handled by X^T); 8 in flight
      const int e0 = tptr[s], e1 = tptr[s + 1];
      for (int eb = e0; eb < e1; eb += 8) {
        double w[8], v[8][NC];
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          const int e = eb + q;
          const int32_t ch = e < e1 ? tidx[e] : 0;
          const bool on = e < e1 && head_pos[ch] < 0;
          w[q] = on ? valT[e] : 0.0;
#pragma unroll
          for (int k = 0; k < NU; ++k) {
            const int c = U * (gl + G * k);
            if (on && c < t) ld_cg_unit<U>(x + (int64_t)ch * ld + c, &v[q][U * k]);
            else
#pragma unroll
              for (int i = 0; i < U; ++i) v[q][U * k + i] = 0.0;
          }
        }
#pragma unroll
        for (int q = 0; q < 8; ++q)
#pragma unroll
          for (int i = 0; i < NC; ++i) ys[i] -= w[q] * v[q][i];
      }
    }
#pragma unroll
    for (int i = 0; i < NC; ++i) {
      const int c = CL::col(gl, i);
      if (c < t) Y[h * t + c] = ys[i];
    }
  }
  if constexpr (NR > 0) {
    block_reduce_cols<G, NU, U, NR, 0>(acc, t, partials + (size_t)(slot_base + blockIdx.x) * NR * t, rsh);
    grid_finalize<NR, 0>(partials, counter, t, fin, rsh, total_slots);
  }
}

// Single column: Xh[r] = sum_q M[r][q] Y[q] with M row-major (X for the
// forward solve, X^T for the backward one).  One CTA per output row: its 8
// warps take 8 contiguous chunks of the row's nonzero range (lanes over q,
// coalesced), then a fixed-order combine -- deterministic, and the longest
// rows (~H entries) no longer set the launch time through one warp's serial
// load chain (warp-per-row: 19 us for H = 3072).  ksplit = 1.
constexpr int kGemvThreads = 256;
template <bool TRANS>
__global__ void __launch_bounds__(kGemvThreads) head_gemv_kernel(int H, const double* __restrict__ M,
                                                                 const double* __restrict__ Y,
                                                                 double* __restrict__ Xh,
                                                                 const int* __restrict__ gate) {
  if (gate != nullptr && *((volatile const int*)gate) == 0) return;
  __shared__ double sp[kGemvThreads / 32];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int r = blockIdx.x;
  const double* row = M + (size_t)r * H;
  // X row r is nonzero for q <= r; X^T row r for q >= r
  const int q0 = TRANS ? r : 0, q1 = TRANS ? H : r + 1;
  const int len = q1 - q0;
  const int cw = ((len + 8 * 32 - 1) / (8 * 32)) * 32;  // chunk per warp, whole 32-entry rounds
  const int a = q0 + w * cw, b = min(q1, a + cw);
  double acc = 0.0;
  int q = a + lane;
  for (; q + 96 < b; q += 128) {
    const double a0 = row[q], a1 = row[q + 32], a2 = row[q + 64], a3 = row[q + 96];
    const double y0 = Y[q], y1 = Y[q + 32], y2 = Y[q + 64], y3 = Y[q + 96];
    acc += a0 * y0;
    acc += a1 * y1;
    acc += a2 * y2;
    acc += a3 * y3;
  }
  for (; q < b; q += 32) acc += row[q] * Y[q];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if (lane == 0) sp[w] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
#pragma unroll
    for (int k = 0; k < kGemvThreads / 32; ++k) s += sp[k];
    Xh[r] = s;
  }
}

// Xh_k = partial of X Y (TRANS = false) or X^T Y (TRANS = true) over the
// q-range of split k = blockIdx.y; X is H x H column-major lower triangular;
// Y is H x t; partials [ksplit][H][t] are summed in fixed order by
// head_out_kernel.  Block: 32 output rows x 8 column groups, tiles in smem.
template <bool TRANS>
__global__ void __launch_bounds__(256) head_apply_kernel(int H, int t, const double* __restrict__ X,
                                                         const double* __restrict__ Y, double* __restrict__ Xh,
                                                         const int* __restrict__ gate) {
  if (gate != nullptr && *((volatile const int*)gate) == 0) return;
  constexpr int TQ = 32;
  __shared__ double xs[TQ][TQ + 1];
  extern __shared__ double ysm[];  // [TQ][t]
  const int lr = threadIdx.x & 31;  // row within tile
  const int cg = threadIdx.x >> 5;  // column group (8)
  const int r = blockIdx.x * 32 + lr;
  constexpr int MAXC = 16;          // columns per thread (t <= 128)
  double acc[MAXC];
#pragma unroll
  for (int j = 0; j < MAXC; ++j) acc[j] = 0.0;
  const int r0 = blockIdx.x * 32;
  const int kspan = (H + gridDim.y - 1) / gridDim.y;
  const int ka = blockIdx.y * kspan, kb = min(H, ka + kspan);
  Xh += (size_t)blockIdx.y * H * t;
  // lower triangular: row r of X uses q <= r ; row r of X^T uses q >= r
  const int qbeg = max(ka, TRANS ? r0 : 0);
  const int qend = min(kb, TRANS ? H : min(H, r0 + 32));
  for (int q0 = qbeg; q0 < qend; q0 += TQ) {
    // stage X tile: elements needed: (row r0+i, col q0+k) of X or X^T
    for (int idx = threadIdx.x; idx < TQ * TQ; idx += blockDim.x) {
      const int a = idx / TQ, b = idx % TQ;  // a: slow, b: fast (coalesced in memory)
      double v = 0.0;
      if (!TRANS) {
        // X(row r0+b, col q0+a) = X[(q0+a)*H + r0+b]
        const int rr = r0 + b, qq = q0 + a;
        if (rr < H && qq < qend && qq <= rr) v = X[(size_t)qq * H + rr];
        xs[b][a] = v;  // xs[row][q]
      } else {
        // X^T(row r0+a, col q0+b) = X(q0+b, r0+a) = X[(r0+a)*H + q0+b]
        const int rr = r0 + a, qq = q0 + b;
        if (rr < H && qq < qend && qq >= rr) v = X[(size_t)rr * H + qq];
        xs[a][b] = v;
      }
    }
    for (int idx = threadIdx.x; idx < TQ * t; idx += blockDim.x) {
      const int a = idx / t, c = idx % t;
      const int qq = q0 + a;
      ysm[a * t + c] = qq < qend ? Y[(size_t)qq * t + c] : 0.0;
    }
    __syncthreads();
#pragma unroll 4
    for (int k = 0; k < TQ; ++k) {
      const double xv = xs[lr][k];
#pragma unroll
      for (int j = 0; j < MAXC; ++j) {
        const int c = cg + 8 * j;
        if (c < t) acc[j] += xv * ysm[k * t + c];
      }
    }
    __syncthreads();
  }
  if (r < H) {
#pragma unroll
    for (int j = 0; j < MAXC; ++j) {
      const int c = cg + 8 * j;
      if (c < t) Xh[(size_t)r * t + c] = acc[j];
    }
  }
}

// x[s_h] = Xh[h]; out() epilogue on the head rows
template <int G, int NU, int U, int NR, class Body, class Fin>
__global__ void __launch_bounds__(kRowsThreads) head_out_kernel(int H, int t, int ld,
                                                                const int32_t* __restrict__ head_rows,
                                                                const double* __restrict__ Xh, int ksplit,
                                                                double* __restrict__ x, Body body, Fin fin,
                                                                double* __restrict__ partials,
                                                                unsigned* __restrict__ counter, int slot_base,
                                                                int total_slots, const int* __restrict__ gate) {
  if (gate != nullptr && *((volatile const int*)gate) == 0) return;
  extern __shared__ double rsh[];
  constexpr int GPW = 32 / G;
  constexpr int NC = NU * U;
  constexpr int NRR = NR > 0 ? NR : 1;
  using CL = Cols<G, NU, U>;
  const int lane = threadIdx.x & 31, gl = lane % G, gi = lane / G;
  const int64_t gwarp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  double acc[NRR][NC];
#pragma unroll
  for (int r = 0; r < NRR; ++r)
#pragma unroll
    for (int i = 0; i < NC; ++i) acc[r][i] = 0.0;
  for (int64_t h0 = gwarp * GPW; h0 < H; h0 += nwarps * GPW) {
    const int64_t h = h0 + gi;
    if (h >= H) continue;
    const int64_t s = head_rows[h];
#pragma unroll
    for (int i = 0; i < NC; ++i) {
      const int c = CL::col(gl, i);
      if (c < t) {
        double xv = Xh[h * t + c];
        for (int k = 1; k < ksplit; ++k) xv += Xh[(size_t)k * H * t + h * t + c];
        __stcg(x + s * ld + c, sanitize(xv));
        body.out(s, c, xv, acc[0][i]);
      }
    }
  }
  if constexpr (NR > 0) {
    block_reduce_cols<G, NU, U, NR, 0>(acc, t, partials + (size_t)(slot_base + blockIdx.x) * NR * t, rsh);
    grid_finalize<NR, 0>(partials, counter, t, fin, rsh, total_slots);
  }
}

// Fused product of a backward solve (PsumOf<Body>) on the head rows, run
// after head_out when all of y is final:  p_s = om_s y_s + sum_c B_cs om_c y_c
// over ALL children c (head or not).  Single column: warp per row.
template <int G, int NU, int U, class Body>
__global__ void __launch_bounds__(kRowsThreads) head_psum_kernel(int H, int t, int ld,
                                                                 const int32_t* __restrict__ head_rows,
                                                                 const int32_t* __restrict__ tptr,
                                                                 const int32_t* __restrict__ tidx,
                                                                 const double* __restrict__ valT,
                                                                 const double* __restrict__ x, Body body,
                                                                 const int* __restrict__ gate) {
  if (gate != nullptr && *((volatile const int*)gate) == 0) return;
  constexpr int GPW = 32 / G;
  constexpr int NC = NU * U;
  const int lane = threadIdx.x & 31, gl = lane % G, gi = lane / G;
  const int64_t gwarp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  if constexpr (G == 1 && NU == 1 && U == 1) {
    for (int64_t h = gwarp; h < H; h += nwarps) {
      const int64_t s = head_rows[h];
      const int e0 = tptr[s], e1 = tptr[s + 1];
      double part = 0.0;
      for (int e = e0 + lane; e < e1; e += 32) {
        const int32_t ch = tidx[e];
        part += (valT[e] * __ldg(body.om + ch)) * __ldcg(x + (int64_t)ch * ld);
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
      if (lane == 0) body.pout[s] = fma(__ldg(body.om + s), __ldcg(x + s), part);
    }
  } else {
    for (int64_t h0 = gwarp * GPW; h0 < H; h0 += nwarps * GPW) {
      const int64_t h = h0 + gi;
      if (h >= H) continue;
      const int64_t s = head_rows[h];
      const double os = __ldg(body.om + s);
      double ps[NC];
#pragma unroll
      for (int k = 0; k < NU; ++k) {
        const int c = U * (gl + G * k);
        double v[U];
        if (c < t) ld_cg_unit<U>(x + s * ld + c, v);
        else
#pragma unroll
          for (int i = 0; i < U; ++i) v[i] = 0.0;
#pragma unroll
        for (int i = 0; i < U; ++i) ps[U * k + i] = os * v[i];
      }
      const int e0 = tptr[s], e1 = tptr[s + 1];
      for (int e = e0; e < e1; ++e) {
        const int32_t ch = tidx[e];
        const double wo = valT[e] * __ldg(body.om + ch);
#pragma unroll
        for (int k = 0; k < NU; ++k) {
          const int c = U * (gl + G * k);
          double v[U];
          if (c < t) ld_cg_unit<U>(x + (int64_t)ch * ld + c, v);
          else
#pragma unroll
            for (int i = 0; i < U; ++i) v[i] = 0.0;
#pragma unroll
          for (int i = 0; i < U; ++i) ps[U * k + i] += wo * v[i];
        }
      }
#pragma unroll
      for (int k = 0; k < NU; ++k) {
        const int c = U * (gl + G * k);
        if (c < t) {
          double* dst = body.pout + s * ld + c;
          if constexpr (U == 2) *reinterpret_cast<double2*>(dst) = make_double2(ps[2 * k], ps[2 * k + 1]);
          else *dst = ps[k];
        }
      }
    }
  }
}

}  // namespace vl
