// Launch helpers: (G, NU, U) dispatch by column count / leading dimension,
// rows/trsv launchers.
#pragma once

#include <algorithm>
#include <type_traits>

#include "context.h"
#include "rows.cuh"

namespace vl {

template <int V>
using IC = std::integral_constant<int, V>;

// Column layout of an n x ld block holding t <= ld columns.
//   U  = 2 (16-byte units) when ld is even and t > 1, else 1
//   G  = lanes per row = min(32, pow2ceil(#units))
//   NU = units per lane
template <class F>
void dispatch_cols(int t, int ld, F&& f) {
  if (t <= 0 || ld < t) fail(kEConfig, "invalid column count / leading dimension");
  const bool pair = (t > 1) && (ld % 2 == 0);
  const int units = pair ? (t + 1) / 2 : t;
  auto go = [&](auto u) {
    constexpr int U = decltype(u)::value;
    if (units == 1) f(IC<1>{}, IC<1>{}, IC<U>{});
    else if (units <= 2) f(IC<2>{}, IC<1>{}, IC<U>{});
    else if (units <= 4) f(IC<4>{}, IC<1>{}, IC<U>{});
    else if (units <= 8) f(IC<8>{}, IC<1>{}, IC<U>{});
    else if (units <= 16) f(IC<16>{}, IC<1>{}, IC<U>{});
    else if (units <= 32) f(IC<32>{}, IC<1>{}, IC<U>{});
    else if (units <= 64) f(IC<32>{}, IC<2>{}, IC<U>{});
    else fail(kECapacity, "more than 128 right-hand sides per call are not supported; shard the probes");
  };
  if (pair) go(IC<2>{});
  else go(IC<1>{});
}

unsigned* next_counter(Ctx& C);
int coop_grid(Ctx& C, const void* func, size_t smem);
cudaEvent_t prof_begin(Ctx& C);
void prof_end(Ctx& C, cudaEvent_t a);

// Tag the kernels launched in a scope (algorithmic bytes per launch).
struct ProfScope {
  Ctx& C;
  const char* old_tag;
  double old_bytes;
  ProfScope(Ctx& c, const char* tag, double bytes) : C(c), old_tag(c.prof.tag), old_bytes(c.prof.bytes) {
    C.prof.tag = tag;
    C.prof.bytes = bytes;
  }
  ~ProfScope() {
    C.prof.tag = old_tag;
    C.prof.bytes = old_bytes;
  }
};

// SURVEY 8(d) algorithmic bytes of one B-apply over n x t (f64 values, int32
// indices and row pointer; x read once, y written once) + 8n per fused diagonal
inline double bapply_bytes(const Pattern& P, int t, int diag_vectors) {
  const double nnz = (double)P.nnz_off + (double)P.n;
  return 12.0 * nnz + 4.0 * (P.n + 1) + 16.0 * (double)P.n * t + 8.0 * P.n * diag_vectors;
}

template <int G, int NU, int U, int NR, int MAXMASK, class Body, class Fin>
void launch_rows(Ctx& C, int64_t n, int t, const Body& body, const Fin& fin, const int* gate = nullptr) {
  auto kern = rows_kernel<G, NU, U, NR, MAXMASK, Body, Fin>;
  const size_t smem = red_smem_bytes<G, NU, U, NR>(kRowsThreads, t);
  int64_t need = (n * G + kRowsThreads - 1) / kRowsThreads;
  int64_t cap = (int64_t)C.num_sms * (2048 / kRowsThreads);
  int blocks = (int)std::max<int64_t>(1, std::min<int64_t>(need, cap));
  C.prof.launches++;
  cudaEvent_t ev = (C.prof.on && C.prof.tag) ? prof_begin(C) : nullptr;
  kern<<<blocks, kRowsThreads, smem, C.stream>>>(n, t, body, fin, C.red_partial.as<double>(), next_counter(C), gate);
  VL_LAUNCH_CHECK();
  if (ev) prof_end(C, ev);
}

// x (n x ld) is overwritten: it is first filled with the "not ready" sentinel.
template <int G, int NU, int U, int NR, class Deps, class Body, class Fin>
void launch_trsv(Ctx& C, int64_t n, int64_t npos, int t, int ld, const int32_t* order, const Deps& deps, double* x,
                 const Body& body, const Fin& fin, const int* gate = nullptr) {
  auto kern = trsv_kernel<G, NU, U, NR, Deps, Body, Fin>;
  const size_t smem = red_smem_bytes<G, NU, U, NR>(kRowsThreads, t);
  int grid = coop_grid(C, (const void*)kern, smem);
  grid = std::min(grid, C.num_sms * C.trsv_blocks_per_sm);
  int64_t need = (npos * G + kRowsThreads - 1) / kRowsThreads;
  if (need < grid) grid = (int)std::max<int64_t>(1, need);
  C.prof.launches++;
  cudaEvent_t ev = (C.prof.on && C.prof.tag) ? prof_begin(C) : nullptr;
  VL_CUDA(cudaMemsetAsync(x, 0xFF, sizeof(double) * (size_t)n * ld, C.stream));
  double* partials = C.red_partial.as<double>();
  unsigned* counter = next_counter(C);
  unsigned smax = (unsigned)C.spin_max_ns;
  long long* tstamp = C.debug_tstamp;
  void* args[] = {(void*)&npos,  (void*)&t,    (void*)&ld,       (void*)&order,   (void*)&deps,
                  (void*)&x,     (void*)&body, (void*)&fin,      (void*)&partials, (void*)&counter,
                  (void*)&gate,  (void*)&smax, (void*)&tstamp};
  VL_CUDA(cudaLaunchCooperativeKernel((const void*)kern, dim3(grid), dim3(kRowsThreads), args, smem, C.stream));
  if (ev) prof_end(C, ev);
}

}  // namespace vl
