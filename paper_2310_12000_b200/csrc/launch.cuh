// Launch helpers: (G, NU, U) dispatch by column count / leading dimension,
// rows/trsv launchers.
#pragma once

#include <algorithm>
#include <type_traits>
#include <vector>

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

// Split a level sequence (padded position pointer, nlev levels) into
// alternating thin / thick segments: a level is thin when it has at most
// `thin_rows` (padded) rows.  Returns {L0, L1, thin}.
struct Seg {
  int L0, L1;
  bool thin;
};
std::vector<Seg> solve_segments(const std::vector<int32_t>& lptr, int thin_rows, int min_thick_levels);

// Triangular solve over the fwd (B) or bwd (B^T) schedule.  x (n x ld) is
// overwritten: it is first filled with the "not ready" sentinel; thin
// segments run on one CTA, thick segments grid-wide (sync-free).  Fused
// column reductions finalise once over all segments' partial slots.
template <int G, int NU, int U, int NR, class Deps, class Body, class Fin>
void launch_trsv(Ctx& C, const Pattern& P, bool fwd, int t, int ld, const Deps& deps, double* x, const Body& body,
                 const Fin& fin, const int* gate = nullptr) {
  const int64_t n = P.n;
  const int32_t* order = fwd ? P.fwd_order.as<int32_t>() : P.bwd_order.as<int32_t>();
  if constexpr (G == 1 && NU == 1 && U == 1) {
    if (C.thin_passes == 0) {
      // single right-hand side: light/heavy work items, one sync-free launch
      auto k1 = trsv1_kernel<NR, Deps, Body, Fin>;
      const size_t smem1 = red_smem_bytes<1, 1, 1, NR>(kRowsThreads, 1);
      int grid = coop_grid(C, (const void*)k1, smem1);
      grid = std::min(grid, C.num_sms * C.trsv_blocks_per_sm);
      const int64_t nitems = fwd ? P.fwd_nitems : P.bwd_nitems;
      const int64_t npos = fwd ? P.fwd_len : P.bwd_len;
      const uint32_t* items = fwd ? P.fwd_items.as<uint32_t>() : P.bwd_items.as<uint32_t>();
      C.prof.launches += 2;
      cudaEvent_t ev = (C.prof.on && C.prof.tag) ? prof_begin(C) : nullptr;
      VL_CUDA(cudaMemsetAsync(x, 0xFF, sizeof(double) * (size_t)n * ld, C.stream));
      double* partials = C.red_partial.as<double>();
      unsigned* counter = next_counter(C);
      unsigned smax = (unsigned)C.spin_max_ns;
      long long* tstamp = C.debug_tstamp;
      void* args[] = {(void*)&nitems, (void*)&npos,     (void*)&items,   (void*)&order, (void*)&deps,
                      (void*)&x,      (void*)&body,     (void*)&fin,     (void*)&partials, (void*)&counter,
                      (void*)&gate,   (void*)&smax,     (void*)&tstamp};
      VL_CUDA(cudaLaunchCooperativeKernel((const void*)k1, dim3(grid), dim3(kRowsThreads), args, smem1, C.stream));
      if (ev) prof_end(C, ev);
      return;
    }
  }
  const int32_t* lptr_d = fwd ? P.fwd_lptr.as<int32_t>() : P.bwd_lptr.as<int32_t>();
  const std::vector<int32_t>& lptr = fwd ? P.fwd_level_ptr : P.bwd_level_ptr;
  auto kern = trsv_kernel<G, NU, U, NR, Deps, Body, Fin>;
  auto tkern = trsv_thin_kernel<G, NU, U, NR, Deps, Body, Fin>;
  const size_t smem = red_smem_bytes<G, NU, U, NR>(kRowsThreads, t);
  const size_t tsmem = red_smem_bytes<G, NU, U, NR>(kThinThreads, t);
  const int thin_rows = C.thin_passes * (kThinThreads / G);
  std::vector<Seg> segs = solve_segments(lptr, thin_rows, C.min_thick_levels);
  int gcap = coop_grid(C, (const void*)kern, smem);
  gcap = std::min(gcap, C.num_sms * C.trsv_blocks_per_sm);
  std::vector<int> grids(segs.size(), 1);
  int total = 0;
  for (size_t i = 0; i < segs.size(); ++i) {
    if (!segs[i].thin) {
      const int64_t npos = (int64_t)lptr[segs[i].L1] - lptr[segs[i].L0];
      const int64_t need = (npos * G + kRowsThreads - 1) / kRowsThreads;
      grids[i] = (int)std::max<int64_t>(1, std::min<int64_t>(need, gcap));
    }
    total += grids[i];
  }
  C.prof.launches += 1 + (long long)segs.size();
  cudaEvent_t ev = (C.prof.on && C.prof.tag) ? prof_begin(C) : nullptr;
  VL_CUDA(cudaMemsetAsync(x, 0xFF, sizeof(double) * (size_t)n * ld, C.stream));
  double* partials = C.red_partial.as<double>();
  unsigned* counter = next_counter(C);
  unsigned smax = (unsigned)C.spin_max_ns;
  long long* tstamp = C.debug_tstamp;
  int slot = 0;
  for (size_t i = 0; i < segs.size(); ++i) {
    TrsvLaunch L;
    L.L0 = segs[i].L0;
    L.L1 = segs[i].L1;
    L.p0 = lptr[segs[i].L0];
    L.p1 = lptr[segs[i].L1];
    L.lptr = lptr_d;
    L.slot_base = slot;
    L.total_slots = total;
    slot += grids[i];
    if (segs[i].thin) {
      if (tsmem > 48 * 1024) VL_CUDA(cudaFuncSetAttribute(tkern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)tsmem));
      tkern<<<1, kThinThreads, tsmem, C.stream>>>(L, t, ld, order, deps, x, body, fin, partials, counter, gate,
                                                  tstamp);
      VL_LAUNCH_CHECK();
    } else {
      void* args[] = {(void*)&L,     (void*)&t,       (void*)&ld,       (void*)&order,   (void*)&deps,
                      (void*)&x,     (void*)&body,    (void*)&fin,      (void*)&partials, (void*)&counter,
                      (void*)&gate,  (void*)&smax,    (void*)&tstamp};
      VL_CUDA(cudaLaunchCooperativeKernel((const void*)kern, dim3(grids[i]), dim3(kRowsThreads), args, smem,
                                          C.stream));
    }
  }
  if (ev) prof_end(C, ev);
}

}  // namespace vl
