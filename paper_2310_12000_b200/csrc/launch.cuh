// Launch helpers: (G, NC) dispatch by column count, rows/trsv launchers.
#pragma once

#include <type_traits>

#include "context.h"
#include "rows.cuh"

namespace vl {

template <int V>
using IC = std::integral_constant<int, V>;

// Lanes-per-row G and columns-per-lane NC for a given t.
template <class F>
void dispatch_t(int t, F&& f) {
  if (t <= 0) fail(kEConfig, "column count must be >= 1");
  if (t == 1) f(IC<1>{}, IC<1>{});
  else if (t <= 2) f(IC<2>{}, IC<1>{});
  else if (t <= 4) f(IC<4>{}, IC<1>{});
  else if (t <= 8) f(IC<8>{}, IC<1>{});
  else if (t <= 16) f(IC<16>{}, IC<1>{});
  else if (t <= 32) f(IC<32>{}, IC<1>{});
  else if (t <= 64) f(IC<32>{}, IC<2>{});
  else if (t <= 128) f(IC<32>{}, IC<4>{});
  else fail(kECapacity, "more than 128 right-hand sides per call are not supported; shard the probes");
}

unsigned* next_counter(Ctx& C);
void ensure_flags(Ctx& C, int64_t n);
int coop_grid(Ctx& C, const void* func, size_t smem);

template <int G, int NC, int NR, int MAXMASK, class Body, class Fin>
void launch_rows(Ctx& C, int64_t n, int t, const Body& body, const Fin& fin, const int* gate = nullptr) {
  auto kern = rows_kernel<G, NC, NR, MAXMASK, Body, Fin>;
  const size_t smem = red_smem_bytes<G, NC, NR>(kRowsThreads, t);
  int64_t need = (n * G + kRowsThreads - 1) / kRowsThreads;
  int64_t cap = (int64_t)C.num_sms * (2048 / kRowsThreads);
  int blocks = (int)std::max<int64_t>(1, std::min<int64_t>(need, cap));
  kern<<<blocks, kRowsThreads, smem, C.stream>>>(n, t, body, fin, C.red_partial.as<double>(), next_counter(C), gate);
  VL_LAUNCH_CHECK();
}

template <int G, int NC, int NR, class Deps, class Body, class Fin>
void launch_trsv(Ctx& C, int64_t n, int t, const int32_t* order, const Deps& deps, double* x, const Body& body,
                 const Fin& fin, const int* gate = nullptr) {
  auto kern = trsv_kernel<G, NC, NR, Deps, Body, Fin>;
  const size_t smem = red_smem_bytes<G, NC, NR>(kRowsThreads, t);
  ensure_flags(C, n);
  int grid = coop_grid(C, (const void*)kern, smem);
  int64_t need = (n * G + kRowsThreads - 1) / kRowsThreads;
  if (need < grid) grid = (int)std::max<int64_t>(1, need);
  int epoch = C.next_flag_epoch();
  int* flags = C.flags.as<int>();
  double* partials = C.red_partial.as<double>();
  unsigned* counter = next_counter(C);
  void* args[] = {(void*)&n, (void*)&t, (void*)&order, (void*)&deps, (void*)&x, (void*)&flags, (void*)&epoch,
                  (void*)&body, (void*)&fin, (void*)&partials, (void*)&counter, (void*)&gate};
  VL_CUDA(cudaLaunchCooperativeKernel((const void*)kern, dim3(grid), dim3(kRowsThreads), args, smem, C.stream));
}

}  // namespace vl
