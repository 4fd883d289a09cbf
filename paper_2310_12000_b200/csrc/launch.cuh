// Launch helpers: (G, NU, U) dispatch by column count / leading dimension,
// rows/trsv launchers.
#pragma once

#include <algorithm>
#include <cstdlib>
#include <string>
#include <type_traits>
#include <vector>

#include "context.h"
#include "head.cuh"
#include "rows.cuh"

namespace vl {

template <int V>
using IC = std::integral_constant<int, V>;

// Column layout of an n x ld block holding t <= ld columns.
//   U  = 2 (16-byte units) when ld is even and t > 1, else 1
//   G  = lanes per row = min(32, pow2ceil(#units))
//   NU = units per lane
#ifndef VL_G16
#define VL_G16 0
#endif
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
#if VL_G16
    else if (units <= 32) f(IC<16>{}, IC<2>{}, IC<U>{});   // two rows per warp, two units per lane
#else
    else if (units <= 32) f(IC<32>{}, IC<1>{}, IC<U>{});
#endif
    else if (units <= 64) f(IC<32>{}, IC<2>{}, IC<U>{});
    else fail(kECapacity, "more than 128 right-hand sides per call are not supported; shard the probes");
  };
  if (pair) go(IC<2>{});
  else go(IC<1>{});
}

// VL_DEBUG_SYNC=1: synchronise after every launch of the row / solve launchers and name the
// failing instantiation (compute-sanitizer is not always available)
inline void debug_sync(Ctx& C, const char* what) {
  static const bool on = std::getenv("VL_DEBUG_SYNC") != nullptr;
  if (!on) return;
  const cudaError_t e = cudaStreamSynchronize(C.stream);
  if (e != cudaSuccess) fail(kECuda, std::string("kernel failed: ") + what + ": " + cudaGetErrorString(e));
}

unsigned* next_counter(Ctx& C);

// Dependencies of the forward solve: the solve-ordered copy of the ELL rows when the pattern
// has one (late parents last, pattern.cpp), else the rows as the factor build wrote them.
inline DepsEll deps_fwd(const Factor& F) {
  const Pattern& P = *F.pat;
  if (F.val_s.p != nullptr && P.has_solve_order)
    return DepsEll{P.nbr_s.as<int32_t>(), P.cnt.as<int32_t>(), F.val_s.as<double>(), P.m};
  return DepsEll{P.nbr.as<int32_t>(), P.cnt.as<int32_t>(), F.val.as<double>(), P.m};
}
int coop_grid(Ctx& C, const void* func, size_t smem);
cudaEvent_t prof_begin(Ctx& C, cudaStream_t st = nullptr);  // nullptr: C.stream
void prof_end(Ctx& C, cudaEvent_t a, cudaStream_t st = nullptr);

// Tag the kernels launched in a scope (algorithmic bytes per launch).
struct ProfScope {
  Ctx& C;
  const char* old_tag;
  double old_bytes;
  ProfScope(Ctx& c, const char* tag, double bytes) : C(c), old_tag(c.prof.tag), old_bytes(c.prof.bytes) {
    C.prof.tag = (c.prof.only.empty() || c.prof.only == tag) ? tag : nullptr;
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
void launch_rows(Ctx& C, int64_t n, int t, const Body& body, const Fin& fin, const int* gate = nullptr,
                 const int32_t* wptr = nullptr) {
  auto kern = rows_kernel<G, NU, U, NR, MAXMASK, Body, Fin>;
  const size_t smem = red_smem_bytes<G, NU, U, NR>(kRowsThreads, t);
  int64_t need = (n * G + kRowsThreads - 1) / kRowsThreads;
  int64_t cap = (int64_t)C.num_sms * (2048 / kRowsThreads);
  int blocks = (int)std::max<int64_t>(1, std::min<int64_t>(need, cap));
  C.prof.launches++;
  cudaEvent_t ev = (C.prof.on && C.prof.tag) ? prof_begin(C) : nullptr;
  kern<<<blocks, kRowsThreads, smem, C.stream>>>(n, t, body, fin, C.red_partial.as<double>(), next_counter(C), gate,
                                                 wptr);
  VL_LAUNCH_CHECK();
  if (ev) prof_end(C, ev);
  debug_sync(C, __PRETTY_FUNCTION__);
}

// SM-local sweep (rows_local_kernel) for gather bodies over a spatially
// ordered pattern; falls back to launch_rows when it does not apply.
template <int G, int NU, int U, int NR, int MAXMASK, class Body, class Fin>
void launch_rows_local(Ctx& C, const Pattern& P, int64_t n, int t, const Body& body, const Fin& fin,
                       const int* gate = nullptr, const int32_t* wptr = nullptr) {
  // wptr (B^T products): work-balanced runs in either kernel
  if (!(C.use_local && P.order_kind != 0 && (G > 1 || U > 1) && n >= (int64_t)C.num_sms * 64)) {
    launch_rows<G, NU, U, NR, MAXMASK>(C, n, t, body, fin, gate, wptr);
    return;
  }
  auto kern = rows_local_kernel<G, NU, U, NR, MAXMASK, Body, Fin>;
  const size_t smem = red_smem_bytes<G, NU, U, NR>(kLocalThreads, t);
  static bool carve = false;  // prefer L1 over shared memory (per instantiation)
  if (!carve) {
    VL_CUDA(cudaFuncSetAttribute((const void*)kern, cudaFuncAttributePreferredSharedMemoryCarveout, 0));
    if (smem > 48 * 1024)
      VL_CUDA(cudaFuncSetAttribute((const void*)kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    carve = true;
  }
  C.prof.launches++;
  cudaEvent_t ev = (C.prof.on && C.prof.tag) ? prof_begin(C) : nullptr;
  kern<<<C.num_sms, kLocalThreads, smem, C.stream>>>(n, t, body, fin, C.red_partial.as<double>(), next_counter(C),
                                                     gate, wptr);
  VL_LAUNCH_CHECK();
  if (ev) prof_end(C, ev);
  debug_sync(C, __PRETTY_FUNCTION__);
}

// Split a level sequence (padded position pointer, nlev levels) into
// alternating thin / thick segments: a level is thin when it has at most
// `thin_rows` (padded) rows.  Returns {L0, L1, thin}.
struct Seg {
  int L0, L1;
  bool thin;
};
std::vector<Seg> solve_segments(const std::vector<int32_t>& lptr, int thin_rows, int min_thick_levels);

// Triangular solve over the fwd (B) or bwd (B^T) schedule of factor F.
// x (n x ld) is overwritten: it is first filled with the "not ready"
// sentinel.  Phases (one stream, one partial-slot space, one finalisation):
//   forward : [head rhs] [X . rhs_H] [head out] [sync-free rest]
//   backward: [sync-free rest] [head rhs - B_RH^T x_R] [X^T . ] [head out]
// The sync-free part runs as light/heavy work items (t == 1) or as
// thin (single-CTA) / thick (grid) level segments (t > 1).
template <int G, int NU, int U, int NR, class Deps, class Body, class Fin>
void launch_trsv(Ctx& C, const Factor& F, bool fwd, int t, int ld, const Deps& deps, double* x, const Body& body,
                 const Fin& fin, const int* gate = nullptr) {
  const Pattern& P = *F.pat;
  const int64_t n = P.n;
  const bool head = C.use_head && P.head_H > 0 && F.headX.p != nullptr;
  const int H = head ? (int)P.head_H : 0;
  // ---- main (non-head) schedule ----
  const int32_t* order;
  const int32_t* lptr_d;
  const std::vector<int32_t>* lptr;
  int L0;
  const uint32_t* items;
  int64_t nitems, npos;
  Slab sl{nullptr, nullptr, nullptr, nullptr};
  auto pick = [&](const Pattern::Slabs& S, const DevBuf& sv, int64_t skip) {
    sl.off = S.off.as<uint32_t>() + skip;  // also the heavy items' descriptors
    sl.w = S.w.as<uint32_t>() + skip;
    if (!C.use_slabs || S.nent == 0 || sv.p == nullptr) return;
    sl.idx = S.idx.as<int32_t>();
    sl.val = sv.as<double>();
  };
  if (fwd) {
    order = P.fwd_order.as<int32_t>();
    lptr_d = P.fwd_lptr.as<int32_t>();
    lptr = &P.fwd_level_ptr;
    L0 = head ? P.head_L : 0;
    items = P.fwd_items.as<uint32_t>() + (head ? P.fwd_items_head_end : 0);
    nitems = P.fwd_nitems - (head ? P.fwd_items_head_end : 0);
    npos = P.fwd_len;
    pick(P.fwd_sl, F.sv_fwd, head ? P.fwd_items_head_end : 0);
  } else if (head) {
    order = P.bwdnh_order.as<int32_t>();
    lptr_d = P.bwdnh_lptr.as<int32_t>();
    lptr = &P.bwdnh_level_ptr;
    L0 = 0;
    items = P.bwdnh_items.as<uint32_t>();
    nitems = P.bwdnh_nitems;
    npos = P.bwdnh_len;
    pick(P.bwdnh_sl, F.sv_bwdnh, 0);
  } else {
    order = P.bwd_order.as<int32_t>();
    lptr_d = P.bwd_lptr.as<int32_t>();
    lptr = &P.bwd_level_ptr;
    L0 = 0;
    items = P.bwd_items.as<uint32_t>();
    nitems = P.bwd_nitems;
    npos = P.bwd_len;
    pick(P.bwd_sl, F.sv_bwd, 0);
  }
  const bool single = (G == 1 && NU == 1 && U == 1) && C.thin_passes == 0;
  if (single) {  // light items skip the rows that run as warp-per-row items of their own
    const DevBuf& o1 = fwd ? P.fwd_order1 : (head ? P.bwdnh_order1 : P.bwd_order1);
    if (o1.p != nullptr) order = o1.as<int32_t>();
  }
  // launch geometry and slot counts
  auto k1 = trsv1_kernel<NR, Deps, Body, Fin>;
  auto kern = trsv_kernel<G, NU, U, NR, Deps, Body, Fin>;
  auto tkern = trsv_thin_kernel<G, NU, U, NR, Deps, Body, Fin>;
  const size_t smem1 = red_smem_bytes<1, 1, 1, NR>(kRowsThreads, 1);
  const size_t smem = red_smem_bytes<G, NU, U, NR>(kRowsThreads, t);
  const size_t tsmem = red_smem_bytes<G, NU, U, NR>(kThinThreads, t);
  std::vector<Seg> segs;
  std::vector<int> grids;
  int main_slots = 0;
  int grid1 = 0;
  // tile-blocked order (pattern.cpp) of the multi-column solves, when x does not fit in L2 anyway.
  // One row per warp only: with 32 / G > 1 rows per warp the rows in flight outnumber a
  // (tile, level) cell several times and the walk turns into a latency chain (measured at
  // t = 16, G = 8: B^-1 0.553 -> 0.660 ms, B^-T 0.967 -> 1.411 ms; the order itself is valid
  // for any G, its level runs are padded to 32).
  bool tiled = false;
  if constexpr (G == 32) {
    const int64_t tl = fwd ? P.fwd_tlen : P.bwd_tlen;
    tiled = !single && tl > 0 && C.use_tiles && sizeof(double) * (size_t)n * ld >= P.tile_min_bytes;
    if (tiled) {
      order = fwd ? P.fwd_torder.as<int32_t>() : P.bwd_torder.as<int32_t>();
      npos = tl;
    }
  }
  if (single) {
    grid1 = std::min(coop_grid(C, (const void*)k1, smem1), C.num_sms * C.trsv_blocks_per_sm);
    main_slots = grid1;
  } else if (tiled) {
    segs.push_back({L0, (int)lptr->size() - 1, false});
    const int gcap = std::min(coop_grid(C, (const void*)kern, smem), C.num_sms * C.trsv_blocks_per_sm);
    grids.push_back((int)std::max<int64_t>(1, std::min<int64_t>((npos * G + kRowsThreads - 1) / kRowsThreads, gcap)));
    main_slots = grids[0];
  } else {
    std::vector<int32_t> sub(lptr->begin() + L0, lptr->end());
    segs = solve_segments(sub, C.thin_passes * (kThinThreads / G), C.min_thick_levels);
    int gcap = std::min(coop_grid(C, (const void*)kern, smem), C.num_sms * C.trsv_blocks_per_sm);
    for (auto& sg : segs) {
      sg.L0 += L0;
      sg.L1 += L0;
      int gsz = 1;
      if (!sg.thin) {
        const int64_t np = (int64_t)(*lptr)[sg.L1] - (*lptr)[sg.L0];
        gsz = (int)std::max<int64_t>(1, std::min<int64_t>((np * G + kRowsThreads - 1) / kRowsThreads, gcap));
      }
      grids.push_back(gsz);
      main_slots += gsz;
    }
  }
  // head kernels: rows per group (warp per row for the single-column backward gather)
  const int hlanes = (t == 1 && !fwd) ? 32 : G;
  const int hgrid = head ? std::max(1, std::min(4 * C.num_sms, (int)((H * hlanes + kRowsThreads - 1) / kRowsThreads))) : 0;
  const int total = main_slots + 2 * hgrid;
  C.prof.launches += 1 + (single ? 1 : (long long)segs.size()) + (head ? 3 : 0) +
                     ((head && !fwd && PsumOf<Body>::value) ? 1 : 0);
  cudaEvent_t ev = (C.prof.on && C.prof.tag) ? prof_begin(C) : nullptr;
  VL_CUDA(cudaMemsetAsync(x, 0xFF, sizeof(double) * (size_t)n * ld, C.stream));
  double* partials = C.red_partial.as<double>();
  unsigned* counter = next_counter(C);
  unsigned smax = (unsigned)(single ? C.spin_max_ns1 : C.spin_max_ns);
  long long* tstamp = C.debug_tstamp;
  double *Y = nullptr, *Xh = nullptr;
  const int ksplit = (t == 1) ? 1 : std::max(1, std::min(16, H / 256));
  if (head) {
    C.head_Y.alloc(sizeof(double) * (size_t)H * t);
    C.head_Xh.alloc(sizeof(double) * (size_t)H * t * ksplit);
    Y = C.head_Y.as<double>();
    Xh = C.head_Xh.as<double>();
  }
  const int32_t* hrows = P.head_rows.as<int32_t>();
  auto run_head = [&](int slot_rhs, int slot_out) {
    const size_t hsm = red_smem_bytes<G, NU, U, NR>(kRowsThreads, t);
    if (fwd)
      head_rhs_kernel<G, NU, U, NR, false, Body, Fin><<<hgrid, kRowsThreads, hsm, C.stream>>>(
          H, t, ld, hrows, P.head_pos.as<int32_t>(), P.tptr.as<int32_t>(), P.tidx.as<int32_t>(),
          F.valT.as<double>(), x, Y, body, fin, partials, counter, slot_rhs, total, gate);
    else
      head_rhs_kernel<G, NU, U, NR, true, Body, Fin><<<hgrid, kRowsThreads, hsm, C.stream>>>(
          H, t, ld, hrows, P.head_pos.as<int32_t>(), P.tptr.as<int32_t>(), P.tidx.as<int32_t>(),
          F.valT.as<double>(), x, Y, body, fin, partials, counter, slot_rhs, total, gate);
    VL_LAUNCH_CHECK();
    if (t == 1) {
      if (fwd) head_gemv_kernel<false><<<H, kGemvThreads, 0, C.stream>>>(H, F.headXr.as<double>(), Y, Xh, gate);
      else head_gemv_kernel<true><<<H, kGemvThreads, 0, C.stream>>>(H, F.headX.as<double>(), Y, Xh, gate);
    } else {
      const size_t asm_ = sizeof(double) * 32 * (size_t)t;
      const dim3 ga((H + 31) / 32, ksplit);
      if (fwd) head_apply_kernel<false><<<ga, 256, asm_, C.stream>>>(H, t, F.headX.as<double>(), Y, Xh, gate);
      else head_apply_kernel<true><<<ga, 256, asm_, C.stream>>>(H, t, F.headX.as<double>(), Y, Xh, gate);
    }
    VL_LAUNCH_CHECK();
    head_out_kernel<G, NU, U, NR, Body, Fin><<<hgrid, kRowsThreads, hsm, C.stream>>>(
        H, t, ld, hrows, Xh, ksplit, x, body, fin, partials, counter, slot_out, total, gate);
    VL_LAUNCH_CHECK();
    if constexpr (PsumOf<Body>::value) {
      if (!fwd) {
        const int pl = (t == 1) ? 32 : G;
        const int pg = std::max(1, std::min(4 * C.num_sms, (int)((H * pl + kRowsThreads - 1) / kRowsThreads)));
        head_psum_kernel<G, NU, U, Body><<<pg, kRowsThreads, 0, C.stream>>>(
            H, t, ld, hrows, P.tptr.as<int32_t>(), P.tidx.as<int32_t>(), F.valT.as<double>(), x, body, gate);
        VL_LAUNCH_CHECK();
      }
    }
  };
  auto run_main = [&](int slot0) {
    if (single) {
      int sb = slot0;
      void* args[] = {(void*)&nitems, (void*)&npos,  (void*)&items,    (void*)&order,  (void*)&deps,
                      (void*)&x,      (void*)&body,  (void*)&fin,      (void*)&partials, (void*)&counter,
                      (void*)&gate,   (void*)&smax,  (void*)&tstamp,   (void*)&sb,     (void*)&total,
                      (void*)&sl};
#if VL_FRONT
      if (C.front.p == nullptr) {
        C.front.alloc(sizeof(unsigned) * 32);
        VL_CUDA(cudaMemsetAsync(C.front.p, 0, sizeof(unsigned) * 32, C.stream));
        C.front_total = 0;
      }
      sl.front = C.front.as<unsigned>();
      sl.fbase = C.front_total;
      if (nitems > 0) C.front_total += (unsigned)nitems;
#endif
      if (nitems > 0)
        VL_CUDA(cudaLaunchCooperativeKernel((const void*)k1, dim3(grid1), dim3(kRowsThreads), args, smem1,
                                            C.stream));
      return;
    }
    int slot = slot0;
    for (size_t i = 0; i < segs.size(); ++i) {
      TrsvLaunch Lc;
      Lc.L0 = segs[i].L0;
      Lc.L1 = segs[i].L1;
      Lc.p0 = tiled ? 0 : (*lptr)[segs[i].L0];
      Lc.p1 = tiled ? npos : (*lptr)[segs[i].L1];
      Lc.lptr = lptr_d;
      Lc.slot_base = slot;
      Lc.total_slots = total;
      slot += grids[i];
      if (segs[i].thin) {
        if (tsmem > 48 * 1024)
          VL_CUDA(cudaFuncSetAttribute(tkern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)tsmem));
        tkern<<<1, kThinThreads, tsmem, C.stream>>>(Lc, t, ld, order, deps, x, body, fin, partials, counter, gate,
                                                    tstamp);
        VL_LAUNCH_CHECK();
      } else {
        void* args[] = {(void*)&Lc,   (void*)&t,    (void*)&ld,       (void*)&order,   (void*)&deps,
                        (void*)&x,    (void*)&body, (void*)&fin,      (void*)&partials, (void*)&counter,
                        (void*)&gate, (void*)&smax, (void*)&tstamp};
        VL_CUDA(cudaLaunchCooperativeKernel((const void*)kern, dim3(grids[i]), dim3(kRowsThreads), args, smem,
                                            C.stream));
      }
    }
  };
  if (fwd) {
    if (head) run_head(main_slots, main_slots + hgrid);
    run_main(0);
  } else {
    run_main(0);
    if (head) run_head(main_slots, main_slots + hgrid);
  }
  if (ev) prof_end(C, ev);
  debug_sync(C, __PRETTY_FUNCTION__);
}

}  // namespace vl
