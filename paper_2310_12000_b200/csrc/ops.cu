// Kernel-level operators on a factor: B x, B^T x, dB x, B^-1 x, B^-T x.
// (vecchia.py:161-192 solve_B / apply_precision / apply_sigma_tilde and the
//  csr/csc matvecs they call.)  All vectors are n x t row-major, storage order.
#include <map>
#include <mutex>

#include "bodies.cuh"
#include "launch.cuh"
#include "ops.h"

namespace vl {

unsigned* next_counter(Ctx& C) {
  unsigned* base = C.red_counter.as<unsigned>();
  int slot = C.red_slot;
  C.red_slot = (C.red_slot + 1) & 63;
  return base + slot;
}

cudaEvent_t prof_begin(Ctx& C, cudaStream_t st) {
  Prof& P = C.prof;
  auto take = [&]() {
    cudaEvent_t e;
    if (!P.free_events.empty()) {
      e = P.free_events.back();
      P.free_events.pop_back();
    } else {
      VL_CUDA(cudaEventCreate(&e));
    }
    return e;
  };
  cudaEvent_t a = take();
  VL_CUDA(cudaEventRecord(a, st ? st : C.stream));
  return a;
}

void prof_end(Ctx& C, cudaEvent_t a, cudaStream_t st) {
  Prof& P = C.prof;
  cudaEvent_t b;
  if (!P.free_events.empty()) {
    b = P.free_events.back();
    P.free_events.pop_back();
  } else {
    VL_CUDA(cudaEventCreate(&b));
  }
  VL_CUDA(cudaEventRecord(b, st ? st : C.stream));
  P.pending.push_back({std::string(P.tag), a, b, P.bytes});
}

void prof_collect(Ctx& C) {
  Prof& P = C.prof;
  if (P.pending.empty()) return;
  VL_CUDA(cudaStreamSynchronize(C.stream));
  for (auto& r : P.pending) {
    float ms = 0.f;
    VL_CUDA(cudaEventElapsedTime(&ms, r.a, r.b));
    Prof::Agg* g = nullptr;
    for (auto& kv : P.agg)
      if (kv.first == r.tag) g = &kv.second;
    if (!g) {
      P.agg.push_back({r.tag, Prof::Agg{}});
      g = &P.agg.back().second;
    }
    g->count += 1;
    g->ms += ms;
    g->bytes += r.bytes;
    P.free_events.push_back(r.a);
    P.free_events.push_back(r.b);
  }
  P.pending.clear();
}

std::vector<Seg> solve_segments(const std::vector<int32_t>& lptr, int thin_rows, int min_thick_levels) {
  std::vector<Seg> segs;
  const int nl = (int)lptr.size() - 1;
  int L = 0;
  while (L < nl) {
    const bool thin = (lptr[L + 1] - lptr[L]) <= thin_rows;
    int E = L + 1;
    while (E < nl && ((lptr[E + 1] - lptr[E]) <= thin_rows) == thin) ++E;
    segs.push_back({L, E, thin});
    L = E;
  }
  // short thick runs are cheaper on the single CTA than a grid launch
  for (auto& s : segs)
    if (!s.thin && s.L1 - s.L0 < min_thick_levels) s.thin = true;
  std::vector<Seg> merged;
  for (auto& s : segs) {
    if (!merged.empty() && merged.back().thin == s.thin) merged.back().L1 = s.L1;
    else merged.push_back(s);
  }
  return merged;
}

int coop_grid(Ctx& C, const void* func, size_t smem) {
  static std::mutex mu;
  static std::map<std::pair<const void*, size_t>, int> cache;
  std::lock_guard<std::mutex> lk(mu);
  auto key = std::make_pair(func, smem);
  auto it = cache.find(key);
  if (it != cache.end()) return it->second;
  int occ = 0;
  VL_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, func, kRowsThreads, smem));
  if (occ < 1) fail(kEInternal, "triangular-solve kernel cannot be made resident");
  int g = occ * C.num_sms;
  cache[key] = g;
  return g;
}

BView bview(const Factor& F, bool grad) {
  const Pattern& P = *F.pat;
  BView v;
  v.nbr = P.nbr.as<int32_t>();
  v.cnt = P.cnt.as<int32_t>();
  v.val = grad ? F.dval.as<double>() : F.val.as<double>();
  v.tptr = P.tptr.as<int32_t>();
  v.tidx = P.tidx.as<int32_t>();
  v.valT = F.valT.as<double>();
  v.m = P.m;
  v.nnzT = P.nnz_off;
  return v;
}

void op_spmm(Ctx& C, const Factor& F, int op, int t, int ld, const double* x, double* y) {
  const Pattern& P = *F.pat;
  if (op == 2 && !F.has_grad) fail(kEConfig, "factor was built without gradient");
  BView B = bview(F, false);
  dispatch_cols(t, ld, [&](auto g, auto nu, auto u) {
    constexpr int G = decltype(g)::value, NU = decltype(nu)::value, U = decltype(u)::value;
    if (op == 0) launch_rows_local<G, NU, U, 0, 0>(C, P, P.n, t, BodyBx{B, F.val.as<double>(), x, y, ld, 1}, Fin0<0>{});
    else if (op == 1)
      launch_rows_local<G, NU, U, 0, 0>(C, P, P.n, t, BodyBtx{B, x, y, ld}, Fin0<0>{}, nullptr, P.tptr.as<int32_t>());
    else if (op == 2)
      launch_rows_local<G, NU, U, 0, 0>(C, P, P.n, t, BodyBx{B, F.dval.as<double>(), x, y, ld, 0}, Fin0<0>{});
    else fail(kEConfig, "unknown product op");
  });
}

void op_trsv(Ctx& C, const Factor& F, bool transpose, int t, int ld, const double* b, double* x) {
  const Pattern& P = *F.pat;
  if (b == x) fail(kEConfig, "triangular solve cannot run in place");
  // the dense head block works on H x t panels: a padded leading dimension would leave the
  // pad column of the head rows at the "not ready" sentinel and the dependent rows polling
  if (t > 1 && ld != t) fail(kEConfig, "multi-column triangular solves need contiguous columns (ld == t)");
  dispatch_cols(t, ld, [&](auto g, auto nu, auto u) {
    constexpr int G = decltype(g)::value, NU = decltype(nu)::value, U = decltype(u)::value;
    if (!transpose) {
      DepsEll deps = deps_fwd(F);
      launch_trsv<G, NU, U, 0>(C, F,true, t, ld, deps, x, TrsvPlain{b, ld},
                               Fin0<0>{});
    } else {
      DepsCsr deps{P.tptr.as<int32_t>(), P.tidx.as<int32_t>(), F.valT.as<double>()};
      launch_trsv<G, NU, U, 0>(C, F,false, t, ld, deps, x, TrsvPlain{b, ld},
                               Fin0<0>{});
    }
  });
}

}  // namespace vl
