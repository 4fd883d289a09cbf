// Host-side pattern analysis (once per dataset): exact nearest-preceding
// neighbour search, storage permutation, dependency levels of B and B^T,
// children CSR (= B^T structure).  Follows the reference's definitions:
//   neighbour sets  vecchia.py:59-98  (m nearest among earlier points, ties
//                   to the smaller permuted index)
//   B pattern       vecchia.py:272-282 (row i = [N(i) in distance order, i])
#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstring>
#include <numeric>
#include <thread>
#include <vector>

#include "context.h"

namespace vl {

// ---------------------------------------------------------------------------
// Exact kNN among predecessors
// ---------------------------------------------------------------------------
namespace {

struct Cand {
  double d;
  int32_t i;
};
inline bool cand_less(const Cand& a, const Cand& b) { return a.d < b.d || (a.d == b.d && a.i < b.i); }

inline double dist(const double* a, const double* b, int d) {
  double s = 0.0;
  for (int k = 0; k < d; ++k) {
    double t = a[k] - b[k];
    s += t * t;
  }
  return std::sqrt(s);
}

// keep the `m` best candidates (sorted) in `best`
inline void offer(std::vector<Cand>& best, int m, Cand c) {
  if ((int)best.size() < m) {
    best.insert(std::upper_bound(best.begin(), best.end(), c, cand_less), c);
  } else if (cand_less(c, best.back())) {
    best.pop_back();
    best.insert(std::upper_bound(best.begin(), best.end(), c, cand_less), c);
  }
}

struct Grid {
  int d = 2;
  int dims[3] = {1, 1, 1};
  double lo[3] = {0, 0, 0};
  double h = 1.0;
  std::vector<int32_t> start;  // cell -> first index in items
  std::vector<int32_t> items;  // point ids sorted by cell

  int cell_coord(double x, int k) const {
    int c = (int)std::floor((x - lo[k]) / h);
    return std::min(std::max(c, 0), dims[k] - 1);
  }
};

void build_grid(Grid& g, const double* xy, int64_t npts, int d, int per_cell) {
  g.d = d;
  double hi[3] = {0, 0, 0};
  for (int k = 0; k < d; ++k) { g.lo[k] = 1e300; hi[k] = -1e300; }
  for (int64_t i = 0; i < npts; ++i)
    for (int k = 0; k < d; ++k) {
      g.lo[k] = std::min(g.lo[k], xy[i * d + k]);
      hi[k] = std::max(hi[k], xy[i * d + k]);
    }
  double vol = 1.0;
  int dd = 0;
  for (int k = 0; k < d; ++k) {
    double ext = hi[k] - g.lo[k];
    if (ext > 0) { vol *= ext; ++dd; }
  }
  double cells = std::max(1.0, (double)npts / per_cell);
  g.h = (dd == 0) ? 1.0 : std::pow(vol / cells, 1.0 / dd);
  if (!(g.h > 0)) g.h = 1.0;
  int64_t total = 1;
  for (int k = 0; k < 3; ++k) g.dims[k] = 1;
  for (int k = 0; k < d; ++k) {
    double ext = hi[k] - g.lo[k];
    g.dims[k] = std::max(1, (int)std::min(1e6, std::floor(ext / g.h) + 1));
    total *= g.dims[k];
  }
  std::vector<int32_t> cellof(npts);
  std::vector<int32_t> count(total + 1, 0);
  for (int64_t i = 0; i < npts; ++i) {
    int64_t c = 0;
    for (int k = d - 1; k >= 0; --k) c = c * g.dims[k] + g.cell_coord(xy[i * d + k], k);
    cellof[i] = (int32_t)c;
    count[c + 1]++;
  }
  for (int64_t c = 0; c < total; ++c) count[c + 1] += count[c];
  g.start = count;
  g.items.assign(npts, 0);
  std::vector<int32_t> fill(count.begin(), count.end() - 1);
  for (int64_t i = 0; i < npts; ++i) g.items[fill[cellof[i]]++] = (int32_t)i;  // ascending ids per cell
}

// ring search for query q among points with index < q
void grid_query(const Grid& g, const double* xy, int d, int64_t q, int take, std::vector<Cand>& best) {
  best.clear();
  const double* p = xy + q * d;
  int cq[3] = {0, 0, 0};
  for (int k = 0; k < d; ++k) cq[k] = g.cell_coord(p[k], k);
  int maxr = 0;
  for (int k = 0; k < d; ++k) maxr = std::max(maxr, std::max(cq[k], g.dims[k] - 1 - cq[k]));
  for (int r = 0; r <= maxr; ++r) {
    // lower bound on the distance of any point in ring r (cells at Chebyshev distance r)
    if ((int)best.size() == take && r > 0) {
      double lb = 1e300;
      for (int k = 0; k < d; ++k) {
        double frac_lo = (p[k] - (g.lo[k] + cq[k] * g.h));
        double frac_hi = (g.lo[k] + (cq[k] + 1) * g.h) - p[k];
        lb = std::min(lb, std::min(frac_lo, frac_hi) + (r - 1) * g.h);
      }
      if (lb > best.back().d) break;
    }
    int lo0 = cq[0] - r, hi0 = cq[0] + r;
    int lo1 = (d > 1) ? cq[1] - r : 0, hi1 = (d > 1) ? cq[1] + r : 0;
    int lo2 = (d > 2) ? cq[2] - r : 0, hi2 = (d > 2) ? cq[2] + r : 0;
    for (int c2 = lo2; c2 <= hi2; ++c2) {
      if (c2 < 0 || c2 >= g.dims[2]) continue;
      for (int c1 = lo1; c1 <= hi1; ++c1) {
        if (c1 < 0 || c1 >= g.dims[1]) continue;
        for (int c0 = lo0; c0 <= hi0; ++c0) {
          if (c0 < 0 || c0 >= g.dims[0]) continue;
          int cheb = std::max(std::abs(c0 - cq[0]), std::max(std::abs(c1 - (d > 1 ? cq[1] : 0)),
                                                             std::abs(c2 - (d > 2 ? cq[2] : 0))));
          if (cheb != r) continue;
          int64_t cell = ((int64_t)c2 * g.dims[1] + c1) * g.dims[0] + c0;
          for (int32_t it = g.start[cell]; it < g.start[cell + 1]; ++it) {
            int32_t j = g.items[it];
            if (j >= q) break;  // items are ascending within a cell
            offer(best, take, Cand{dist(p, xy + (int64_t)j * d, d), j});
          }
        }
      }
    }
  }
}

}  // namespace

// out: n*m int32, padded with -1. Exact: m nearest among indices < i, ties to
// the smaller index (the reference's brute-force definition).
void knn_previous(const double* xy, int64_t n, int d, int m, int32_t* out, int nthreads) {
  if (m <= 0) return;
  for (int64_t i = 0; i < n * m; ++i) out[i] = -1;
  if (n <= 1) return;
  if (nthreads <= 0) nthreads = (int)std::max(1u, std::thread::hardware_concurrency());
  const int64_t nbrute = std::min<int64_t>(n, 4096);
  auto brute = [&](int64_t i, std::vector<Cand>& best) {
    best.clear();
    int take = (int)std::min<int64_t>(i, m);
    for (int64_t j = 0; j < i; ++j) offer(best, take, Cand{dist(xy + i * d, xy + j * d, d), (int32_t)j});
  };
  auto write = [&](int64_t i, const std::vector<Cand>& best) {
    for (size_t k = 0; k < best.size(); ++k) out[i * m + k] = best[k].i;
  };
  // brute-force head (also used for d > 3)
  int64_t head = (d > 3) ? n : nbrute;
  {
    std::atomic<int64_t> next(1);
    std::vector<std::thread> th;
    for (int w = 0; w < nthreads; ++w)
      th.emplace_back([&] {
        std::vector<Cand> best;
        for (;;) {
          int64_t i = next.fetch_add(64);
          if (i >= head) break;
          for (int64_t q = i; q < std::min(head, i + 64); ++q) { brute(q, best); write(q, best); }
        }
      });
    for (auto& t : th) t.join();
  }
  // grid-accelerated tail on geometrically growing prefixes
  int64_t lo = head;
  while (lo < n) {
    int64_t hi = std::min<int64_t>(n, lo * 4);
    Grid g;
    build_grid(g, xy, hi, d, std::max(4, m / 2));
    std::atomic<int64_t> next(lo);
    std::vector<std::thread> th;
    for (int w = 0; w < nthreads; ++w)
      th.emplace_back([&] {
        std::vector<Cand> best;
        for (;;) {
          int64_t i = next.fetch_add(256);
          if (i >= hi) break;
          for (int64_t q = i; q < std::min(hi, i + 256); ++q) {
            grid_query(g, xy, d, q, (int)std::min<int64_t>(q, m), best);
            write(q, best);
          }
        }
      });
    for (auto& t : th) t.join();
    lo = hi;
  }
}

// ---------------------------------------------------------------------------
// Storage order
// ---------------------------------------------------------------------------
namespace {

uint64_t hilbert2(uint32_t x, uint32_t y, int order) {
  uint64_t dd = 0;
  for (int64_t s = (int64_t)1 << (order - 1); s > 0; s >>= 1) {
    uint32_t rx = (x & s) > 0, ry = (y & s) > 0;
    dd += (uint64_t)s * (uint64_t)s * ((3 * rx) ^ ry);
    if (ry == 0) {
      if (rx == 1) { x = (uint32_t)(s - 1) - x; y = (uint32_t)(s - 1) - y; }
      std::swap(x, y);
    }
  }
  return dd;
}

uint64_t morton3(uint32_t a, uint32_t b, uint32_t c) {
  auto spread = [](uint64_t v) {
    v &= 0x1fffff;
    v = (v | v << 32) & 0x1f00000000ffffULL;
    v = (v | v << 16) & 0x1f0000ff0000ffULL;
    v = (v | v << 8) & 0x100f00f00f00f00fULL;
    v = (v | v << 4) & 0x10c30c30c30c30c3ULL;
    v = (v | v << 2) & 0x1249249249249249ULL;
    return v;
  };
  return spread(a) | (spread(b) << 1) | (spread(c) << 2);
}

std::vector<uint64_t> spatial_keys(const double* xy, int64_t n, int d) {
  std::vector<uint64_t> key(n);
  double lo[3] = {1e300, 1e300, 1e300}, hi[3] = {-1e300, -1e300, -1e300};
  int dk = std::min(d, 3);
  for (int64_t i = 0; i < n; ++i)
    for (int k = 0; k < dk; ++k) {
      lo[k] = std::min(lo[k], xy[i * d + k]);
      hi[k] = std::max(hi[k], xy[i * d + k]);
    }
  auto q = [&](double v, int k, int bits) -> uint32_t {
    double ext = hi[k] - lo[k];
    if (!(ext > 0)) return 0;
    double f = (v - lo[k]) / ext;
    uint32_t mx = (1u << bits) - 1;
    double s = f * mx;
    return (uint32_t)std::min<double>(mx, std::max(0.0, s));
  };
  for (int64_t i = 0; i < n; ++i) {
    const double* p = xy + i * d;
    if (dk == 1) key[i] = q(p[0], 0, 31);
    else if (dk == 2) key[i] = hilbert2(q(p[0], 0, 16), q(p[1], 1, 16), 16);
    else key[i] = morton3(q(p[0], 0, 21), q(p[1], 1, 21), q(p[2], 2, 21));
  }
  return key;
}

}  // namespace

void pattern_build_host(Pattern& P, const double* xy, const int32_t* nbr, std::vector<int32_t>& ell,
                        std::vector<int32_t>& cnt, std::vector<int32_t>& fwd, std::vector<int32_t>& bwd,
                        std::vector<int32_t>& tptr, std::vector<int32_t>& tidx, std::vector<int32_t>& tmap) {
  const int64_t n = P.n;
  const int m = P.m;
  const int d = P.d;
  // neighbour counts + validation (factor order)
  std::vector<int32_t> cf(n, 0);
  for (int64_t i = 0; i < n; ++i) {
    int c = 0;
    for (int k = 0; k < m; ++k) {
      int32_t j = nbr[i * m + k];
      if (j < 0) break;
      if (j >= i) fail(kEConfig, "neighbour sets must reference earlier points only (row " + std::to_string(i) + ")");
      ++c;
    }
    for (int k = c; k < m; ++k)
      if (nbr[i * m + k] >= 0) fail(kEConfig, "neighbour rows must be left-packed (-1 padding at the end)");
    cf[i] = c;
  }
  // levels (forward) and heights (backward) in factor order
  std::vector<int32_t> lev(n, 0), hgt(n, 0);
  for (int64_t i = 0; i < n; ++i) {
    int L = 0;
    for (int k = 0; k < cf[i]; ++k) L = std::max(L, lev[nbr[i * m + k]] + 1);
    lev[i] = L;
  }
  for (int64_t i = n - 1; i >= 0; --i)
    for (int k = 0; k < cf[i]; ++k) {
      int32_t j = nbr[i * m + k];
      hgt[j] = std::max(hgt[j], hgt[i] + 1);
    }
  int nlev = 0, nhgt = 0;
  for (int64_t i = 0; i < n; ++i) { nlev = std::max(nlev, lev[i] + 1); nhgt = std::max(nhgt, hgt[i] + 1); }
  // storage permutation
  P.sperm.resize(n);
  std::iota(P.sperm.begin(), P.sperm.end(), 0);
  if (P.order_kind == 1 || P.order_kind == 2) {
    auto key = spatial_keys(xy, n, d);
    if (P.order_kind == 1) {
      std::stable_sort(P.sperm.begin(), P.sperm.end(), [&](int32_t a, int32_t b) { return key[a] < key[b]; });
    } else {
      std::stable_sort(P.sperm.begin(), P.sperm.end(), [&](int32_t a, int32_t b) {
        return lev[a] < lev[b] || (lev[a] == lev[b] && key[a] < key[b]);
      });
    }
  }
  P.iperm.assign(n, 0);
  for (int64_t s = 0; s < n; ++s) P.iperm[P.sperm[s]] = (int32_t)s;
  // ELL in storage order (pad with the storage slot of factor row 0, never read)
  ell.assign((size_t)n * std::max(m, 1), P.iperm[0]);
  cnt.assign(n, 0);
  int64_t nnz = 0;
  for (int64_t s = 0; s < n; ++s) {
    int32_t i = P.sperm[s];
    cnt[s] = cf[i];
    nnz += cf[i];
    for (int k = 0; k < cf[i]; ++k) ell[s * m + k] = P.iperm[nbr[(int64_t)i * m + k]];
  }
  P.nnz_off = nnz;
  if (nnz >= (int64_t)INT32_MAX) fail(kECapacity, "pattern too large for int32 CSR offsets");
  // schedules: rows ordered by (level, storage position)
  // each level padded with -1 to a multiple of 32 (rows of one warp-iteration
  // of the solve kernels are then always independent)
  auto bucket = [&](const std::vector<int32_t>& lv, int nl, std::vector<int32_t>& order, std::vector<int32_t>& ptr) {
    std::vector<int64_t> size(nl, 0);
    for (int64_t s = 0; s < n; ++s) size[lv[P.sperm[s]]]++;
    ptr.assign(nl + 1, 0);
    for (int l = 0; l < nl; ++l) ptr[l + 1] = ptr[l] + (int32_t)((size[l] + 31) / 32 * 32);
    order.assign(ptr[nl], -1);
    std::vector<int32_t> fill(ptr.begin(), ptr.end() - 1);
    for (int64_t s = 0; s < n; ++s) order[fill[lv[P.sperm[s]]]++] = (int32_t)s;
  };
  bucket(lev, nlev, fwd, P.fwd_level_ptr);
  bucket(hgt, nhgt, bwd, P.bwd_level_ptr);
  P.nlev_fwd = nlev;
  P.nlev_bwd = nhgt;
  // children CSR (transpose) in storage order, children ascending by storage row
  tptr.assign(n + 1, 0);
  for (int64_t s = 0; s < n; ++s)
    for (int k = 0; k < cnt[s]; ++k) tptr[ell[s * m + k] + 1]++;
  for (int64_t s = 0; s < n; ++s) tptr[s + 1] += tptr[s];
  tidx.assign(nnz, 0);
  tmap.assign(nnz, 0);
  std::vector<int32_t> fill(tptr.begin(), tptr.end() - 1);
  int maxc = 0;
  for (int64_t s = 0; s < n; ++s)
    for (int k = 0; k < cnt[s]; ++k) {
      int32_t p = ell[s * m + k];
      int32_t pos = fill[p]++;
      tidx[pos] = (int32_t)s;
      tmap[pos] = (int32_t)(s * m + k);
    }
  for (int64_t s = 0; s < n; ++s) maxc = std::max(maxc, tptr[s + 1] - tptr[s]);
  P.max_children = maxc;
  // Children that finish late in the backward solve (height within child_late of the parent's)
  // go to the end of the parent's list, by height: the multi-column solve gathers a row's
  // dependencies batch by batch, so the batches of long-finished children no longer queue
  // behind the one child the row is actually waiting for.  The others stay in storage order.
  if (P.child_late > 0) {
    std::vector<std::pair<int32_t, int32_t>> early, late;
    for (int64_t s = 0; s < n; ++s) {
      const int32_t e0 = tptr[s], e1 = tptr[s + 1];
      if (e1 - e0 < 2) continue;
      const int hp = hgt[P.sperm[s]];
      early.clear();
      late.clear();
      for (int32_t e = e0; e < e1; ++e) {
        const int hc = hgt[P.sperm[tidx[e]]];
        (hc >= hp - P.child_late ? late : early).push_back({tidx[e], tmap[e]});
      }
      if (late.empty()) continue;
      std::stable_sort(late.begin(), late.end(), [&](const auto& a, const auto& b) {
        return hgt[P.sperm[a.first]] < hgt[P.sperm[b.first]];
      });
      int32_t e = e0;
      for (auto& c : early) { tidx[e] = c.first; tmap[e] = c.second; ++e; }
      for (auto& c : late) { tidx[e] = c.first; tmap[e] = c.second; ++e; }
    }
  }
  // The same for the forward solve: a copy of the ELL rows with the late parents (level within
  // child_late of the row's) last, by level; map_s = slot of the value in Factor::val.  The
  // reference's in-row order (ell / Factor::val) stays what the factor build and the products use.
  P.nbr_s_h.clear();
  P.map_s_h.clear();
  if (P.child_late > 0 && m > 0) {
    P.nbr_s_h = ell;
    P.map_s_h.assign((size_t)n * m, -1);
    std::vector<int> early, late;
    for (int64_t s = 0; s < n; ++s) {
      const int lr = lev[P.sperm[s]];
      early.clear();
      late.clear();
      for (int k = 0; k < cnt[s]; ++k)
        (lev[P.sperm[ell[s * m + k]]] >= lr - P.child_late ? late : early).push_back(k);
      std::stable_sort(late.begin(), late.end(), [&](int a, int b) {
        return lev[P.sperm[ell[s * m + a]]] < lev[P.sperm[ell[s * m + b]]];
      });
      int q = 0;
      for (int k : early) { P.nbr_s_h[s * m + q] = ell[s * m + k]; P.map_s_h[s * m + q] = (int32_t)(s * m + k); ++q; }
      for (int k : late) { P.nbr_s_h[s * m + q] = ell[s * m + k]; P.map_s_h[s * m + q] = (int32_t)(s * m + k); ++q; }
    }
  }

  // ---- dense head block -----------------------------------------------------
  // Rows of forward levels < Lh form a closed block (their neighbours have
  // lower levels) and no row outside it has a child inside it.  Its inverse
  // X = B_HH^-1 (dense, recomputed per factor) replaces Lh dependency hops in
  // both solves: forward x_H = X y_H first; backward x_H = X^T (y_H - B_RH^T x_R)
  // last.  Lh is the largest prefix with at most head_max rows.
  std::vector<int64_t> lsize(nlev, 0);
  for (int64_t i = 0; i < n; ++i) lsize[lev[i]]++;
  int Lh = 0;
  int64_t H = 0;
  while (Lh < nlev && H + lsize[Lh] <= P.head_max) H += lsize[Lh++];
  if (Lh < 8 || Lh >= nlev) { Lh = 0; H = 0; }
  P.head_L = Lh;
  P.head_H = H;
  P.head_rows_h.clear();
  P.head_pos_h.assign(n, -1);
  for (int32_t p = P.fwd_level_ptr[0]; p < (Lh ? P.fwd_level_ptr[Lh] : 0); ++p) {
    const int32_t s = fwd[p];
    if (s < 0) continue;
    P.head_pos_h[s] = (int32_t)P.head_rows_h.size();
    P.head_rows_h.push_back(s);
  }
  P.head_nbr_h.assign((size_t)std::max<int64_t>(H, 1) * std::max(m, 1), -1);
  for (int64_t h = 0; h < H; ++h) {
    const int32_t s = P.head_rows_h[h];
    for (int k = 0; k < cnt[s]; ++k) {
      const int32_t hp = P.head_pos_h[ell[s * m + k]];
      if (hp < 0) fail(kEInternal, "head block is not closed");
      P.head_nbr_h[h * m + k] = hp;
    }
  }
  // backward schedule restricted to the rows outside the head (by height)
  {
    std::vector<int64_t> size(nhgt, 0);
    for (int64_t s = 0; s < n; ++s)
      if (P.head_pos_h[s] < 0) size[hgt[P.sperm[s]]]++;
    P.bwdnh_level_ptr.assign(nhgt + 1, 0);
    for (int l = 0; l < nhgt; ++l) P.bwdnh_level_ptr[l + 1] = P.bwdnh_level_ptr[l] + (int32_t)((size[l] + 31) / 32 * 32);
    P.bwdnh_order_h.assign(P.bwdnh_level_ptr[nhgt], -1);
    std::vector<int32_t> fl(P.bwdnh_level_ptr.begin(), P.bwdnh_level_ptr.end() - 1);
    for (int64_t s = 0; s < n; ++s)
      if (P.head_pos_h[s] < 0) P.bwdnh_order_h[fl[hgt[P.sperm[s]]]++] = (int32_t)s;
  }

  // ---- tile-blocked order of the multi-column solves --------------------------
  // In level order a row's m gathered rows of x were written (or last read) tens
  // of levels ago; with t = 50 columns x is 3x the L2, so most gathers go to HBM
  // (ncu: L2 hit 35 %, 4.6x the algorithmic bytes).  The sync-free solve only
  // needs SOME topological order of the rows, so the wide levels are cut into
  // bands of tile_K levels and every band is walked tile by tile (a tile = a run
  // of storage positions, i.e. a Hilbert-contiguous patch), level by level inside
  // the tile: a patch's neighbour rows are then gathered K times while they sit
  // in L2.  A row whose dependency (same band) lies in a later tile moves to that
  // tile, which keeps the order topological without any geometric assumption; a
  // pattern without locality degenerates to the level order.  Each row's own
  // arithmetic is unchanged.  (LRU model of the bench pattern, 60 MB of rows:
  // forward gather misses 12.1 M -> 0.8 M, backward 15.6 M -> 7.1 M.)
  P.fwd_torder_h.clear();
  P.bwd_torder_h.clear();
  if (P.tile_K > 0 && P.tile_S > 1 && P.order_kind == 1 && n >= P.tile_min_n) {
    auto tiled = [&](bool fwd_dir, std::vector<int32_t>& out) {
      const std::vector<int32_t>& lvf = fwd_dir ? lev : hgt;
      const int nl = fwd_dir ? nlev : nhgt;
      auto ndeps = [&](int32_t s) { return fwd_dir ? cnt[s] : tptr[s + 1] - tptr[s]; };
      auto dep = [&](int32_t s, int k) { return fwd_dir ? ell[(size_t)s * m + k] : tidx[tptr[s] + k]; };
      std::vector<int32_t> lv(n);
      std::vector<int64_t> sz(nl, 0);
      for (int64_t s = 0; s < n; ++s) {
        lv[s] = lvf[P.sperm[s]];
        if (P.head_pos_h[s] < 0) sz[lv[s]]++;
      }
      // the wide run of levels around the largest one
      const int lmax = (int)(std::max_element(sz.begin(), sz.end()) - sz.begin());
      if (sz[lmax] < P.tile_min_rows) return;
      int b0 = lmax, b1 = lmax + 1;
      while (b0 > 0 && sz[b0 - 1] >= P.tile_min_rows) --b0;
      while (b1 < nl && sz[b1] >= P.tile_min_rows) ++b1;
      const int wide1 = b1;
      // a short narrow tail after the wide run joins the last band: its rows then run inside
      // their tiles, hidden behind the later tiles, instead of as a latency chain at the end
      if (P.tile_tail) {
        int64_t tail = 0;
        for (int l = b1; l < nl; ++l) tail += sz[l];
        if (tail * 20 < n) b1 = nl;
      }
      // rows outside the head in (level, storage position) order
      std::vector<int64_t> ptr(nl + 1, 0);
      for (int l = 0; l < nl; ++l) ptr[l + 1] = ptr[l] + sz[l];
      std::vector<int32_t> lo(ptr[nl]);
      {
        std::vector<int64_t> fl(ptr.begin(), ptr.end() - 1);
        for (int64_t s = 0; s < n; ++s)
          if (P.head_pos_h[s] < 0) lo[fl[lv[s]]++] = (int32_t)s;
      }
      // bands of tile_K levels; the tail levels (if joined) belong to the last band of the wide run
      const int nband = std::max(1, (wide1 - b0 + P.tile_K - 1) / P.tile_K);
      std::vector<int32_t> tile(n, 0);
      for (int64_t q = ptr[b0]; q < ptr[b1]; ++q) {
        const int32_t s = lo[q];
        const int band = std::min((lv[s] - b0) / P.tile_K, nband - 1);
        int tl = (int)((int64_t)s * P.tile_S / n);
        for (int k = 0; k < ndeps(s); ++k) {
          const int32_t dd = dep(s, k);
          if (P.head_pos_h[dd] >= 0 || lv[dd] < b0 || lv[dd] >= b1) continue;
          if (std::min((lv[dd] - b0) / P.tile_K, nband - 1) == band) tl = std::max(tl, tile[dd]);
        }
        tile[s] = tl;
      }
      std::vector<int32_t> bulk(lo.begin() + ptr[b0], lo.begin() + ptr[b1]);
      std::stable_sort(bulk.begin(), bulk.end(), [&](int32_t a, int32_t b) {
        const int ba = std::min((lv[a] - b0) / P.tile_K, nband - 1), bb = std::min((lv[b] - b0) / P.tile_K, nband - 1);
        if (ba != bb) return ba < bb;
        if (tile[a] != tile[b]) return tile[a] < tile[b];
        return lv[a] < lv[b];  // stable: storage position within a level
      });
      // every run of one level (inside one tile) is padded to 32 positions with -1, like the
      // levels of the level order: the rows a warp takes together (32 / G of them) are then
      // always independent, whatever G is
      out.clear();
      auto pad = [&]() { out.resize((out.size() + 31) / 32 * 32, -1); };
      for (int l = 0; l < b0; ++l) {
        out.insert(out.end(), lo.begin() + ptr[l], lo.begin() + ptr[l + 1]);
        pad();
      }
      for (size_t q = 0; q < bulk.size(); ++q) {
        if (q > 0 && (lv[bulk[q]] != lv[bulk[q - 1]] || tile[bulk[q]] != tile[bulk[q - 1]])) pad();
        out.push_back(bulk[q]);
      }
      pad();
      for (int l = b1; l < nl; ++l) {
        out.insert(out.end(), lo.begin() + ptr[l], lo.begin() + ptr[l + 1]);
        pad();
      }
    };
    tiled(true, P.fwd_torder_h);
    tiled(false, P.bwd_torder_h);
  }
}

}  // namespace vl
