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
}

}  // namespace vl
