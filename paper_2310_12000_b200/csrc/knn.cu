// Exact k-nearest-neighbour search on the device (once per dataset / per
// prediction set):
//   * nearest PRECEDING neighbours along the ordering (vecchia.py:59-98):
//     the min(i, m) points among positions 0..i-1 closest in Euclidean
//     distance, ties to the smaller index;
//   * nearest TRAINING neighbours of prediction points (vecchia.py:411-421):
//     the min(m, n) closest training points, ties to the smaller index.
// Brute force below 4096 points (one thread per query), then uniform grids
// over geometrically growing prefixes (points [0, hi) for the queries in
// [lo, hi), hi = 4 lo, so at least a quarter of a grid's points precede every
// query) searched ring by ring with the same lower-bound stop rule and the
// same (distance, index) order as the host implementation in pattern.cpp.
#include <algorithm>
#include <cmath>
#include <vector>

#include "common.cuh"
#include "context.h"
#include "ops.h"

namespace vl {

namespace {

constexpr int kBrute = 4096;

struct DevGrid {
  const int32_t* start;  // cell -> first slot
  const int32_t* items;  // point ids, ascending within a cell
  int dims[3];
  double lo[3];
  double h;
};

struct HostGrid {
  int dims[3] = {1, 1, 1};
  double lo[3] = {0, 0, 0};
  double h = 1.0;
  std::vector<int32_t> start, items;
};

int cell_coord(const HostGrid& g, double x, int k) {
  int c = (int)std::floor((x - g.lo[k]) / g.h);
  return std::min(std::max(c, 0), g.dims[k] - 1);
}

void build_grid(HostGrid& g, const double* xy, int64_t npts, int d, int per_cell) {
  double hi[3] = {0, 0, 0};
  for (int k = 0; k < d; ++k) {
    g.lo[k] = 1e300;
    hi[k] = -1e300;
  }
  for (int64_t i = 0; i < npts; ++i)
    for (int k = 0; k < d; ++k) {
      g.lo[k] = std::min(g.lo[k], xy[i * d + k]);
      hi[k] = std::max(hi[k], xy[i * d + k]);
    }
  double vol = 1.0;
  int dd = 0;
  for (int k = 0; k < d; ++k) {
    const double ext = hi[k] - g.lo[k];
    if (ext > 0) {
      vol *= ext;
      ++dd;
    }
  }
  const double cells = std::max(1.0, (double)npts / per_cell);
  g.h = (dd == 0) ? 1.0 : std::pow(vol / cells, 1.0 / dd);
  if (!(g.h > 0)) g.h = 1.0;
  int64_t total = 1;
  for (int k = 0; k < 3; ++k) g.dims[k] = 1;
  for (int k = 0; k < d; ++k) {
    const double ext = hi[k] - g.lo[k];
    g.dims[k] = std::max(1, (int)std::min(1e6, std::floor(ext / g.h) + 1));
    total *= g.dims[k];
  }
  std::vector<int32_t> cellof(npts);
  std::vector<int32_t> count(total + 1, 0);
  for (int64_t i = 0; i < npts; ++i) {
    int64_t c = 0;
    for (int k = d - 1; k >= 0; --k) c = c * g.dims[k] + cell_coord(g, xy[i * d + k], k);
    cellof[i] = (int32_t)c;
    count[c + 1]++;
  }
  for (int64_t c = 0; c < total; ++c) count[c + 1] += count[c];
  g.start = count;
  g.items.assign(npts, 0);
  std::vector<int32_t> fill(count.begin(), count.end() - 1);
  for (int64_t i = 0; i < npts; ++i) g.items[fill[cellof[i]]++] = (int32_t)i;
}

VL_D double pdist(const double* a, const double* b, int d) {
  double s = 0.0;
  for (int k = 0; k < d; ++k) {
    const double t = a[k] - b[k];
    s += t * t;
  }
  return sqrt(s);
}

// sorted candidate list (distance, index) of capacity K, `take` kept
template <int K>
struct Best {
  double d[K];
  int32_t i[K];
  int n = 0;
  VL_D void offer(double dc, int32_t ic, int take) {
    if (n == take) {
      if (!(dc < d[n - 1] || (dc == d[n - 1] && ic < i[n - 1]))) return;
      --n;
    }
    int p = n;
    while (p > 0 && (dc < d[p - 1] || (dc == d[p - 1] && ic < i[p - 1]))) {
      d[p] = d[p - 1];
      i[p] = i[p - 1];
      --p;
    }
    d[p] = dc;
    i[p] = ic;
    ++n;
  }
};

// queries q in [q0, q1); candidates j < lim(q) (= q for preceding, = n_all for training)
template <int K>
__global__ void knn_brute_kernel(const double* __restrict__ pts, const double* __restrict__ qxy, int64_t q0,
                                 int64_t q1, int64_t n_all, int d, int m, int preceding, int32_t* __restrict__ out,
                                 double* __restrict__ dmin) {
  for (int64_t q = q0 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < q1;
       q += (int64_t)gridDim.x * blockDim.x) {
    const int64_t lim = preceding ? q : n_all;
    const int take = (int)(lim < m ? lim : m);
    const double* p = (preceding ? pts : qxy) + q * d;
    Best<K> b;
    for (int64_t j = 0; j < lim; ++j) b.offer(pdist(p, pts + j * d, d), (int32_t)j, take);
    for (int k = 0; k < b.n; ++k) out[q * m + k] = b.i[k];
    if (dmin) dmin[q] = b.n ? b.d[0] : INFINITY;
  }
}

template <int K>
__global__ void knn_grid_kernel(const double* __restrict__ pts, const double* __restrict__ qxy, DevGrid g,
                                int64_t q0, int64_t q1, int64_t n_all, int d, int m, int preceding,
                                int32_t* __restrict__ out, double* __restrict__ dmin) {
  for (int64_t q = q0 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < q1;
       q += (int64_t)gridDim.x * blockDim.x) {
    const int64_t lim = preceding ? q : n_all;
    const int take = (int)(lim < m ? lim : m);
    const double* p = (preceding ? pts : qxy) + q * d;
    int cq[3] = {0, 0, 0};
    for (int k = 0; k < d; ++k) {
      int c = (int)floor((p[k] - g.lo[k]) / g.h);
      cq[k] = c < 0 ? 0 : (c > g.dims[k] - 1 ? g.dims[k] - 1 : c);
    }
    int maxr = 0;
    for (int k = 0; k < d; ++k) {
      const int a = cq[k] > g.dims[k] - 1 - cq[k] ? cq[k] : g.dims[k] - 1 - cq[k];
      maxr = a > maxr ? a : maxr;
    }
    Best<K> b;
    for (int r = 0; r <= maxr; ++r) {
      if (b.n == take && r > 0) {
        double lb = 1e300;
        for (int k = 0; k < d; ++k) {
          const double flo = p[k] - (g.lo[k] + cq[k] * g.h);
          const double fhi = (g.lo[k] + (cq[k] + 1) * g.h) - p[k];
          lb = fmin(lb, fmin(flo, fhi) + (r - 1) * g.h);
        }
        if (lb > b.d[b.n - 1]) break;
      }
      const int lo0 = cq[0] - r, hi0 = cq[0] + r;
      const int lo1 = d > 1 ? cq[1] - r : 0, hi1 = d > 1 ? cq[1] + r : 0;
      const int lo2 = d > 2 ? cq[2] - r : 0, hi2 = d > 2 ? cq[2] + r : 0;
      for (int c2 = lo2; c2 <= hi2; ++c2) {
        if (c2 < 0 || c2 >= g.dims[2]) continue;
        for (int c1 = lo1; c1 <= hi1; ++c1) {
          if (c1 < 0 || c1 >= g.dims[1]) continue;
          const bool edge12 = abs(c1 - cq[1]) == r || abs(c2 - cq[2]) == r;
          // interior rows of the ring only touch its two end cells
          const int step = edge12 ? 1 : (hi0 - lo0 > 0 ? hi0 - lo0 : 1);
          for (int c0 = lo0; c0 <= hi0; c0 += step) {
            if (c0 < 0 || c0 >= g.dims[0]) continue;
            const int64_t cell = ((int64_t)c2 * g.dims[1] + c1) * g.dims[0] + c0;
            const int32_t e = g.start[cell + 1];
            for (int32_t it = g.start[cell]; it < e; ++it) {
              const int32_t j = g.items[it];
              if (j >= lim) break;  // ascending within a cell
              b.offer(pdist(p, pts + (int64_t)j * d, d), j, take);
            }
          }
        }
      }
    }
    for (int k = 0; k < b.n; ++k) out[q * m + k] = b.i[k];
    if (dmin) dmin[q] = b.n ? b.d[0] : INFINITY;
  }
}

template <int K>
void launch_brute(Ctx& C, const double* pts, const double* qxy, int64_t q0, int64_t q1, int64_t n_all, int d, int m,
                  int preceding, int32_t* out, double* dmin) {
  if (q1 <= q0) return;
  const int blocks = (int)std::min<int64_t>((q1 - q0 + 127) / 128, (int64_t)C.num_sms * 8);
  knn_brute_kernel<K><<<blocks, 128, 0, C.stream>>>(pts, qxy, q0, q1, n_all, d, m, preceding, out, dmin);
  VL_LAUNCH_CHECK();
}

template <int K>
void launch_grid(Ctx& C, const double* pts, const double* qxy, const DevGrid& g, int64_t q0, int64_t q1,
                 int64_t n_all, int d, int m, int preceding, int32_t* out, double* dmin) {
  if (q1 <= q0) return;
  const int blocks = (int)std::min<int64_t>((q1 - q0 + 127) / 128, (int64_t)C.num_sms * 16);
  knn_grid_kernel<K><<<blocks, 128, 0, C.stream>>>(pts, qxy, g, q0, q1, n_all, d, m, preceding, out, dmin);
  VL_LAUNCH_CHECK();
}

template <class F>
void with_k(int m, F&& f) {
  if (m <= 16) f(std::integral_constant<int, 16>{});
  else if (m <= 32) f(std::integral_constant<int, 32>{});
  else if (m <= 64) f(std::integral_constant<int, 64>{});
  else if (m <= 128) f(std::integral_constant<int, 128>{});
  else f(std::integral_constant<int, 256>{});
}

DevGrid upload_grid(Ctx& C, const HostGrid& hg, DevBuf& bs, DevBuf& bi) {
  bs.alloc(sizeof(int32_t) * hg.start.size());
  bi.alloc(sizeof(int32_t) * std::max<size_t>(hg.items.size(), 1));
  VL_CUDA(cudaMemcpyAsync(bs.p, hg.start.data(), sizeof(int32_t) * hg.start.size(), cudaMemcpyHostToDevice,
                          C.stream));
  if (!hg.items.empty())
    VL_CUDA(cudaMemcpyAsync(bi.p, hg.items.data(), sizeof(int32_t) * hg.items.size(), cudaMemcpyHostToDevice,
                            C.stream));
  DevGrid g;
  g.start = bs.as<int32_t>();
  g.items = bi.as<int32_t>();
  for (int k = 0; k < 3; ++k) {
    g.dims[k] = hg.dims[k];
    g.lo[k] = hg.lo[k];
  }
  g.h = hg.h;
  return g;
}

}  // namespace

// out (host): n*m int32 padded with -1
void knn_previous_dev(Ctx& C, const double* xy_host, int64_t n, int d, int m, int32_t* out_host) {
  if (m < 0) fail(kEConfig, "m must be >= 0");
  if (d < 1 || d > 3) fail(kECapability, "device neighbour search supports 1 <= d <= 3");
  if (m > 256) fail(kECapability, "device neighbour search supports m <= 256");
  for (int64_t i = 0; i < n * (int64_t)m; ++i) out_host[i] = -1;
  if (m == 0 || n <= 1) return;
  DevBuf pts, out;
  pts.alloc(sizeof(double) * n * d);
  out.alloc(sizeof(int32_t) * n * m);
  VL_CUDA(cudaMemcpyAsync(pts.p, xy_host, sizeof(double) * n * d, cudaMemcpyHostToDevice, C.stream));
  VL_CUDA(cudaMemsetAsync(out.p, 0xFF, sizeof(int32_t) * n * m, C.stream));
  const int64_t head = std::min<int64_t>(n, kBrute);
  with_k(m, [&](auto kk) {
    constexpr int K = decltype(kk)::value;
    launch_brute<K>(C, pts.as<double>(), nullptr, 1, head, n, d, m, 1, out.as<int32_t>(), nullptr);
    int64_t lo = head;
    std::vector<HostGrid> grids;
    std::vector<DevBuf> bufs;
    bufs.reserve(64);
    while (lo < n) {
      const int64_t hi = std::min<int64_t>(n, lo * 4);
      grids.emplace_back();
      build_grid(grids.back(), xy_host, hi, d, std::max(4, m / 2));
      bufs.emplace_back();
      bufs.emplace_back();
      DevGrid g = upload_grid(C, grids.back(), bufs[bufs.size() - 2], bufs.back());
      launch_grid<K>(C, pts.as<double>(), nullptr, g, lo, hi, n, d, m, 1, out.as<int32_t>(), nullptr);
      lo = hi;
    }
    VL_CUDA(cudaMemcpyAsync(out_host, out.p, sizeof(int32_t) * n * m, cudaMemcpyDeviceToHost, C.stream));
    VL_CUDA(cudaStreamSynchronize(C.stream));
  });
}

// m nearest training points of each query (take = min(m, n)); dmin_host: nearest distance
void knn_query_dev(Ctx& C, const double* train_host, int64_t n, const double* q_host, int64_t nq, int d, int m,
                   int32_t* out_host, double* dmin_host) {
  if (m < 1) fail(kEConfig, "prediction requires m >= 1");
  if (d < 1 || d > 3) fail(kECapability, "device neighbour search supports 1 <= d <= 3");
  if (m > 256) fail(kECapability, "device neighbour search supports m <= 256");
  if (nq == 0) return;
  DevBuf pts, qp, out, dm;
  pts.alloc(sizeof(double) * n * d);
  qp.alloc(sizeof(double) * nq * d);
  out.alloc(sizeof(int32_t) * nq * m);
  dm.alloc(sizeof(double) * nq);
  VL_CUDA(cudaMemcpyAsync(pts.p, train_host, sizeof(double) * n * d, cudaMemcpyHostToDevice, C.stream));
  VL_CUDA(cudaMemcpyAsync(qp.p, q_host, sizeof(double) * nq * d, cudaMemcpyHostToDevice, C.stream));
  VL_CUDA(cudaMemsetAsync(out.p, 0xFF, sizeof(int32_t) * nq * m, C.stream));
  with_k(m, [&](auto kk) {
    constexpr int K = decltype(kk)::value;
    HostGrid hg;
    DevBuf bs, bi;
    if (n <= kBrute) {
      launch_brute<K>(C, pts.as<double>(), qp.as<double>(), 0, nq, n, d, m, 0, out.as<int32_t>(), dm.as<double>());
    } else {
      build_grid(hg, train_host, n, d, std::max(4, m / 2));
      DevGrid g = upload_grid(C, hg, bs, bi);
      launch_grid<K>(C, pts.as<double>(), qp.as<double>(), g, 0, nq, n, d, m, 0, out.as<int32_t>(), dm.as<double>());
    }
    VL_CUDA(cudaMemcpyAsync(out_host, out.p, sizeof(int32_t) * nq * m, cudaMemcpyDeviceToHost, C.stream));
    VL_CUDA(cudaMemcpyAsync(dmin_host, dm.p, sizeof(double) * nq, cudaMemcpyDeviceToHost, C.stream));
    VL_CUDA(cudaStreamSynchronize(C.stream));
  });
}

}  // namespace vl
