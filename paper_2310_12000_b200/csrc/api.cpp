// C-ABI entry points (include/vlgpx.h).  Exceptions never cross the ABI:
// every call maps failures onto a status code + thread-local message.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>
#include <map>
#include <mutex>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/vlgpx.h"
#include "laplace.h"
#include "lrac.h"
#include "ops.h"
#include "predict.h"
#include "dense.h"
#include "pcg.h"

struct vl_ctx {
  vl::Ctx c;
};
struct vl_pattern {
  vl::Pattern p;
  vl_ctx* ctx;
};
struct vl_factor {
  vl::Factor f;
};
struct vl_pred {
  vl::PredBlocks b;
};
struct vl_lrac {
  vl::LracFactor lf;
  const vl_factor* f;
};
struct vl_lracw {
  vl::LracPrec p;
};

namespace vl {

static thread_local std::string g_last_error;

struct VlException : std::runtime_error {
  int code;
  VlException(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

[[noreturn]] void fail(int code, const std::string& msg) { throw VlException(code, msg); }

void cuda_check(cudaError_t e, const char* what, const char* file, int line) {
  if (e != cudaSuccess) {
    std::string m = std::string("CUDA error ") + cudaGetErrorName(e) + " (" + cudaGetErrorString(e) + ") in " + what +
                    " at " + file + ":" + std::to_string(line);
    throw VlException(kECuda, m);
  }
}

// Caching device allocator: factor / workspace buffers are re-created for
// every theta of a fit, so blocks go back to a per-(device, size) free list
// instead of cudaFree (which would synchronise the device).  All library work
// is ordered on one stream, so stream-ordered reuse is safe.
namespace {
std::mutex g_pool_mu;
std::multimap<std::pair<int, size_t>, void*> g_pool;

void* pool_get(size_t bytes) {
  int dev = 0;
  cudaGetDevice(&dev);
  {
    std::lock_guard<std::mutex> lk(g_pool_mu);
    auto it = g_pool.find({dev, bytes});
    if (it != g_pool.end()) {
      void* p = it->second;
      g_pool.erase(it);
      return p;
    }
  }
  void* p = nullptr;
  cudaError_t e = cudaMalloc(&p, bytes);
  if (e != cudaSuccess) {
    cudaGetLastError();
    // release cached blocks of this device and retry once
    std::lock_guard<std::mutex> lk(g_pool_mu);
    for (auto it = g_pool.begin(); it != g_pool.end();) {
      if (it->first.first == dev) { cudaFree(it->second); it = g_pool.erase(it); }
      else ++it;
    }
    VL_CUDA(cudaMalloc(&p, bytes));
  }
  return p;
}

void pool_put(void* p, size_t bytes) {
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lk(g_pool_mu);
  g_pool.insert({{dev, bytes}, p});
}

size_t round_bytes(size_t b) {
  if (b <= 4096) return 4096;
  return (b + (1u << 20) - 1) & ~(size_t)((1u << 20) - 1);  // 1 MiB granularity
}
}  // namespace

void DevBuf::release() {
  if (p) pool_put(p, bytes);
  p = nullptr;
  bytes = 0;
}
void DevBuf::alloc(size_t nbytes) {
  if (nbytes <= bytes && p) return;
  release();
  size_t r = round_bytes(nbytes);
  p = pool_get(r);
  bytes = r;
}

template <class F>
static int guard(F&& f) {
  try {
    f();
    return kOk;
  } catch (const VlException& e) {
    g_last_error = e.what();
    return e.code;
  } catch (const std::bad_alloc&) {
    g_last_error = "host out of memory";
    return kECapacity;
  } catch (const std::exception& e) {
    g_last_error = e.what();
    return kEInternal;
  }
}

// Every handle-based entry point runs on its context's device and restores
// the caller's current device on return (contexts on several devices in one
// process stay independent: the caching pool files blocks by current device).
struct DeviceScope {
  int prev = -1;
  explicit DeviceScope(int d) {
    int cur = 0;
    VL_CUDA(cudaGetDevice(&cur));
    if (cur != d) {
      VL_CUDA(cudaSetDevice(d));
      prev = cur;
    }
  }
  ~DeviceScope() {
    if (prev >= 0) cudaSetDevice(prev);
  }
};

template <class F>
static int guard_dev(vl_ctx* h, F&& f) {
  if (h == nullptr) {
    g_last_error = "null context handle";
    return kEConfig;
  }
  const int device = h->c.device;
  return guard([&] {
    DeviceScope ds(device);
    f();
  });
}

template <class T>
static void upload(Ctx& C, DevBuf& dst, const std::vector<T>& src) {
  dst.alloc(sizeof(T) * std::max<size_t>(src.size(), 1));
  if (!src.empty())
    VL_CUDA(cudaMemcpyAsync(dst.p, src.data(), sizeof(T) * src.size(), cudaMemcpyHostToDevice, C.stream));
}

void pattern_upload(Ctx& C, Pattern& P, const double* xy, const int32_t* nbr) {
  std::vector<int32_t> ell, cnt, fwd, bwd, tptr, tidx, tmap;
  pattern_build_host(P, xy, nbr, ell, cnt, fwd, bwd, tptr, tidx, tmap);
  std::vector<double> xys((size_t)P.n * P.d);
  for (int64_t s = 0; s < P.n; ++s)
    for (int k = 0; k < P.d; ++k) xys[s * P.d + k] = xy[(int64_t)P.sperm[s] * P.d + k];
  upload(C, P.xy, xys);
  upload(C, P.nbr, ell);
  upload(C, P.cnt, cnt);
  upload(C, P.fidx, P.sperm);
  upload(C, P.fwd_order, fwd);
  upload(C, P.bwd_order, bwd);
  upload(C, P.tptr, tptr);
  upload(C, P.tidx, tidx);
  upload(C, P.tmap, tmap);
  P.fwd_len = (int64_t)fwd.size();
  P.bwd_len = (int64_t)bwd.size();
  upload(C, P.fwd_lptr, P.fwd_level_ptr);
  upload(C, P.bwd_lptr, P.bwd_level_ptr);
  // single-RHS work items: 32-row chunks, expanded to per-row (warp-per-row)
  // items on thin levels and for chunks holding a row with many dependencies
  // (measured at n = 1e6, profiles/r2k_heavy_sweep.jsonl: level rows 64 / 128 / 256 / 512 / 1024 ->
  // forward solve 0.344 / 0.338 / 0.327 / 0.323 / 0.328 ms; dependencies 32 / 64 / 128 ->
  // backward solve 0.553 / 0.357 / 0.473 ms)
  int heavy_rows = 512, heavy_deps = 64;
  if (const char* e = std::getenv("VL_HEAVY_LEVEL_ROWS")) heavy_rows = std::atoi(e);
  if (const char* e = std::getenv("VL_HEAVY_DEPS")) heavy_deps = std::atoi(e);
  bool slab_sort = false;
  if (const char* e = std::getenv("VL_SLAB_SORT")) slab_sort = std::atoi(e) != 0;
  // A chunk on a wide level whose rows all have <= heavy_deps dependencies is one light item.
  // Rows above that become warp-per-row items of their own and are masked out of the chunk
  // (mask[p] = 1: the light item skips position p), so their chunk-mates stay thread-per-row
  // (VL_HEAVY_SPLIT=0: the whole chunk turns into warp-per-row items, as before).
  bool heavy_split = true;
  if (const char* e = std::getenv("VL_HEAVY_SPLIT")) heavy_split = std::atoi(e) != 0;
  auto items = [&](const std::vector<int32_t>& order, const std::vector<int32_t>& lptr, bool fwd_dir,
                   std::vector<char>& mask) {
    std::vector<uint32_t> it;
    mask.assign(order.size(), 0);
    for (size_t L = 0; L + 1 < lptr.size(); ++L) {
      const int32_t q0 = lptr[L], q1 = lptr[L + 1];
      const bool thin = (q1 - q0) <= heavy_rows;
      for (int32_t c = q0; c < q1; c += 32) {
        int nheavy = 0, nrows = 0;
        for (int32_t p = c; p < c + 32; ++p) {
          const int32_t s = order[p];
          if (s < 0) continue;
          ++nrows;
          const int deg = fwd_dir ? cnt[s] : (tptr[s + 1] - tptr[s]);
          if (deg > heavy_deps) ++nheavy;
        }
        if (!thin && nheavy == 0) {
          it.push_back((uint32_t)c);
        } else if (thin || !heavy_split) {
          for (int32_t p = c; p < c + 32; ++p)
            if (order[p] >= 0) it.push_back((uint32_t)p | 0x80000000u);
        } else {
          for (int32_t p = c; p < c + 32; ++p) {
            const int32_t s = order[p];
            if (s < 0) continue;
            const int deg = fwd_dir ? cnt[s] : (tptr[s + 1] - tptr[s]);
            if (deg > heavy_deps) {
              it.push_back((uint32_t)p | 0x80000000u);
              mask[p] = 1;
            }
          }
          if (nheavy < nrows) it.push_back((uint32_t)c);
        }
      }
    }
    return it;
  };
  auto masked = [&](const std::vector<int32_t>& order, const std::vector<char>& mask) {
    std::vector<int32_t> o(order);
    for (size_t p = 0; p < o.size(); ++p)
      if (mask[p]) o[p] = -1;
    return o;
  };
  // Heavy items carry their row, dependency base and count in the item
  // descriptor (items = row | bit, off = ELL / CSR base, w = count), so the
  // solve issues their coalesced dependency loads without the order -> row
  // pointer chain.
  auto slabs = [&](const std::vector<int32_t>& order, std::vector<uint32_t>& its, bool fwd_dir,
                   Pattern::Slabs& S, const std::vector<char>& mask) {
    std::vector<uint32_t> off(std::max<size_t>(its.size(), 1), 0), w(std::max<size_t>(its.size(), 1), 0);
    int64_t tot = 0;
    auto deg = [&](int32_t s) { return fwd_dir ? cnt[s] : (tptr[s + 1] - tptr[s]); };
    for (size_t k = 0; k < its.size(); ++k) {
      if (its[k] & 0x80000000u) {
        const int32_t s = order[its[k] & 0x7fffffffu];
        const int64_t base = fwd_dir ? (int64_t)s * P.m : (int64_t)tptr[s];
        if (base > (int64_t)UINT32_MAX) fail(kECapacity, "dependency base exceeds 32 bits");
        off[k] = (uint32_t)base;
        w[k] = (uint32_t)deg(s);
        continue;
      }
      const int32_t c = (int32_t)its[k];
      int wk = 0;
      for (int32_t p = c; p < c + 32; ++p)
        if (order[p] >= 0 && !mask[p]) wk = std::max(wk, deg(order[p]));
      off[k] = (uint32_t)tot;
      w[k] = (uint32_t)wk;
      tot += wk;
    }
    if (tot * 32 > (int64_t)INT32_MAX * 2) fail(kECapacity, "single-RHS slab too large");
    std::vector<int32_t> idx((size_t)tot * 32, -1), map((size_t)tot * 32, -1);
    for (size_t k = 0; k < its.size(); ++k) {
      if (its[k] & 0x80000000u) continue;
      const int32_t c = (int32_t)its[k];
      for (int l = 0; l < 32; ++l) {
        const int32_t s = order[c + l];
        if (s < 0 || mask[c + l]) continue;
        const int d = deg(s);
        std::vector<std::pair<int32_t, int32_t>> ent(d);  // (dependency row, ELL slot of its value)
        for (int e = 0; e < d; ++e) {
          if (fwd_dir) {
            ent[e] = {ell[(size_t)s * P.m + e], (int32_t)((int64_t)s * P.m + e)};
          } else {
            const int32_t pos = tptr[s] + e;
            ent[e] = {tidx[pos], tmap[pos]};
          }
        }
        // VL_SLAB_SORT=1: a row's entries by dependency storage row, so entry e of the 32
        // spatially adjacent rows of an item falls into nearby lines of x
        if (slab_sort) std::sort(ent.begin(), ent.end());
        for (int e = 0; e < d; ++e) {
          const size_t q = ((size_t)off[k] + e) * 32 + l;
          idx[q] = ent[e].first;
          map[q] = ent[e].second;
        }
      }
    }
    S.nent = tot * 32;
    for (auto& it : its)
      if (it & 0x80000000u) it = (uint32_t)order[it & 0x7fffffffu] | 0x80000000u;
    upload(C, S.off, off);
    upload(C, S.w, w);
    upload(C, S.idx, idx);
    upload(C, S.map, map);
  };
  std::vector<char> fmask, bmask, bnmask;
  auto fi = items(fwd, P.fwd_level_ptr, true, fmask);
  auto bi = items(bwd, P.bwd_level_ptr, false, bmask);
  P.fwd_nitems = (int64_t)fi.size();
  P.bwd_nitems = (int64_t)bi.size();
  // dense head block + backward schedule without it
  upload(C, P.head_rows, P.head_rows_h);
  upload(C, P.head_pos, P.head_pos_h);
  upload(C, P.head_nbr, P.head_nbr_h);
  upload(C, P.bwdnh_order, P.bwdnh_order_h);
  upload(C, P.bwdnh_lptr, P.bwdnh_level_ptr);
  P.bwdnh_len = (int64_t)P.bwdnh_order_h.size();
  P.fwd_items_head_end = 0;
  if (P.head_L > 0)
    for (uint32_t it : fi)
      if ((int64_t)(it & 0x7fffffffu) < P.fwd_level_ptr[P.head_L]) ++P.fwd_items_head_end;
  auto bni = items(P.bwdnh_order_h, P.bwdnh_level_ptr, false, bnmask);
  P.bwdnh_nitems = (int64_t)bni.size();
  slabs(fwd, fi, true, P.fwd_sl, fmask);
  slabs(bwd, bi, false, P.bwd_sl, bmask);
  slabs(P.bwdnh_order_h, bni, false, P.bwdnh_sl, bnmask);
  // the light items' view of the orders: positions of rows that run as their own items are -1
  upload(C, P.fwd_order1, masked(fwd, fmask));
  upload(C, P.bwd_order1, masked(bwd, bmask));
  upload(C, P.bwdnh_order1, masked(P.bwdnh_order_h, bnmask));
  upload(C, P.nbr_s, P.nbr_s_h);
  upload(C, P.map_s, P.map_s_h);
  P.has_solve_order = !P.map_s_h.empty();
  upload(C, P.fwd_torder, P.fwd_torder_h);
  upload(C, P.bwd_torder, P.bwd_torder_h);
  P.fwd_tlen = (int64_t)P.fwd_torder_h.size();
  P.bwd_tlen = (int64_t)P.bwd_torder_h.size();
  upload(C, P.fwd_items, fi);
  upload(C, P.bwd_items, bi);
  upload(C, P.bwdnh_items, bni);
  VL_CUDA(cudaStreamSynchronize(C.stream));
  std::vector<int32_t>().swap(P.nbr_s_h);
  std::vector<int32_t>().swap(P.map_s_h);
}

}  // namespace vl

using namespace vl;

extern "C" {

int vl_version(void) { return 100; }
const char* vl_last_error(void) { return g_last_error.c_str(); }

int vl_ctx_create(int device, void* stream, vl_ctx** out) {
  return guard([&] {
    if (!out) fail(kEConfig, "null output handle");
    int ndev = 0;
    VL_CUDA(cudaGetDeviceCount(&ndev));
    if (device < 0 || device >= ndev) fail(kEConfig, "invalid CUDA device ordinal " + std::to_string(device));
    VL_CUDA(cudaSetDevice(device));
    cudaDeviceProp prop;
    VL_CUDA(cudaGetDeviceProperties(&prop, device));
    if (prop.major != 10) fail(kECapability, std::string("vlgpx is built for sm_100a (B200); found ") + prop.name);
    auto* h = new vl_ctx();
    Ctx& C = h->c;
    C.device = device;
    C.num_sms = prop.multiProcessorCount;
    if (const char* e = std::getenv("VL_TRSV_BPS")) C.trsv_blocks_per_sm = std::max(1, std::atoi(e));
    if (const char* e = std::getenv("VL_SPIN_MAX_NS")) C.spin_max_ns = std::max(0, std::atoi(e));
    if (const char* e = std::getenv("VL_SPIN_MAX_NS1")) C.spin_max_ns1 = std::max(0, std::atoi(e));
    if (const char* e = std::getenv("VL_THIN_PASSES")) C.thin_passes = std::max(0, std::atoi(e));
    if (const char* e = std::getenv("VL_MIN_THICK")) C.min_thick_levels = std::max(0, std::atoi(e));
    if (const char* e = std::getenv("VL_USE_HEAD")) C.use_head = std::atoi(e) != 0;
    if (const char* e = std::getenv("VL_USE_SLABS")) C.use_slabs = std::atoi(e) != 0;
    if (const char* e = std::getenv("VL_USE_TILES")) C.use_tiles = std::atoi(e) != 0;
    if (const char* e = std::getenv("VL_USE_LOCAL")) C.use_local = std::atoi(e) != 0;
    if (const char* e = std::getenv("VL_PMODE1")) C.pmode1 = std::max(0, std::min(3, std::atoi(e)));
    if (const char* e = std::getenv("VL_PMODET")) C.pmodeT = std::max(0, std::min(1, std::atoi(e)));
    try {
      // NULL selects the legacy default stream (same as torch's default stream)
      C.stream = (cudaStream_t)stream;
      C.own_stream = false;
      C.red_partial.alloc(16u << 20);
      C.red_counter.alloc(64 * sizeof(unsigned));
      VL_CUDA(cudaMemsetAsync(C.red_counter.p, 0, 64 * sizeof(unsigned), C.stream));
      C.dev_scalars.alloc(1 << 16);
      VL_CUDA(cudaMallocHost(&C.host_scalars, 4096));
      VL_CUDA(cudaStreamSynchronize(C.stream));
    } catch (...) {
      delete h;
      throw;
    }
    *out = h;
  });
}

int vl_ctx_destroy(vl_ctx* h) {
  return guard_dev(h, [&] {
    if (!h) return;
    cudaSetDevice(h->c.device);
    if (h->c.stream) cudaStreamSynchronize(h->c.stream);
    if (h->c.host_scalars) cudaFreeHost(h->c.host_scalars);
    if (h->c.own_stream) cudaStreamDestroy(h->c.stream);
    if (h->c.side) cudaStreamDestroy(h->c.side);
    if (h->c.ev_fork) cudaEventDestroy(h->c.ev_fork);
    if (h->c.ev_join) cudaEventDestroy(h->c.ev_join);
    delete h;
  });
}

int vl_ctx_sync(vl_ctx* h) {
  return guard_dev(h, [&] { VL_CUDA(cudaStreamSynchronize(h->c.stream)); });
}

int vl_ctx_info(vl_ctx* h, int64_t* info) {
  return guard_dev(h, [&] {
    info[0] = h->c.device;
    info[1] = h->c.num_sms;
  });
}

int vl_knn_previous(const double* xy, int64_t n, int d, int m, int32_t* out, int n_threads) {
  return guard([&] {
    if (n < 1 || d < 1 || m < 0) fail(kEConfig, "invalid knn sizes");
    knn_previous(xy, n, d, m, out, n_threads);
  });
}

int vl_knn_previous_dev(vl_ctx* h, const double* xy, int64_t n, int d, int m, int32_t* out) {
  return guard_dev(h, [&] {
    if (!xy || !out) fail(kEConfig, "null pointer");
    knn_previous_dev(h->c, xy, n, d, m, out);
  });
}

int vl_knn_query(vl_ctx* h, const double* train, int64_t n, const double* q, int64_t nq, int d, int m, int32_t* out,
                 double* dmin) {
  return guard_dev(h, [&] {
    if (!train || (nq > 0 && (!q || !out || !dmin))) fail(kEConfig, "null pointer");
    knn_query_dev(h->c, train, n, q, nq, d, m, out, dmin);
  });
}

int vl_pattern_create(vl_ctx* h, int64_t n, int d, int m, const double* xy, const int32_t* nbr, int order_kind,
                      vl_pattern** out) {
  return guard_dev(h, [&] {
    if (!h || !out) fail(kEConfig, "null handle");
    if (n < 1 || d < 1 || m < 0) fail(kEConfig, "invalid pattern sizes");
    if (order_kind < 0 || order_kind > 2) fail(kEConfig, "unknown storage order");
    VL_CUDA(cudaSetDevice(h->c.device));
    auto* p = new vl_pattern();
    p->ctx = h;
    p->p.n = n;
    p->p.d = d;
    p->p.m = m;
    p->p.order_kind = order_kind;
    if (const char* e = std::getenv("VL_HEAD_MAX")) p->p.head_max = std::max(0, std::atoi(e));
    if (const char* e = std::getenv("VL_CHILD_LATE")) p->p.child_late = std::max(0, std::atoi(e));
    if (const char* e = std::getenv("VL_TILE_K")) p->p.tile_K = std::max(0, std::atoi(e));  // 0: level order
    if (const char* e = std::getenv("VL_TILE_S")) p->p.tile_S = std::max(1, std::atoi(e));
    if (const char* e = std::getenv("VL_TILE_MIN_ROWS")) p->p.tile_min_rows = std::max(1, std::atoi(e));
    if (const char* e = std::getenv("VL_TILE_TAIL")) p->p.tile_tail = std::atoi(e) != 0;
    if (const char* e = std::getenv("VL_TILE_MIN_MB")) p->p.tile_min_bytes = (size_t)std::max(0, std::atoi(e)) << 20;
    if (const char* e = std::getenv("VL_TILE_MIN_N")) p->p.tile_min_n = std::max(0, std::atoi(e));
    try {
      std::vector<int32_t> empty;
      const int32_t* nb = nbr;
      if (m == 0) nb = empty.data();
      pattern_upload(h->c, p->p, xy, nb);
    } catch (...) {
      delete p;
      throw;
    }
    *out = p;
  });
}

int vl_pattern_destroy(vl_pattern* p) {
  return guard([&] { delete p; });
}

int vl_pattern_perm(const vl_pattern* p, int32_t* out) {
  return guard([&] { std::memcpy(out, p->p.sperm.data(), sizeof(int32_t) * p->p.n); });
}

int vl_pattern_info(const vl_pattern* p, int64_t* info) {
  return guard([&] {
    const Pattern& P = p->p;
    info[0] = P.n;
    info[1] = P.d;
    info[2] = P.m;
    info[3] = P.nnz_off;
    info[4] = P.nlev_fwd;
    info[5] = P.nlev_bwd;
    info[6] = P.max_children;
    info[7] = P.order_kind;
    info[8] = P.head_L;
    info[9] = P.head_H;
  });
}

int vl_pattern_solve_order(const vl_pattern* p, int transpose, int64_t* len, int32_t* order_host) {
  return guard([&] {
    if (!p || !len) fail(kEConfig, "null handle");
    const std::vector<int32_t>& o = transpose ? p->p.bwd_torder_h : p->p.fwd_torder_h;
    *len = (int64_t)o.size();
    if (order_host != nullptr && !o.empty()) std::memcpy(order_host, o.data(), sizeof(int32_t) * o.size());
  });
}

int vl_factor_build(vl_ctx* h, const vl_pattern* p, double sigma2, double rho, double nu, int want_grad,
                    vl_factor** out) {
  return guard_dev(h, [&] {
    if (!h || !p || !out) fail(kEConfig, "null handle");
    VL_CUDA(cudaSetDevice(h->c.device));
    auto* f = new vl_factor();
    try {
      factor_build(h->c, p->p, f->f, sigma2, rho, nu, want_grad != 0);
    } catch (...) {
      delete f;
      throw;
    }
    *out = f;
  });
}

int vl_factor_destroy(vl_factor* f) {
  return guard([&] { delete f; });
}

int vl_factor_get(vl_ctx* h, const vl_factor* f, int which, double* out) {
  return guard_dev(h, [&] {
    const Factor& F = f->f;
    const Pattern& P = *F.pat;
    const DevBuf* src = nullptr;
    size_t cnt = P.n;
    switch (which) {
      case 0: src = &F.D; break;
      case 1: src = &F.dD_sig; break;
      case 2: src = &F.dD_rho; break;
      case 3: src = &F.val; cnt = (size_t)P.n * P.m; break;
      case 4: src = &F.dval; cnt = (size_t)P.n * P.m; break;
      default: fail(kEConfig, "unknown factor field");
    }
    if ((which == 1 || which == 2 || which == 4) && !F.has_grad) fail(kEConfig, "factor was built without gradient");
    if (cnt == 0) return;
    VL_CUDA(cudaMemcpyAsync(out, src->p, sizeof(double) * cnt, cudaMemcpyDeviceToHost, h->c.stream));
    VL_CUDA(cudaStreamSynchronize(h->c.stream));
  });
}

int vl_factor_set(vl_ctx* h, vl_factor* f, int which, const double* in) {
  return guard_dev(h, [&] {
    Factor& F = f->f;
    const Pattern& P = *F.pat;
    DevBuf* dst = nullptr;
    size_t cnt = P.n;
    switch (which) {
      case 0: dst = &F.D; break;
      case 1: dst = &F.dD_sig; break;
      case 2: dst = &F.dD_rho; break;
      case 3: dst = &F.val; cnt = (size_t)P.n * P.m; break;
      case 4: dst = &F.dval; cnt = (size_t)P.n * P.m; break;
      default: fail(kEConfig, "unknown factor field");
    }
    if ((which == 1 || which == 2 || which == 4) && !F.has_grad) fail(kEConfig, "factor was built without gradient");
    if (cnt == 0) return;
    VL_CUDA(cudaMemcpyAsync(dst->p, in, sizeof(double) * cnt, cudaMemcpyHostToDevice, h->c.stream));
    if (which == 3) factor_refresh_transpose(h->c, F);
    VL_CUDA(cudaStreamSynchronize(h->c.stream));
  });
}

int vl_prof_enable(vl_ctx* h, int on) {
  return guard_dev(h, [&] {
    prof_collect(h->c);
    h->c.prof.on = on != 0;
  });
}

int vl_prof_only(vl_ctx* h, const char* tag) {
  return guard_dev(h, [&] {
    prof_collect(h->c);
    h->c.prof.only = tag ? tag : "";
  });
}

int vl_prof_reset(vl_ctx* h) {
  return guard_dev(h, [&] {
    prof_collect(h->c);
    h->c.prof.agg.clear();
    h->c.prof.launches = 0;
  });
}

int vl_prof_report(vl_ctx* h, char* buf, int len, int64_t* launches) {
  return guard_dev(h, [&] {
    prof_collect(h->c);
    std::string s;
    for (auto& kv : h->c.prof.agg) {
      char line[256];
      snprintf(line, sizeof(line), "%s\t%ld\t%.6f\t%.1f\n", kv.first.c_str(), kv.second.count, kv.second.ms,
               kv.second.bytes);
      s += line;
    }
    if (buf && len > 0) {
      std::strncpy(buf, s.c_str(), (size_t)len - 1);
      buf[len - 1] = 0;
    }
    if (launches) *launches = h->c.prof.launches;
  });
}

// debug hook (not in the public header): record per-row completion times of
// subsequent triangular solves into a device buffer of n int64 (NULL disables)
int vl_debug_set_tstamp(vl_ctx* h, void* dev_buf) {
  return guard_dev(h, [&] { h->c.debug_tstamp = (long long*)dev_buf; });
}

// ---- Laplace path -----------------------------------------------------------

int vl_find_mode(vl_ctx* h, const vl_factor* f, const vl_lik* lik, const vl_newton_cfg* cfg, const double* y,
                 const double* Fv, double* b, double* W, double* d1, double* d3, double* out, int32_t* cg_iters,
                 int cg_iters_cap) {
  return guard_dev(h, [&] {
    if (!h || !f || !lik || !cfg || !out) fail(kEConfig, "null argument");
    LikSpec L{lik->family, lik->shape};
    NewtonCfg nc{cfg->mode_cg_tol, cfg->cg_max_iter, cfg->newton_max_iter, cfg->newton_grad_tol, cfg->newton_obj_tol,
                 cfg->precond};
    NewtonOut no;
    auto fill = [&] {
      out[0] = no.logp;
      out[1] = no.quad;
      out[2] = no.objective;
      out[3] = no.grad_norm;
      out[4] = no.iters;
      out[5] = no.converged;
      out[6] = (double)no.cg_iters.size();
      if (cg_iters)
        for (int i = 0; i < (int)no.cg_iters.size() && i < cg_iters_cap; ++i) cg_iters[i] = no.cg_iters[i];
    };
    try {
      newton_mode(h->c, f->f, L, nc, y, Fv, b, W, d1, d3, &no);
    } catch (...) {
      fill();
      throw;
    }
    fill();
  });
}

// ---- LRAC -----------------------------------------------------------------------

int vl_lrac_create(vl_ctx* h, const vl_factor* f, int k, double tol, vl_lrac** out, int32_t* piv_host, int* keff) {
  return guard_dev(h, [&] {
    auto* l = new vl_lrac();
    l->f = f;
    try {
      lrac_pchol(h->c, f->f, l->lf, k, tol);
    } catch (...) {
      delete l;
      throw;
    }
    if (keff) *keff = l->lf.keff;
    if (piv_host)
      for (int q = 0; q < l->lf.keff; ++q) piv_host[q] = l->lf.piv_f[q];
    *out = l;
  });
}

int vl_lrac_destroy(vl_lrac* l) {
  return guard([&] { delete l; });
}

int vl_lrac_get_L(vl_ctx* h, const vl_lrac* l, double* host) {
  return guard_dev(h, [&] {
    const size_t cnt = (size_t)l->f->f.pat->n * l->lf.k;
    VL_CUDA(cudaMemcpyAsync(host, l->lf.L.p, sizeof(double) * cnt, cudaMemcpyDeviceToHost, h->c.stream));
    VL_CUDA(cudaStreamSynchronize(h->c.stream));
  });
}

int vl_lrac_prepare(vl_ctx* h, const vl_lrac* l, const double* W, vl_lracw** out, double* out2) {
  return guard_dev(h, [&] {
    const int64_t n = l->f->f.pat->n;
    if (count_nonpos(h->c, n, W) > 0)
      fail(kECapability, "lrac preconditions SigmaTilde + W^{-1} and needs W > 0 everywhere (eq7 split; log W "
                         "undefined); switch to an eq6 preconditioner such as vadu");
    auto* w = new vl_lracw();
    try {
      lrac_prepare(h->c, l->f->f, l->lf, W, w->p);
      w->p.sumlogW = lrac_sumlogW(h->c, n, W);
    } catch (...) {
      delete w;
      throw;
    }
    if (out2) {
      out2[0] = w->p.logdetM;
      out2[1] = w->p.sumlogW;
    }
    *out = w;
  });
}

int vl_lracw_destroy(vl_lracw* w) {
  return guard([&] { delete w; });
}

int vl_lrac_apply_inv(vl_ctx* h, const vl_lracw* w, int64_t t, const double* r, double* z) {
  return guard_dev(h, [&] { lrac_apply_inv(h->c, w->p, (int)t, r, z); });
}

int vl_lrac_pcg(vl_ctx* h, const vl_lracw* w, int64_t t, const double* bm, double* u, double tol, int max_iter,
                int capture, int32_t* iters, int32_t* conv, double* res, double* alpha, double* beta, int hist_cap) {
  return guard_dev(h, [&] {
    if (t < 1 || t > 128) fail(kECapacity, "right-hand sides per call must be in [1, 128]");
    PcgResult pr;
    pcg_lrac(h->c, w->p, (int)t, bm, u, tol, max_iter, capture != 0, &pr);
    for (int c = 0; c < t; ++c) {
      if (iters) iters[c] = pr.iters[c];
      if (conv) conv[c] = pr.converged[c];
      if (res) res[c] = pr.res[c];
    }
    if (capture && alpha && beta)
      for (int q = 0; q < std::min(pr.max_iters, hist_cap); ++q)
        for (int c = 0; c < t; ++c) {
          alpha[(size_t)q * t + c] = pr.alpha[(size_t)q * t + c];
          beta[(size_t)q * t + c] = pr.beta[(size_t)q * t + c];
        }
  });
}

int vl_lrac_solve_system(vl_ctx* h, const vl_lracw* w, int64_t t, const double* rhs, double* u, double tol,
                         int max_iter, int32_t* iters) {
  return guard_dev(h, [&] {
    PcgResult pr;
    lrac_solve_system(h->c, w->p, (int)t, rhs, u, tol, max_iter, &pr);
    if (iters)
      for (int c = 0; c < t; ++c) iters[c] = pr.iters[c];
  });
}

int vl_apply_sigma_tilde(vl_ctx* h, const vl_factor* f, int64_t t, const double* x, double* y) {
  return guard_dev(h, [&] {
    DevBuf scr;
    scr.alloc(sizeof(double) * (size_t)f->f.pat->n * t);
    apply_sigma_tilde(h->c, f->f, (int)t, x, y, scr.as<double>());
  });
}

int vl_lrac_probes(vl_ctx* h, const vl_lracw* w, int64_t t, const double* Gn, const double* Gk, double* Z, double* V,
                   double* w_host) {
  return guard_dev(h, [&] { lrac_probes(h->c, w->p, (int)t, Gn, Gk, Z, V, w_host); });
}

int vl_lrac_grad(vl_ctx* h, const vl_lracw* w, int64_t t, const double* U, const double* V, const double* d3,
                 const double* md3x, double* s, double* hcols, double* rcols, double* dPt, double* xicols,
                 double* xis, int plain) {
  return guard_dev(h, [&] { lrac_grad(h->c, w->p, (int)t, U, V, d3, md3x, s, hcols, rcols, dPt, xicols, xis, plain); });
}

int vl_probes_rademacher(vl_ctx* h, const vl_pattern* p, int64_t t, int64_t t_glob, int64_t c0, uint64_t seed,
                         double* Z) {
  return guard_dev(h, [&] {
    if (t < 1 || c0 < 0 || c0 + t > t_glob) fail(kEConfig, "invalid probe column range");
    rademacher_probes(h->c, p->p, (int)t, (int)t_glob, (int)c0, seed, Z);
  });
}

int vl_probes_given(vl_ctx* h, const vl_factor* f, const double* dinv, int pkind, int64_t t, const double* Z,
                    double* V, double* w_host) {
  return guard_dev(h, [&] { probes_given(h->c, f->f, dinv, pkind, (int)t, (int)t, Z, V, w_host); });
}

int vl_dgemm(vl_ctx* h, int transa, int transb, int64_t m, int64_t n, int64_t k, double alpha, const double* A,
             int64_t lda, const double* B, int64_t ldb, double beta, double* Cm, int64_t ldc, const double* kw,
             int lower) {
  return guard_dev(h, [&] {
    Gemm g;
    g.ta = transa != 0; g.tb = transb != 0;
    g.m = (int)m; g.n = (int)n; g.k = (int)k;
    g.alpha = alpha; g.beta = beta;
    g.A = A; g.lda = (int)lda; g.B = B; g.ldb = (int)ldb; g.C = Cm; g.ldc = (int)ldc;
    g.kw = kw; g.lower = lower != 0;
    dgemm(h->c, g);
    VL_CUDA(cudaStreamSynchronize(h->c.stream));
  });
}

int vl_dtrtri_lower(vl_ctx* h, int64_t k, const double* L, int64_t ldl, double* Li, int64_t ldi) {
  return guard_dev(h, [&] {
    dtrtri_lower(h->c, (int)k, L, (int)ldl, Li, (int)ldi);
    VL_CUDA(cudaStreamSynchronize(h->c.stream));
  });
}

int vl_lrac_grad_split(vl_ctx* h, const vl_lracw* w, int mode, int64_t t, int64_t t_glob, const double* U,
                       const double* V, const double* d3, const double* md3x, double* rowA, double* rowB, double* s,
                       double* hcols, double* rcols, double* dPt, double* xicols, double* xis, int plain) {
  return guard_dev(h, [&] {
    lrac_grad_split(h->c, w->p, mode, (int)t, (int)t_glob, U, V, d3, md3x, rowA, rowB, s, hcols, rcols, dPt, xicols,
                    xis, plain);
  });
}

int vl_lowrank_create(vl_ctx* h, const vl_factor* f, int kind, int k, double tol, vl_lrac** out, int32_t* piv_host,
                      int* keff) {
  return guard_dev(h, [&] {
    auto* l = new vl_lrac();
    l->f = f;
    try {
      if (kind == 1) pchol_precision(h->c, f->f, l->lf, k, tol);
      else if (kind == 2) rowsel_factor(h->c, f->f, l->lf, k);
      else fail(kEConfig, "kind must be 1 (pchol-precision) or 2 (rowsel)");
    } catch (...) {
      delete l;
      throw;
    }
    if (keff) *keff = l->lf.keff;
    if (piv_host)
      for (int q = 0; q < l->lf.keff; ++q) piv_host[q] = l->lf.piv_f[q];
    *out = l;
  });
}

int vl_lowrank_einv(vl_ctx* h, int64_t n, int kind, const double* W, const double* diag_st, double* einv) {
  return guard_dev(h, [&] { lowrank_einv(h->c, n, kind, W, diag_st, einv); });
}

int vl_lowrank_prepare(vl_ctx* h, const vl_factor* f, const vl_lrac* l, const double* Wop, const double* einv,
                       int eq6, vl_lracw** out, double* out2) {
  return guard_dev(h, [&] {
    auto* w = new vl_lracw();
    try {
      lowrank_prepare(h->c, f->f, l ? &l->lf : nullptr, Wop, einv, eq6, w->p);
    } catch (...) {
      delete w;
      throw;
    }
    if (out2) {
      out2[0] = w->p.logdetM;
      out2[1] = w->p.sumlogW;
    }
    *out = w;
  });
}

int vl_diag_sigma_tilde(vl_ctx* h, const vl_factor* f, double* out) {
  return guard_dev(h, [&] { diag_sigma_tilde(h->c, f->f, out); });
}

int vl_find_mode_lowrank(vl_ctx* h, const vl_factor* f, const vl_lrac* l, int wb_kind, const double* diag_st,
                         const vl_lik* lik, const vl_newton_cfg* cfg, const double* y, const double* Fv, double* b,
                         double* W, double* d1, double* d3, double* out, int32_t* cg_iters, int cg_iters_cap) {
  return guard_dev(h, [&] {
    if (wb_kind != 1 && wb_kind != 2) fail(kEConfig, "wb_kind must be 1 (eq6 low rank) or 2 (l2)");
    if (wb_kind == 1 && !l) fail(kEConfig, "low-rank factor required");
    LikSpec L{lik->family, lik->shape};
    NewtonCfg nc{cfg->mode_cg_tol, cfg->cg_max_iter, cfg->newton_max_iter, cfg->newton_grad_tol, cfg->newton_obj_tol,
                 0, wb_kind, diag_st};
    NewtonOut no;
    auto fill = [&] {
      out[0] = no.logp;
      out[1] = no.quad;
      out[2] = no.objective;
      out[3] = no.grad_norm;
      out[4] = no.iters;
      out[5] = no.converged;
      out[6] = (double)no.cg_iters.size();
      if (cg_iters)
        for (int i = 0; i < (int)no.cg_iters.size() && i < cg_iters_cap; ++i) cg_iters[i] = no.cg_iters[i];
    };
    try {
      newton_mode(h->c, f->f, L, nc, y, Fv, b, W, d1, d3, &no, l ? &l->lf : nullptr);
    } catch (...) {
      fill();
      throw;
    }
    fill();
  });
}

int vl_find_mode_lrac(vl_ctx* h, const vl_factor* f, const vl_lrac* l, const vl_lik* lik, const vl_newton_cfg* cfg,
                      const double* y, const double* Fv, double* b, double* W, double* d1, double* d3, double* out,
                      int32_t* cg_iters, int cg_iters_cap) {
  return guard_dev(h, [&] {
    LikSpec L{lik->family, lik->shape};
    NewtonCfg nc{cfg->mode_cg_tol, cfg->cg_max_iter, cfg->newton_max_iter, cfg->newton_grad_tol, cfg->newton_obj_tol,
                 cfg->precond};
    NewtonOut no;
    auto fill = [&] {
      out[0] = no.logp;
      out[1] = no.quad;
      out[2] = no.objective;
      out[3] = no.grad_norm;
      out[4] = no.iters;
      out[5] = no.converged;
      out[6] = (double)no.cg_iters.size();
      if (cg_iters)
        for (int i = 0; i < (int)no.cg_iters.size() && i < cg_iters_cap; ++i) cg_iters[i] = no.cg_iters[i];
    };
    try {
      newton_mode(h->c, f->f, L, nc, y, Fv, b, W, d1, d3, &no, &l->lf);
    } catch (...) {
      fill();
      throw;
    }
    fill();
  });
}

int vl_probes_vadu(vl_ctx* h, const vl_factor* f, const double* W, int64_t t, const double* G, double* Z, double* V,
                   double* w_host) {
  return guard_dev(h, [&] {
    if (t < 1 || t > 128) fail(kECapacity, "probe count per call must be in [1, 128]");
    probes_vadu(h->c, f->f, W, (int)t, (int)t, G, Z, V, w_host);
  });
}

int vl_pcg_vadu(vl_ctx* h, const vl_factor* f, const double* W, int64_t t, const double* bm, double* u, double tol,
                int max_iter, int capture, int32_t* iters, int32_t* conv, double* res, double* alpha, double* beta,
                int hist_cap) {
  return guard_dev(h, [&] {
    if (t < 1 || t > 128) fail(kECapacity, "right-hand sides per call must be in [1, 128]");
    const Factor& F = f->f;
    const int64_t n = F.pat->n;
    DevBuf Dinv, dinv;
    Dinv.alloc(sizeof(double) * n);
    dinv.alloc(sizeof(double) * n);
    vadu_diags(h->c, F, W, Dinv.as<double>(), dinv.as<double>());
    SysVadu S{&F, W, Dinv.as<double>(), dinv.as<double>()};
    PcgResult pr;
    pcg_vadu(h->c, S, (int)t, (int)t, bm, u, tol, max_iter, capture != 0, &pr);
    for (int c = 0; c < t; ++c) {
      if (iters) iters[c] = pr.iters[c];
      if (conv) conv[c] = pr.converged[c];
      if (res) res[c] = pr.res[c];
    }
    if (capture && alpha && beta) {
      for (int l = 0; l < std::min(pr.max_iters, hist_cap); ++l)
        for (int c = 0; c < t; ++c) {
          alpha[(size_t)l * t + c] = pr.alpha[(size_t)l * t + c];
          beta[(size_t)l * t + c] = pr.beta[(size_t)l * t + c];
        }
    }
  });
}

int vl_factor_sums(vl_ctx* h, const vl_factor* f, const double* W, double* out6) {
  return guard_dev(h, [&] { factor_sums(h->c, f->f, W, out6); });
}

int vl_grad_probe_pass(vl_ctx* h, const vl_factor* f, const double* W, const double* d3, const double* U,
                       const double* V, int64_t t, double* s_out, double* cols4, const double* md3x, double* xicols2,
                       int plain) {
  return guard_dev(h, [&] {
    if (t < 1 || t > 128) fail(kECapacity, "probe count per call must be in [1, 128]");
    grad_probe_pass(h->c, f->f, W, d3, U, V, (int)t, (int)t, s_out, cols4, md3x, xicols2, plain);
  });
}

int vl_precond_dinv(vl_ctx* h, const vl_factor* f, int variant, const double* W, double* dinv) {
  return guard_dev(h, [&] { precond_dinv(h->c, f->f, variant, W, dinv); });
}

int vl_pcg_eq6(vl_ctx* h, const vl_factor* f, const double* W, const double* dinv, int pkind, int64_t t,
               const double* bm, double* u, double tol, int max_iter, int capture, int32_t* iters, int32_t* conv,
               double* res, double* alpha, double* beta, int hist_cap) {
  return guard_dev(h, [&] {
    if (t < 1 || t > 128) fail(kECapacity, "right-hand sides per call must be in [1, 128]");
    if (pkind != 0 && pkind != 1) fail(kEConfig, "pkind must be 0 (sandwich) or 1 (diagonal)");
    const Factor& F = f->f;
    const int64_t n = F.pat->n;
    DevBuf Dinv, tmp;
    Dinv.alloc(sizeof(double) * n);
    tmp.alloc(sizeof(double) * n);
    vadu_diags(h->c, F, W, Dinv.as<double>(), tmp.as<double>());
    SysVadu S{&F, W, Dinv.as<double>(), dinv, pkind};
    PcgResult pr;
    pcg_vadu(h->c, S, (int)t, (int)t, bm, u, tol, max_iter, capture != 0, &pr);
    for (int c = 0; c < t; ++c) {
      if (iters) iters[c] = pr.iters[c];
      if (conv) conv[c] = pr.converged[c];
      if (res) res[c] = pr.res[c];
    }
    if (capture && alpha && beta) {
      for (int l = 0; l < std::min(pr.max_iters, hist_cap); ++l)
        for (int c = 0; c < t; ++c) {
          alpha[(size_t)l * t + c] = pr.alpha[(size_t)l * t + c];
          beta[(size_t)l * t + c] = pr.beta[(size_t)l * t + c];
        }
    }
  });
}

int vl_probes_eq6(vl_ctx* h, const vl_factor* f, const double* dinv, int pkind, int64_t t, const double* G, double* Z,
                  double* V, double* w_host) {
  return guard_dev(h, [&] {
    if (t < 1 || t > 128) fail(kECapacity, "probe count per call must be in [1, 128]");
    probes_eq6(h->c, f->f, dinv, pkind, (int)t, (int)t, G, Z, V, w_host);
  });
}

int vl_sum_log(vl_ctx* h, int64_t n, const double* x, double* out) {
  return guard_dev(h, [&] { *out = sum_log(h->c, n, x); });
}

int vl_grad_probe_pass_split(vl_ctx* h, const vl_factor* f, int mode, const double* W, const double* d3,
                             const double* U, const double* V, int64_t t, int64_t t_glob, double* rowA, double* rowB,
                             double* s_out, double* cols4, const double* md3x, double* xicols2, int plain) {
  return guard_dev(h, [&] {
    if (mode != 3 && (t < 1 || t > 128)) fail(kECapacity, "probe shard width must be in [1, 128]");
    grad_probe_pass_split(h->c, f->f, mode, W, d3, U, V, (int)t, (int)t, (int)t_glob, rowA, rowB, s_out, cols4, md3x,
                          xicols2, plain);
  });
}

int vl_grad_scalar_terms(vl_ctx* h, const vl_factor* f, const double* b, const double* tvec, double* out4) {
  return guard_dev(h, [&] { grad_scalar_terms(h->c, f->f, b, tvec, out4); });
}

int vl_grad_dbeta(vl_ctx* h, int64_t n, const double* d1, const double* s, const double* W, const double* tvec,
                  const double* X, int64_t p, double* dbeta) {
  return guard_dev(h, [&] { grad_dF(h->c, n, d1, s, W, tvec, X, (int)p, dbeta); });
}

int vl_gamma_xi_terms(vl_ctx* h, const vl_factor* f, const double* y, const double* Fv, const double* b,
                      const double* W, const double* tvec, double* md3x, double* out3) {
  return guard_dev(h, [&] { gamma_xi_terms(h->c, f->f, y, Fv, b, W, tvec, md3x, out3); });
}

int vl_spmm(vl_ctx* h, const vl_factor* f, int op, int64_t t, const double* x, double* y) {
  return guard_dev(h, [&] {
    if (t < 1 || t > (1 << 20)) fail(kEConfig, "invalid column count");
    op_spmm(h->c, f->f, op, (int)t, (int)t, x, y);
  });
}

int vl_sptrsv(vl_ctx* h, const vl_factor* f, int transpose, int64_t t, const double* x, double* y) {
  return guard_dev(h, [&] {
    if (t < 1 || t > (1 << 20)) fail(kEConfig, "invalid column count");
    op_trsv(h->c, f->f, transpose != 0, (int)t, (int)t, x, y);
  });
}


int vl_pred_create(vl_ctx* h, const vl_pattern* p, double sigma2, double rho, double nu, const double* qxy, int64_t np,
                   const int32_t* nbr, int take, vl_pred** out) {
  return guard_dev(h, [&] {
    if (!h || !p || !out || (np > 0 && (!qxy || !nbr))) fail(kEConfig, "null pointer");
    auto* b = new vl_pred();
    try {
      pred_create(h->c, p->p, sigma2, rho, nu, qxy, np, nbr, take, b->b);
    } catch (...) {
      delete b;
      throw;
    }
    *out = b;
  });
}

int vl_pred_destroy(vl_pred* b) {
  return guard([&] { delete b; });
}

int vl_pred_get(vl_ctx* h, const vl_pred* b, int which, double* out) {
  return guard_dev(h, [&] {
    const size_t cnt = which == 0 ? (size_t)b->b.np * b->b.take : (size_t)b->b.np;
    const DevBuf& src = which == 0 ? b->b.val : b->b.Dp;
    if (which != 0 && which != 1) fail(kEConfig, "unknown prediction field");
    if (cnt) VL_CUDA(cudaMemcpyAsync(out, src.p, sizeof(double) * cnt, cudaMemcpyDeviceToHost, h->c.stream));
    VL_CUDA(cudaStreamSynchronize(h->c.stream));
  });
}

int vl_pred_mean(vl_ctx* h, const vl_pred* b, const double* b_dev, const double* Fp_dev, double* omega_dev) {
  return guard_dev(h, [&] { pred_mean(h->c, b->b, b_dev, Fp_dev, omega_dev); });
}

int vl_pred_z3(vl_ctx* h, const vl_factor* f, const double* W_dev, int64_t c, const double* z1, const double* z2,
               double* z3) {
  return guard_dev(h, [&] { pred_z3(h->c, f->f, W_dev, (int)c, z1, z2, z3); });
}

int vl_pred_accum(vl_ctx* h, const vl_pred* b, const double* U_dev, int64_t c, double* acc_dev, double* cov_dev) {
  return guard_dev(h, [&] { pred_accum(h->c, b->b, U_dev, (int)c, acc_dev, cov_dev); });
}

int vl_pred_lanczos(vl_ctx* h, const vl_factor* f, const vl_pred* b, const double* W_dev, int variant, int64_t k,
                    const double* start_dev, const double* dsig_dev, double breakdown_tol, double* var_dev,
                    int* achieved) {
  return guard_dev(h, [&] {
    if (!h || !f || !b || !W_dev || !start_dev || !achieved || (b->b.np > 0 && !var_dev))
      fail(kEConfig, "null pointer");
    if (k > (int64_t)1 << 20) fail(kECapacity, "Lanczos rank too large");
    *achieved = pred_lanczos(h->c, f->f, b->b, W_dev, variant, (int)k, start_dev, dsig_dev, breakdown_tol, var_dev);
  });
}

}  // extern "C"
