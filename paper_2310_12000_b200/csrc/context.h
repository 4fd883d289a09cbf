// Internal objects behind the opaque C-ABI handles.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <string>
#include <vector>

#include "common.cuh"

namespace vl {

// Device buffer with RAII (the library owns its workspace; callers hand in
// plain device pointers for inputs/outputs).
struct DevBuf {
  void* p = nullptr;
  size_t bytes = 0;
  DevBuf() = default;
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  DevBuf(DevBuf&& o) noexcept : p(o.p), bytes(o.bytes) { o.p = nullptr; o.bytes = 0; }
  DevBuf& operator=(DevBuf&& o) noexcept {
    if (this != &o) { release(); p = o.p; bytes = o.bytes; o.p = nullptr; o.bytes = 0; }
    return *this;
  }
  ~DevBuf() { release(); }
  void release();
  void alloc(size_t nbytes);          // no-op when already large enough
  template <class T> T* as() const { return static_cast<T*>(p); }
};

// Per-tag kernel timing with CUDA events on the launching stream (bench.py's
// live roofline) + a launch counter (gpu_launches).
struct Prof {
  bool on = false;
  std::string only;           // when non-empty: events only around launches under this tag
  const char* tag = nullptr;  // current tag (set by ProfScope at call sites; null = untimed)
  double bytes = 0;           // algorithmic bytes of one launch under the current tag
  struct Rec {
    std::string tag;
    cudaEvent_t a, b;
    double bytes;
  };
  std::vector<Rec> pending;
  std::vector<cudaEvent_t> free_events;
  struct Agg {
    long count = 0;
    double ms = 0, bytes = 0;
  };
  std::vector<std::pair<std::string, Agg>> agg;
  long long launches = 0;
};

struct Ctx {
  int device = 0;
  Prof prof;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  int num_sms = 148;
  std::string last_error;
  // CTAs per SM for the dependency-driven solves (bounds the spinning warps)
  int trsv_blocks_per_sm = 4;
  // max nanosleep backoff while spinning on a dependency (0 = pure polling)
  int spin_max_ns = 64;
  // the same for the single-RHS solves: pure polling (measured after the warp-per-row items
  // took over the levels of <= 512 rows: 0 / 16 / 32 / 64 / 128 / 256 ns -> PCG iteration
  // 0.787 / 0.797 / 0.799 / 0.804 / 0.815 / 0.839 ms; t = 50 is flat, 4.61-4.64 ms)
  int spin_max_ns1 = 0;
  // thin solve levels: <= thin_passes * (1024 / G) rows run on a single CTA
  int thin_passes = 0;
  int min_thick_levels = 4;
  // dense head block of the solves (see head.cuh) and its scratch
  bool use_slabs = true;  // coalesced dependency slabs for the single-RHS solves
  bool use_local = true;  // SM-local sweeps for multi-column gather passes (rows_local_kernel)
  bool use_head = true;
  // multi-column solves walk the pattern's tile-blocked order (Pattern::fwd_torder) when x is large
  bool use_tiles = true;
  // sandwich-PCG product mode (pcg.cu) for t == 1 / t > 1:
  //   0: B h + B^T tmp passes, 1: B^T(om o y) fused into the backward solve,
  //   2: B^T(om o y) as a side-stream pass concurrent with the forward solve,
  //   3: (t == 1) mode 0 with D^-1 B h carried by recurrence (no B h pass)
  int pmode1 = 3;
  int pmodeT = 1;
  cudaStream_t side = nullptr;  // created on first use
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  DevBuf head_Y, head_Xh;
  // debug: per-row completion timestamps of the next triangular solves (n entries)
  long long* debug_tstamp = nullptr;
  // VL_FRONT: completed single-RHS solve items (device counter) and the host's running total
  DevBuf front;
  unsigned front_total = 0;
  // deterministic reduction scratch: per-block partials + ticket counters
  DevBuf red_partial;   // doubles
  DevBuf red_counter;   // unsigned ints (ring of slots)
  int red_slot = 0;
  // small pinned host staging for scalar read-back
  double* host_scalars = nullptr;
  DevBuf dev_scalars;
};

// Sparsity pattern of the Vecchia factor + solve schedules (once per dataset).
// Everything device-side is in STORAGE order: storage position s holds the
// factor row sperm[s].  Vectors passed to kernels are n x t row-major in
// storage order.
struct Pattern {
  int64_t n = 0;
  int d = 0;
  int m = 0;                // ELL width (max neighbour count)
  int64_t nnz_off = 0;      // number of stored off-diagonal entries
  int order_kind = 0;
  std::vector<int32_t> sperm;   // storage -> factor
  std::vector<int32_t> iperm;   // factor -> storage
  std::vector<int32_t> fwd_level_ptr, bwd_level_ptr;
  int nlev_fwd = 0, nlev_bwd = 0;
  int max_children = 0;
  // device
  DevBuf xy;        // n*d  coords (storage order)
  DevBuf nbr;       // n*m  int32 storage index of neighbour k (reference in-row order)
  DevBuf cnt;       // n    int32 neighbour count
  DevBuf fidx;      // n    int32 factor index of storage row
  DevBuf fwd_order; // fwd_len int32 storage rows in (level, position) order, levels padded to 32 with -1
  DevBuf bwd_order; // bwd_len int32 storage rows in (height, position) order, padded likewise
  int64_t fwd_len = 0, bwd_len = 0;
  DevBuf fwd_lptr, bwd_lptr;  // device copies of the padded level pointers
  DevBuf fwd_items, bwd_items;  // single-RHS work items (light 32-row chunks / heavy rows)
  DevBuf fwd_order1, bwd_order1, bwdnh_order1;  // the orders as the light items see them (api.cpp)
  int64_t fwd_nitems = 0, bwd_nitems = 0;
  // dense head block (see pattern.cpp): rows of forward levels < head_L
  int64_t head_max = 3072;
  int head_L = 0;
  int64_t head_H = 0;
  std::vector<int32_t> head_rows_h, head_pos_h, head_nbr_h;
  std::vector<int32_t> bwdnh_order_h, bwdnh_level_ptr;
  DevBuf head_rows;   // H      storage row of head position h (level order)
  DevBuf head_pos;    // n      head position of a storage row or -1
  DevBuf head_nbr;    // H*m    head positions of the row's neighbours
  DevBuf bwdnh_order, bwdnh_lptr, bwdnh_items;  // backward schedule without the head rows
  int64_t bwdnh_len = 0, bwdnh_nitems = 0;
  int64_t fwd_items_head_end = 0;  // forward items covering the head levels
  // tile-blocked topological orders of the rows outside the head for the multi-column
  // solves (pattern.cpp); empty when the pattern has no wide levels / no spatial order
  int tile_K = 64, tile_S = 6;
  bool tile_tail = false;  // join a short narrow tail of levels to the last band (measured: no gain)
  size_t tile_min_bytes = (size_t)96 << 20;  // x (n x ld doubles) below this stays in level order (fits L2)
  int child_late = 16;  // pattern.cpp: dependencies within this many levels of the row are listed last
  std::vector<int32_t> nbr_s_h, map_s_h;  // host staging, released after the upload
  bool has_solve_order = false;
  DevBuf nbr_s, map_s;  // n*m  solve-ordered copy of nbr / slot of its value in Factor::val (or -1)
  int64_t tile_min_rows = 4096, tile_min_n = 100000;
  std::vector<int32_t> fwd_torder_h, bwd_torder_h;
  DevBuf fwd_torder, bwd_torder;
  int64_t fwd_tlen = 0, bwd_tlen = 0;
  DevBuf tptr;      // n+1  int32 children CSR (= CSR of B^T) in storage order
  DevBuf tidx;      // nnz  int32 child storage row
  DevBuf tmap;      // nnz  int32 ELL slot (child*m + k) holding B[child, s]
  // Coalesced dependency slabs of the light single-RHS items: item k owns
  // entry columns [off[k], off[k] + w[k]) (w = max deps of its 32 rows);
  // entry e of lane l sits at (off + e) * 32 + l, idx = dependency storage
  // row or -1, map = ELL slot of its value in Factor::val or -1.
  struct Slabs {
    DevBuf off, w, idx, map;
    int64_t nent = 0;  // entries (multiple of 32)
  };
  Slabs fwd_sl, bwd_sl, bwdnh_sl;
};

// Factor values at one theta (device resident, storage order).
struct Factor {
  const Pattern* pat = nullptr;
  double sigma2 = 0, rho = 0, nu = 0;
  bool has_grad = false;
  DevBuf val;     // n*m  ELL values of B's off-diagonal (-A_i), zero padded
  DevBuf valT;    // nnz  values of B^T in children-CSR order
  DevBuf D;       // n
  DevBuf dval;    // n*m  d B / d rho (off-diagonal, zero padded)
  DevBuf dD_rho;  // n
  DevBuf dD_sig;  // n    d D / d sigma2 = D / sigma2
  DevBuf err;     // 4 ints: [code, row(factor idx) ...]
  DevBuf headX;   // H*H  dense B_HH^-1, column-major (head order), lower triangular
  DevBuf headXr;  // H*H  the same, row-major
  DevBuf sv_fwd, sv_bwd, sv_bwdnh;  // slab values (Pattern::Slabs::map gathered from val)
  DevBuf val_s;   // n*m  val in the solve order of Pattern::nbr_s
};

}  // namespace vl
