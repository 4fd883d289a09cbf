// Shared per-column scalar machinery of the multi-RHS PCG drivers
// (iterative.py:104-178): alpha/beta/residual recurrences, breakdown checks,
// convergence masks and Lanczos coefficient capture, finalised on the device
// by the last CTA of the reducing kernel.
#pragma once

#include "bodies.cuh"
#include "rows.cuh"

namespace vl {
namespace cg {

struct CgCols {
  double* nb;
  double* rz;
  double* alpha;
  double* beta;
  double* res;
  double* tolnb;
  int* active;
  int* iters;
  int* conv;
  int* status;   // [0] n_active, [1] error code, [2] error column
  double* errval;
  double* ah;    // [cap x t]
  double* bh;
};

VL_D void recount(const CgCols& K, int t) {
  __syncthreads();
  if (threadIdx.x == 0) {
    int na = 0;
    for (int c = 0; c < t; ++c) na += K.active[c];
    if (K.status[1] != 0) na = 0;
    K.status[0] = na;
  }
}

VL_D void set_error(const CgCols& K, int code, int c, double v) {
  if (atomicCAS(K.status + 1, 0, code) == 0) {
    K.status[2] = c;
    *K.errval = v;
  }
}

// ---- init: r = b, u = 0, hprev = 0, ||b||^2 --------------------------------
struct InitBody {
  const double* b;
  double* r;
  double* u;
  double* hprev;
  int ld;
  template <int G, int NU, int U, int NR>
  VL_D void run(int64_t s, bool valid, int gl, int t, double (&acc)[NR][NU * U]) const {
    if (!valid) return;
    double a[NU * U], z[NU * U];
    load_row<G, NU, U>(b, ld, s, gl, t, a);
    zero(z);
    store_row<G, NU, U>(r, ld, s, gl, t, a);
    store_row<G, NU, U>(u, ld, s, gl, t, z);
    store_row<G, NU, U>(hprev, ld, s, gl, t, z);
#pragma unroll
    for (int i = 0; i < NU * U; ++i) acc[0][i] += a[i] * a[i];
  }
};
struct InitFin {
  CgCols K;
  double tol;
  VL_D void operator()(const double* sums, int t) const {
    for (int c = threadIdx.x; c < t; c += blockDim.x) {
      const double nb = sqrt(sums[c]);
      K.nb[c] = nb;
      K.tolnb[c] = tol * nb;
      const bool act = nb != 0.0;
      K.active[c] = act ? 1 : 0;
      K.conv[c] = act ? 0 : 1;
      K.iters[c] = 0;
      K.beta[c] = 0.0;
      K.alpha[c] = 0.0;
      K.rz[c] = 0.0;
      K.res[c] = nb;
    }
    if (threadIdx.x == 0) K.status[1] = 0;
    recount(K, t);
  }
};

// ---- K0: h = z + beta h (elementwise, in place) ------------------------------
struct HUpdBody {
  const double* z;
  double* h;
  const double* beta;
  int ld;
  template <int G, int NU, int U, int NR>
  VL_D void run(int64_t s, bool valid, int gl, int t, double (&)[NR][NU * U]) const {
    if (!valid) return;
    double zs[NU * U], hs[NU * U];
    load_row<G, NU, U>(z, ld, s, gl, t, zs);
    load_row<G, NU, U>(h, ld, s, gl, t, hs);
#pragma unroll
    for (int i = 0; i < NU * U; ++i) {
      const int c = vl::Cols<G, NU, U>::col(gl, i);
      hs[i] = zs[i] + (c < t ? beta[c] : 0.0) * hs[i];
    }
    store_row<G, NU, U>(h, ld, s, gl, t, hs);
  }
};

struct K2Fin {
  CgCols K;
  int l;
  int cap;
  VL_D void operator()(const double* sums, int t) const {
    for (int c = threadIdx.x; c < t; c += blockDim.x) {
      if (!K.active[c]) {
        K.alpha[c] = 0.0;  // a deferred r/u update of a frozen column is then exact no-op
        continue;
      }
      const double hv = sums[c];
      if (hv <= 0.0) set_error(K, kEBreakdown, c, hv);
      const double al = K.rz[c] / hv;
      K.alpha[c] = al;
      if (l < cap) K.ah[(size_t)l * t + c] = al;
    }
    recount(K, t);
  }
};

struct K3Fin {
  CgCols K;
  int l;
  VL_D void operator()(const double* sums, int t) const {
    for (int c = threadIdx.x; c < t; c += blockDim.x) {
      if (!K.active[c]) continue;
      const double res = sqrt(sums[c]);
      K.res[c] = res;
      K.iters[c] = l + 1;
      if (res < K.tolnb[c]) {
        K.active[c] = 0;
        K.conv[c] = 1;
      }
    }
    recount(K, t);
  }
};

struct K4Fin {
  CgCols K;
  int l;
  int cap;
  VL_D void operator()(const double* sums, int t) const {
    for (int c = threadIdx.x; c < t; c += blockDim.x) {
      if (!K.active[c]) continue;
      const double rzn = sums[c];
      if (rzn <= 0.0) set_error(K, kEBreakdown, c, rzn);
      const double be = rzn / K.rz[c];
      K.beta[c] = be;
      K.rz[c] = rzn;
      if (l < cap) K.bh[(size_t)l * t + c] = be;
    }
    recount(K, t);
  }
};

}  // namespace cg
}  // namespace vl
