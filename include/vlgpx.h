/*
 * vlgpx -- B200-native (sm_100a) Vecchia-Laplace hot path, C ABI.
 *
 * Drop-in boundary for the iterative Vecchia-Laplace path of the reference
 * Python package `vlgp` (arXiv 2310.12000).  The reference has no native
 * plugin ABI; its boundary is its Python API.  Each entry
 * point below names the reference function it replaces.  The Python package
 * `paper_2310_12000_b200` binds this library with ctypes and mirrors the
 * reference API on top of it.
 *
 * Conventions
 *  - Opaque handles; plain pointers and sizes; no torch types.
 *  - "host" pointers are CPU memory, "dev" pointers are CUDA device memory
 *    on the context's device.
 *  - Device vectors are n x t row-major (t = columns / right-hand sides) in
 *    STORAGE order: storage row s holds factor row sperm[s]
 *    (vl_pattern_perm).  Host-side factor-order arrays are permuted once by
 *    the caller.
 *  - Every call returns a status: 0 ok, 2 config, 3 data, 5 capability,
 *    6 capacity, 40 factorization, 41 breakdown, 42 convergence, 50 CUDA,
 *    51 internal.  vl_last_error() returns the message of the last failure
 *    on the calling thread.  Status classes map 1:1 onto vlgp/errors.py.
 *  - Work is ordered on the context's stream; calls that return host
 *    scalars synchronise that stream.
 */
#ifndef VLGPX_H
#define VLGPX_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct vl_ctx vl_ctx;
typedef struct vl_pattern vl_pattern;
typedef struct vl_factor vl_factor;
typedef struct vl_mode vl_mode;
typedef struct vl_probes vl_probes;

#define VL_OK 0
#define VL_ECONFIG 2
#define VL_EDATA 3
#define VL_ECAPABILITY 5
#define VL_ECAPACITY 6
#define VL_EFACTORIZATION 40
#define VL_EBREAKDOWN 41
#define VL_ECONVERGENCE 42
#define VL_ECUDA 50
#define VL_EINTERNAL 51

/* ---- library / context ---------------------------------------------------- */
int vl_version(void);
const char* vl_last_error(void);
/* device: CUDA ordinal; stream: cudaStream_t to run on (NULL -> legacy default stream) */
int vl_ctx_create(int device, void* stream, vl_ctx** out);
int vl_ctx_destroy(vl_ctx* ctx);
int vl_ctx_sync(vl_ctx* ctx);
/* info[0]=device, info[1]=SM count */
int vl_ctx_info(vl_ctx* ctx, int64_t* info);

/* ---- neighbour search (replaces vecchia.py:59-98 find_neighbors) ------------
 * xy_host: n x d coordinates ALREADY in factor (permuted) order.
 * out_host: n x m int32, row i = indices (< i) of the min(i,m) nearest earlier
 * points, nearest first, ties to the smaller index; padded with -1. */
int vl_knn_previous(const double* xy_host, int64_t n, int d, int m, int32_t* out_host, int n_threads);

/* ---- pattern (once per dataset) ---------------------------------------------
 * Replaces the structural part of vecchia.py:220-283 (CSR layout of B,
 * diagonal last) and the SuperLU symbolic setup of vecchia.py:159-170.
 * order_kind: 0 factor order, 1 spatial (Hilbert/Morton) order, 2 level-major. */
int vl_pattern_create(vl_ctx* ctx, int64_t n, int d, int m, const double* xy_host, const int32_t* nbr_host,
                      int order_kind, vl_pattern** out);
int vl_pattern_destroy(vl_pattern* p);
/* sperm_host: n int32, storage position -> factor index */
int vl_pattern_perm(const vl_pattern* p, int32_t* sperm_host);
/* info: [n, d, m, nnz_off, n_levels_fwd, n_levels_bwd, max_children, order_kind] */
int vl_pattern_info(const vl_pattern* p, int64_t* info);

/* ---- factor (per theta) ------------------------------------------------------
 * Replaces vecchia.py:220-283 build_factor (values) and vecchia.py:286-337
 * factor_gradient when want_grad != 0 (d/d sigma2 and d/d rho). */
int vl_factor_build(vl_ctx* ctx, const vl_pattern* p, double sigma2, double rho, double nu, int want_grad,
                    vl_factor** out);
int vl_factor_destroy(vl_factor* f);
/* which: 0 D, 1 dD/dsigma2, 2 dD/drho (n doubles); 3 B off-diagonal ELL values,
 * 4 dB/drho ELL values (n*m doubles, storage order, zero padded) */
int vl_factor_get(vl_ctx* ctx, const vl_factor* f, int which, double* host_out);
/* overwrite one field from host values (same layout as vl_factor_get); used to
 * replay externally computed factors (kernel-level parity on identical B). */
int vl_factor_set(vl_ctx* ctx, vl_factor* f, int which, const double* host_in);

/* ---- kernel-level operators (device pointers, n x t, storage order) -------
 * op: 0 -> y = B x, 1 -> y = B^T x, 2 -> y = (dB/drho) x
 * (the csr/csc matvecs of vecchia.py:176-183, 349-353). */
int vl_spmm(vl_ctx* ctx, const vl_factor* f, int op, int64_t t, const double* x_dev, double* y_dev);
/* y = B^-1 x (transpose=0) or B^-T x (transpose=1)  (vecchia.py:172-174) */
int vl_sptrsv(vl_ctx* ctx, const vl_factor* f, int transpose, int64_t t, const double* x_dev, double* y_dev);

#ifdef __cplusplus
}
#endif

#endif /* VLGPX_H */
