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
/* The same search on the device (1 <= d <= 3, m <= 256): brute force below
 * 4096 points, uniform grids over growing prefixes above; identical output. */
int vl_knn_previous_dev(vl_ctx* ctx, const double* xy_host, int64_t n, int d, int m, int32_t* out_host);
/* Nearest TRAINING neighbours of prediction points (replaces the cKDTree query
 * + lexsort of vecchia.py:411-421): row q = the min(m, n) training indices
 * closest to query q, nearest first, ties to the smaller index; dmin_host[q] =
 * distance to the nearest (the caller rejects duplicates, vecchia.py:416-420). */
int vl_knn_query(vl_ctx* ctx, const double* train_host, int64_t n, const double* q_host, int64_t nq, int d, int m,
                 int32_t* out_host, double* dmin_host);

/* ---- pattern (once per dataset) ---------------------------------------------
 * Replaces the structural part of vecchia.py:220-283 (CSR layout of B,
 * diagonal last) and the SuperLU symbolic setup of vecchia.py:159-170.
 * order_kind: 0 factor order, 1 spatial (Hilbert/Morton) order, 2 level-major. */
int vl_pattern_create(vl_ctx* ctx, int64_t n, int d, int m, const double* xy_host, const int32_t* nbr_host,
                      int order_kind, vl_pattern** out);
int vl_pattern_destroy(vl_pattern* p);
/* sperm_host: n int32, storage position -> factor index */
int vl_pattern_perm(const vl_pattern* p, int32_t* sperm_host);
/* info (10 entries): [n, d, m, nnz_off, n_levels_fwd, n_levels_bwd, max_children, order_kind,
 *   head_levels, head_rows] -- the last two describe the dense head block of the solves (0 = off) */
int vl_pattern_info(const vl_pattern* p, int64_t* info);
/* Row order the multi-column solves walk when x does not fit in L2 (transpose = 0: B, 1: B^T):
 * storage rows outside the head block, wide levels cut into bands and walked tile by tile
 * (a topological order of the dependency graph).  *len = 0 when the pattern keeps the level
 * order.  order_host may be NULL (length query) or hold *len int32.  No reference counterpart:
 * scipy's spsolve_triangular (vecchia.py:161-174) walks rows in index order. */
int vl_pattern_solve_order(const vl_pattern* p, int transpose, int64_t* len, int32_t* order_host);

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

/* ---- instrumentation ----------------------------------------------------------
 * Per-tag kernel timing with CUDA events on the context stream (tags mark the
 * hot kernels: cg_*, probe_*, grad_*, newton_*, factor_*) and a launch
 * counter.  vl_prof_report writes "tag\tlaunches\tms\talgorithmic_bytes\n"
 * lines into buf. */
int vl_prof_enable(vl_ctx* ctx, int on);
int vl_prof_reset(vl_ctx* ctx);
/* restrict the events to launches under one tag (NULL / "": every tagged launch);
 * the launch counter keeps counting every launch */
int vl_prof_only(vl_ctx* ctx, const char* tag);
int vl_prof_report(vl_ctx* ctx, char* buf, int len, int64_t* launches);

/* ---- Laplace objective (iterative backend, VADU preconditioner) ---------- */

/* likelihood family: 0 bernoulli-logit, 1 bernoulli-probit, 2 gamma
 * (likelihoods.py:62-181); shape = gamma shape xi */
typedef struct {
  int family;
  double shape;
} vl_lik;

/* subset of BackendConfig (laplace.py:51-84) driving find_mode */
typedef struct {
  double mode_cg_tol; /* min(cg_tol, 1e-4), laplace.py:80-84 */
  int cg_max_iter;
  int newton_max_iter;
  double newton_grad_tol;
  double newton_obj_tol;
  int precond; /* eq6 preconditioner of the Newton systems: 0 vadu, 1 l1, 2 lva, 3 diag, 4 identity */
} vl_newton_cfg;

/* Damped-Newton mode b* (replaces laplace.py:204-287 find_mode).  Device
 * vectors of length n (storage order): y, F in; b, W, d1, d3 out.
 * out[0..6] = logp, quad, objective, grad_norm, newton_iters, converged,
 * n_cg_solves; cg_iters (host, optional) = CG iterations per Newton step.
 * Returns VL_ECONVERGENCE when not converged (outputs still written). */
int vl_find_mode(vl_ctx* ctx, const vl_factor* f, const vl_lik* lik, const vl_newton_cfg* cfg, const double* y_dev,
                 const double* F_dev, double* b_dev, double* W_dev, double* d1_dev, double* d3_dev, double* out_host,
                 int32_t* cg_iters_host, int cg_iters_cap);

/* Probes for VADU (replaces preconditioners.py:121-122 sample_block with the
 * reference's Gaussian base draws G, and iterative.py:268-271 psolves):
 * Z = B^T (sqrt(d) o G), V = P^-1 Z = B^-1 (G / sqrt(d)), w_host[c] = z_c . v_c.
 * G, Z, V: n x t device (storage order). */
int vl_probes_vadu(vl_ctx* ctx, const vl_factor* f, const double* W_dev, int64_t t, const double* G_dev, double* Z_dev,
                   double* V_dev, double* w_host);

/* PCG on (W + B^T D^-1 B) U = Bm with the VADU preconditioner, t columns
 * (replaces iterative.py:104-178 pcg_solve per column, laplace.py:290-309).
 * Host outputs per column: iterations, converged flag, residual norm; with
 * capture, alpha/beta histories [hist_cap x t] (row l = CG iteration l). */
int vl_pcg_vadu(vl_ctx* ctx, const vl_factor* f, const double* W_dev, int64_t t, const double* B_dev, double* U_dev,
                double tol, int max_iter, int capture, int32_t* iters_host, int32_t* conv_host, double* res_host,
                double* alpha_host, double* beta_host, int hist_cap);

/* out6 = [sum log D, sum log(W + 1/D), sum dD_s2/D, sum dD_rho/D,
 *         -sum dD_s2/(D(DW+1)), -sum dD_rho/(D(DW+1))]
 * (laplace.py:331-336, 502, 511-513) */
int vl_factor_sums(vl_ctx* ctx, const vl_factor* f, const double* W_dev, double* out6_host);

/* Fused gradient pass over the probe solves U and psolves V (n x t):
 * s_out = 0.5 dlogdet/dmu (laplace.py:389-436, VADU control variates) and the
 * per-probe STE terms cols4 = [h_s2 | r_s2 | h_rho | r_rho] (4 x t, host)
 * (laplace.py:493-541, iterative.py:280-304).  With md3x (gamma), xicols2 =
 * [h_xi | r_xi] (laplace.py:543-576). */
int vl_grad_probe_pass(vl_ctx* ctx, const vl_factor* f, const double* W_dev, const double* d3_dev, const double* U_dev,
                       const double* V_dev, int64_t t, double* s_dev, double* cols4_host, const double* md3x_dev,
                       double* xicols2_host, int plain);
/* plain != 0: preconditioners without a control variate (laplace.py:433-436):
 * s = 0.5 md3 mean_t(U o V) and only the h columns are meaningful. */

/* ---- other eq6 preconditioners (preconditioners.py:338-387) -------------------
 * variant 0 vadu, 1 l1 (P = B^T diag(W + 1/D) B), 2 lva (B^T diag(1/D) B),
 * 3 diag (diag(W + diag(B^T D^-1 B))), 4 identity.  vl_precond_dinv writes 1/d
 * of the sandwich / diagonal; pkind = 0 for variants 0-2 (sandwich), 1 for 3-4
 * (diagonal).  vl_pcg_eq6 / vl_probes_eq6 are vl_pcg_vadu / vl_probes_vadu for
 * any variant (sample_block + solve of the chosen P); vl_sum_log returns
 * sum_i log x_i (log det P = -sum log dinv). */
int vl_precond_dinv(vl_ctx* ctx, const vl_factor* f, int variant, const double* W_dev, double* dinv_dev);
int vl_pcg_eq6(vl_ctx* ctx, const vl_factor* f, const double* W_dev, const double* dinv_dev, int pkind, int64_t t,
               const double* b_dev, double* u_dev, double tol, int max_iter, int capture, int32_t* iters_host,
               int32_t* converged_host, double* res_host, double* alpha_host, double* beta_host, int hist_cap);
int vl_probes_eq6(vl_ctx* ctx, const vl_factor* f, const double* dinv_dev, int pkind, int64_t t, const double* G_dev,
                  double* Z_dev, double* V_dev, double* w_host);
int vl_sum_log(vl_ctx* ctx, int64_t n, const double* x_dev, double* out_host);

/* ---- LRAC preconditioner and the eq7 system (preconditioners.py:167-214,
 * 249-320; laplace.py:118-182) ------------------------------------------------ */
typedef struct vl_pred vl_pred;    /* prediction blocks Bpo, Dp (vecchia.py:364-441) */
typedef struct vl_lrac vl_lrac;    /* rank-k pivoted Cholesky of Sigma (theta only) */
typedef struct vl_lracw vl_lracw;  /* Woodbury core M = I + L^T W L for one W       */

/* greedy pivoted Cholesky (pivoted_cholesky_with_pivots, preconditioners.py:288-320);
 * piv_host: factor-order pivots (>= k entries), keff: achieved rank */
int vl_lrac_create(vl_ctx* ctx, const vl_factor* f, int k, double tol, vl_lrac** out, int32_t* piv_host, int* keff);
int vl_lrac_destroy(vl_lrac* l);
/* L (n x k row-major, storage order) to host */
int vl_lrac_get_L(vl_ctx* ctx, const vl_lrac* l, double* host);
/* LowRankPlusDiagonal(L, 1/W) (preconditioners.py:176-190); out2 = [log det M, sum log W];
 * VL_ECAPABILITY when some W <= 0 (laplace.py:122-127) */
int vl_lrac_prepare(vl_ctx* ctx, const vl_lrac* l, const double* W_dev, vl_lracw** out, double* out2_host);
int vl_lracw_destroy(vl_lracw* w);
/* z = P^-1 r (Woodbury, preconditioners.py:192-196), n x t */
int vl_lrac_apply_inv(vl_ctx* ctx, const vl_lracw* w, int64_t t, const double* r_dev, double* z_dev);
/* PCG on (SigmaTilde + W^-1) U = Bm with the LRAC preconditioner (eq7 probes) */
int vl_lrac_pcg(vl_ctx* ctx, const vl_lracw* w, int64_t t, const double* B_dev, double* U_dev, double tol,
                int max_iter, int capture, int32_t* iters_host, int32_t* conv_host, double* res_host,
                double* alpha_host, double* beta_host, int hist_cap);
/* u = (W + SigmaTilde^-1)^-1 rhs through the eq7 form (laplace.py:176-179) */
int vl_lrac_solve_system(vl_ctx* ctx, const vl_lracw* w, int64_t t, const double* rhs_dev, double* u_dev, double tol,
                         int max_iter, int32_t* iters_host);
/* y = SigmaTilde x = B^-1 (D o B^-T x) (vecchia.py:185-192) */
int vl_apply_sigma_tilde(vl_ctx* ctx, const vl_factor* f, int64_t t, const double* x_dev, double* y_dev);
/* Z = sqrt(1/W) o Gn + L Gk (preconditioners.py:204-207), V = P^-1 Z, w_c = z_c . v_c */
int vl_lrac_probes(vl_ctx* ctx, const vl_lracw* w, int64_t t, const double* Gn_dev, const double* Gk_dev,
                   double* Z_dev, double* V_dev, double* w_host);
/* find_mode with the LRAC preconditioner / eq7 system */
int vl_find_mode_lrac(vl_ctx* ctx, const vl_factor* f, const vl_lrac* l, const vl_lik* lik, const vl_newton_cfg* cfg,
                      const double* y_dev, const double* F_dev, double* b_dev, double* W_dev, double* d1_dev,
                      double* d3_dev, double* out_host, int32_t* cg_iters_host, int cg_iters_cap);
/* LRAC gradient pieces (replaces the preconditioner == "lrac" branches of
 * laplace.py:421-431 d logdet/d mu, 369-386 _lrac_dL, 527-533 dP_trace/dP_op and
 * the eq7 dA_op = -SigmaTilde dQ SigmaTilde of 493-541).  U = A^-1 Z, V = P^-1 Z
 * (n x t device).  s_dev (n) = 0.5 d logdet / d mu; host outputs: hcols/rcols
 * 2 x t (sigma2, rho) STE samples, dPt 2 control-variate traces; md3x_dev
 * (gamma only, else NULL): xicols 2 x t (h_xi, r_xi), xis = [sum G2 m3, sum m3/W]. */
int vl_lrac_grad(vl_ctx* ctx, const vl_lracw* w, int64_t t, const double* U_dev, const double* V_dev,
                 const double* d3_dev, const double* md3x_dev, double* s_dev, double* hcols_host, double* rcols_host,
                 double* dPt_host, double* xicols_host, double* xis_host, int plain);
/* plain != 0: the eq7 plain estimator (l2; laplace.py:433-434, no control variate). */

/* Probe-sharded vl_lrac_grad (multi-GPU; the LRAC mu-derivative of
 * laplace.py:421-431 needs per-row statistics over all t_glob probes):
 *   mode 1: rowA = [sum_c H, sum_c R] over the local t columns, plus every
 *           per-column / scalar output of vl_lrac_grad (hcols, rcols, dPt, xicols, xis);
 *   -- caller allreduces rowA (n x 2) --
 *   mode 2: rowB = [sum_c (H - hbar)(R - rbar), sum_c (R - rbar)^2];
 *   -- caller allreduces rowB --
 *   mode 3: s from rowA, rowB and diag(L M^-1 L^T). */
int vl_lrac_grad_split(vl_ctx* ctx, const vl_lracw* w, int mode, int64_t t, int64_t t_glob, const double* U_dev,
                       const double* V_dev, const double* d3_dev, const double* md3x_dev, double* rowA_dev,
                       double* rowB_dev, double* s_dev, double* hcols_host, double* rcols_host, double* dPt_host,
                       double* xicols_host, double* xis_host, int plain);

/* ---- other low-rank-plus-diagonal preconditioners ----------------------------
 * (LowRankPlusDiagonalPreconditioner, preconditioners.py:161-214, 338-387)
 * vl_lowrank_create: kind 1 pchol-precision (pivoted Cholesky of B^T D^-1 B,
 * PrecisionAccessor 228-246), kind 2 rowsel (U = B_S^T D_S^-1/2 over the k rows
 * with the largest sum_j B_ij^2 / D_i, ties to the lower index, 323-335).
 * vl_lowrank_einv: 1/e for kind 1 (e = W) or kind 2 = l2 (e = diag(SigmaTilde)
 * + 1/W).  vl_lowrank_prepare: Woodbury core for P = U U^T + diag(e) (l may be
 * NULL: k = 0, the l2 diagonal) with the eq6 (W + Q) or eq7 (SigmaTilde + 1/W)
 * system; out2 = [log det M, sum log(1/e)]; the vl_lrac_pcg / _solve_system /
 * _probes / _apply_inv entry points then work on it.  vl_diag_sigma_tilde:
 * diag(SigmaTilde) (vecchia.py:198-212), storage order.  vl_find_mode_lowrank:
 * find_mode with these preconditioners (wb_kind 1 eq6 low rank, 2 l2). */
int vl_lowrank_create(vl_ctx* ctx, const vl_factor* f, int kind, int k, double tol, vl_lrac** out,
                      int32_t* pivots_host, int* keff);
int vl_lowrank_einv(vl_ctx* ctx, int64_t n, int kind, const double* W_dev, const double* diag_st_dev,
                    double* einv_dev);
int vl_lowrank_prepare(vl_ctx* ctx, const vl_factor* f, const vl_lrac* l, const double* Wop_dev,
                       const double* einv_dev, int eq6, vl_lracw** out, double* out2_host);
int vl_diag_sigma_tilde(vl_ctx* ctx, const vl_factor* f, double* out_dev);
int vl_find_mode_lowrank(vl_ctx* ctx, const vl_factor* f, const vl_lrac* l, int wb_kind, const double* diag_st_dev,
                         const vl_lik* lik, const vl_newton_cfg* cfg, const double* y_dev, const double* F_dev,
                         double* b_dev, double* W_dev, double* d1_dev, double* d3_dev, double* out_host,
                         int32_t* cg_iters_host, int cg_iters_cap);

/* Probe-sharded split of vl_grad_probe_pass for multi-GPU runs (the per-row
 * control-variate weights need all t_glob probes):
 *   mode 1: rowA = [sum_c U*V, sum_c (BV)^2] over the local t columns (n x 2,
 *           device) + local STE partials cols4 (and xicols2);
 *   -- caller allreduces rowA --
 *   mode 2: rowB = [sum_c (H - hbar)(R - rbar), sum_c (R - rbar)^2];
 *   -- caller allreduces rowB --
 *   mode 3: s_out from rowA, rowB (elementwise). */
int vl_grad_probe_pass_split(vl_ctx* ctx, const vl_factor* f, int mode, const double* W_dev, const double* d3_dev,
                             const double* U_dev, const double* V_dev, int64_t t, int64_t t_glob, double* rowA_dev,
                             double* rowB_dev, double* s_dev, double* cols4_host, const double* md3x_dev,
                             double* xicols2_host, int plain);

/* out4 = [b^T dQ_s2 b, tvec^T dQ_s2 b, b^T dQ_rho b, tvec^T dQ_rho b]
 * (vecchia.py:357-361 quad_dprecision; laplace.py:537-541) */
int vl_grad_scalar_terms(vl_ctx* ctx, const vl_factor* f, const double* b_dev, const double* tvec_dev,
                         double* out4_host);

/* dbeta = X^T (-d1 + s - W o tvec)  (laplace.py:578-580); X: n x p device */
int vl_grad_dbeta(vl_ctx* ctx, int64_t n, const double* d1_dev, const double* s_dev, const double* W_dev,
                  const double* tvec_dev, const double* X_dev, int64_t p, double* dbeta_host);

/* gamma shape terms (likelihoods.py:164-170 at mu = F + b):
 * md3x = y e^{-mu} (device), out3 = [sum(log y - mu - y e^{-mu}),
 * sum(tvec (-1 + y e^{-mu})), sum(md3x / (W + 1/D))] */
int vl_gamma_xi_terms(vl_ctx* ctx, const vl_factor* f, const double* y_dev, const double* F_dev, const double* b_dev,
                      const double* W_dev, const double* tvec_dev, double* md3x_dev, double* out3_host);

/* ---- prediction (predict.py:45-101, vecchia.py:364-441) ----------------------
 * vl_pred_create: Bpo rows (-A, A = K^-1 k over the `take` nearest training
 * points given by nbr_host = np x take FACTOR-order indices, nearest first)
 * and Dp = sigma2 - k.A for the np prediction points qxy_host (np x d);
 * status 40 when a neighbour covariance submatrix is not positive definite
 * (_chol_or_report).  vl_pred_get: which 0 = Bpo values (np x take), 1 = Dp.
 * vl_pred_mean: omega = F_p - Bpo b* (device, b in storage order).
 * vl_pred_z3: z3 = W^1/2 z1 + B^T (D^-1/2 z2) for c samples (n x c storage
 * order; the rhs of one CG solve per sample, predict.py:90-93).
 * vl_pred_accum: z4 = Bpo u for the c solved samples; acc[q] += sum_c z4^2 in
 * sample order; cov (np x np, optional) += z4 z4^T (predict.py:94-98). */
int vl_pred_create(vl_ctx* ctx, const vl_pattern* p, double sigma2, double rho, double nu, const double* qxy_host,
                   int64_t np, const int32_t* nbr_host, int take, vl_pred** out);
int vl_pred_destroy(vl_pred* b);
int vl_pred_get(vl_ctx* ctx, const vl_pred* b, int which, double* out_host);
int vl_pred_mean(vl_ctx* ctx, const vl_pred* b, const double* b_dev, const double* Fp_dev, double* omega_dev);
int vl_pred_z3(vl_ctx* ctx, const vl_factor* f, const double* W_dev, int64_t c, const double* z1_dev,
               const double* z2_dev, double* z3_dev);
int vl_pred_accum(vl_ctx* ctx, const vl_pred* b, const double* U_dev, int64_t c, double* acc_dev, double* cov_dev);
/* vl_pred_lanczos: rank-k Lanczos approximation of diag(Omega_p) (predict.py:104-172
 * latent_var_lanczos / _lanczos_correction, iterative.py:181-219 lanczos_partial).
 * variant 0 "none", 1 "l1", 2 "l2" (needs W > 0: status 5, and dsig_dev =
 * diag(SigmaTilde), n).  start_dev (n, storage order) = the column mean of
 * RT = Bpo^T, i.e. (1/np) Bpo^T 1; the variant's transformation of RT is applied
 * by the library.  RT is never materialised densely: S = Q^T RT is formed as
 * Bpo Q' over the transformed Lanczos basis, O((n + np) k) memory.  var_dev (np)
 * receives Dp + correction; *achieved = Krylov order reached (k unless a
 * recurrence norm fell below breakdown_tol; 0 = zero start vector, var = Dp). */
int vl_pred_lanczos(vl_ctx* ctx, const vl_factor* f, const vl_pred* b, const double* W_dev, int variant, int64_t k,
                    const double* start_dev, const double* dsig_dev, double breakdown_tol, double* var_dev,
                    int* achieved);

/* ---- dense fp64 kernels of the low-rank paths (debug / test entry points) ----
 * Column-major, BLAS argument meaning: C = alpha op(A) [diag(kw)] op(B) + beta C with
 * op(A) m x k, op(B) k x n; kw (length k, device) optional; lower != 0 writes only
 * C(i, j), i >= j.  Replaces the cublasDgemm / cublasDsyrk calls of the LRAC Woodbury
 * core (preconditioners.py:176-202) and of _lrac_dL (laplace.py:369-386). */
int vl_dgemm(vl_ctx* ctx, int transa, int transb, int64_t m, int64_t n, int64_t k, double alpha, const double* A_dev,
             int64_t lda, const double* B_dev, int64_t ldb, double beta, double* C_dev, int64_t ldc,
             const double* kw_dev, int lower);
/* Linv = L^-1 for lower-triangular L (k x k, column-major); replaces cublasDtrsm
 * (triangular solves are applied as products with the inverse). */
int vl_dtrtri_lower(vl_ctx* ctx, int64_t k, const double* L_dev, int64_t ldl, double* Linv_dev, int64_t ldi);

/* Probes supplied by the caller instead of drawn from N(0, P) -- the reference's
 * ProbeSet injection into neg_marginal_loglik / gradient (laplace.py:340, 439;
 * iterative.py:222-244), e.g. Rademacher probes.
 * vl_probes_rademacher: Z (n x t, storage order) with entry (factor row i, column c) =
 *   -1 if the top bit of splitmix64(seed * 0x9E3779B97F4A7C15 + i * t_glob + c0 + c) is set, else +1.
 * vl_probes_given: V = P^-1 Z (eq6 sandwich / diagonal preconditioner of vl_precond_dinv) and
 *   w_host[c] = z_c . v_c (the SLQ weights, iterative.py:268-271). */
int vl_probes_rademacher(vl_ctx* ctx, const vl_pattern* p, int64_t t, int64_t t_glob, int64_t c0, uint64_t seed,
                         double* Z_dev);
int vl_probes_given(vl_ctx* ctx, const vl_factor* f, const double* dinv_dev, int pkind, int64_t t, const double* Z_dev,
                    double* V_dev, double* w_host);

#ifdef __cplusplus
}
#endif

#endif /* VLGPX_H */
