// Internal (C++) entry points behind the C-ABI.
#pragma once

#include "bodies.cuh"
#include "context.h"

namespace vl {

void knn_previous(const double* xy, int64_t n, int d, int m, int32_t* out, int nthreads);
void knn_previous_dev(Ctx& C, const double* xy_host, int64_t n, int d, int m, int32_t* out_host);
void knn_query_dev(Ctx& C, const double* train_host, int64_t n, const double* q_host, int64_t nq, int d, int m,
                   int32_t* out_host, double* dmin_host);
void pattern_build_host(Pattern& P, const double* xy, const int32_t* nbr, std::vector<int32_t>& ell,
                        std::vector<int32_t>& cnt, std::vector<int32_t>& fwd, std::vector<int32_t>& bwd,
                        std::vector<int32_t>& tptr, std::vector<int32_t>& tidx, std::vector<int32_t>& tmap);
void pattern_upload(Ctx& C, Pattern& P, const double* xy_factor_order, const int32_t* nbr_factor_order);

void factor_build(Ctx& C, const Pattern& P, Factor& F, double sigma2, double rho, double nu, bool want_grad);

void factor_refresh_transpose(Ctx& C, Factor& F);
void prof_collect(Ctx& C);
BView bview(const Factor& F, bool grad);
void op_spmm(Ctx& C, const Factor& F, int op, int t, int ld, const double* x, double* y);
void op_trsv(Ctx& C, const Factor& F, bool transpose, int t, int ld, const double* b, double* x);

}  // namespace vl
