// Prediction blocks and the simulation variance estimator on the device.
#pragma once

#include "context.h"

namespace vl {

struct PredBlocks {
  int64_t np = 0;
  int take = 0;
  int d = 0;
  DevBuf qxy;  // np x d prediction coordinates
  DevBuf nbr;  // np x take  training STORAGE rows, nearest first
  DevBuf cnt;  // np         (= take)
  DevBuf val;  // np x take  Bpo values (-A)
  DevBuf Dp;   // np
};

void pred_create(Ctx& C, const Pattern& P, double sigma2, double rho, double nu, const double* qxy_host, int64_t np,
                 const int32_t* nbr_factor_host, int take, PredBlocks& B);
void pred_mean(Ctx& C, const PredBlocks& B, const double* b_dev, const double* Fp_dev, double* omega_dev);
void pred_z3(Ctx& C, const Factor& F, const double* W, int c, const double* z1, const double* z2, double* z3);
void pred_accum(Ctx& C, const PredBlocks& B, const double* U_dev, int c, double* acc_dev, double* cov_dev);
// Rank-k Lanczos variances (lanczos.cu); returns the achieved rank (0: zero start vector).
int pred_lanczos(Ctx& C, const Factor& F, const PredBlocks& B, const double* W, int variant, int k,
                 const double* start_raw, const double* dsig, double breakdown_tol, double* var_out);

}  // namespace vl
