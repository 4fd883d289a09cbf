"""B200-native Vecchia-Laplace hot path (drop-in for the iterative path of vlgp).

The public names mirror the reference package's re-exports
(vlgp/__init__.py:10-64).  All heavy arithmetic runs in the in-tree sm_100a
library ``libvlgpx.so``; there is no CPU fallback.
"""

from .covariance import CovarianceSpec, Locations, cov_grad, cov_submatrix, cov_value
from .errors import (
    BreakdownError,
    CapabilityError,
    CapacityError,
    ConfigError,
    ConvergenceError,
    DataError,
    DeviceError,
    FactorizationError,
    NumericalError,
    VlgpError,
)
from .vecchia import (
    VecchiaFactor,
    build_factor,
    factor_gradient,
    find_neighbors,
    make_factor,
    order_random,
)

__version__ = "0.1.0"
from .laplace import (BackendConfig, LaplaceState, find_mode, gradient, make_probes, neg_marginal_loglik,
                      probes_from_Z, rademacher_probes)
from .likelihoods import get_likelihood
from .iterative import ProbeSet, Tridiag
from .predict import (
    PredictionBlocks,
    PredictiveDistribution,
    crps_from_samples,
    gaussian_log_score,
    latent_mean,
    latent_var_exact,
    latent_var_lanczos,
    latent_var_sim,
    predict_latent,
    prediction_blocks,
    response_moments,
    rmse,
    scores,
)
from .estimate import FitConfig, FitResult, fit, glm_initial_beta, initial_parameters, profile_xi
