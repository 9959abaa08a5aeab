"""B200-native Sparse Bessel Decomposition apply path (arXiv 1711.07877).

q_k = sum_l G(z_k - z_l) f_l for 2D point clouds with G = log r (Laplace) or
-(i/4) H0^(1)(k r) (Helmholtz), evaluated as two type-III NUFFTs around a sparse
Bessel-ring spectrum plus a near-field CSR correction -- all on sm_100a kernels
behind the C ABI in include/sbd_b200.h. See DESIGN.md.
"""
from .sbd import (AssembleOptions, OpOptions, CompressedOperator, FrequencyQuadrature, KernelSpec,  # noqa: F401
                  MINUS, NufftOptions, NufftPlan, PLUS, PointCloud, SparsePairMatrix,
                  choose_parameters, cloud_diameter, kernel_helmholtz, kernel_laplace, make_cloud, ndft_direct)
from ._capi import (CudaError, DomainError, SbdConvergenceError, SbdError,  # noqa: F401
                    launch_count)

__version__ = "0.1.0"
