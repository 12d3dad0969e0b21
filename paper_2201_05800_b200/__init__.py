"""B200-native (sm_100a) space-time DG-SEM slab operator.

Drop-in for the hot path of the reference ``stdgsem`` library: the slab
residual R(U), the matrix-free Jacobian action J.v, the Krylov (GMRES) vector
kernels and the Lobatto IIIC stage-system apply, as hand-written fp64 CUDA
kernels behind a C ABI (include/stg_cuda.h).  See DESIGN.md.
"""
from .api import (  # noqa: F401
    CudaError, DgSpace, FluxModel, JacobianForm, LinearMethod, Mesh, NewtonConfig,
    NonconvergenceError, SemiDiscreteSystem, SlabOperator, TimeElementSystem, advection_model,
    assemble_semidiscrete, burgers_model, dg_space, integrate, lobatto_tableau, rk_step,
    sbp_operators, st_jacobian, st_residual, stdg_integrate, stdg_step, uniform_mesh,
)
from ._lib import (  # noqa: F401
    STG_FORM_A, STG_FORM_A_INV, STG_KERNEL_AUTO, STG_KERNEL_FAST, STG_KERNEL_GENERIC,
    STG_MODEL_ADVECTION, STG_MODEL_BURGERS,
)
