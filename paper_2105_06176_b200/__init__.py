"""paper_2105_06176_b200 -- B200-native PIPECG, a drop-in for the reference
``pipecg`` package's solve path (/root/reference/pkg/src/pipecg).

    import paper_2105_06176_b200 as pipecg
    x, report = pipecg.pipecg_solve(A, b, x0, pipecg.jacobi_setup(A), cfg)

Layers: ``sparse`` (CsrMatrix + device layout + on-device stencil
generators), ``kernels`` (the reference's operator surface on sm_100a
kernels), ``solvers`` (PIPECG / PCG drivers, report and breakdown types),
``distributed`` (row-block sharding over NCCL, one process per GPU).  All
arithmetic runs in ``_lib/libpipecg_b200.so`` (include/pipecg_b200.h).
"""

import os as _os

# Several solvers of one process whose kernels wait on each other (virtual
# ranks sharing a GPU, ``devices=[0, 0]``) need their streams on distinct
# hardware work queues: with the default 8, two streams can share a queue
# and a rank's kernels then sit behind a peer's kernel that spins on that
# very rank's arrival until the 10 s timeout (measured: 2-4 stalls per 100
# 8-rank solves at 8 connections, 0 in 200 at 32).  Effective only if set
# before the process initialises CUDA.
_os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")

from .sparse import (
    CapacityError,
    CsrMatrix,
    DeviceCsr,
    MatrixMarketError,
    as_device_csr,
    csr_from_dense,
    generate_poisson125,
    generate_powerlaw,
    load_matrix_market,
    parse_matrix_market,
    poisson125_shape,
    stencil_device,
    stencil_host,
    stencil_shape,
)
from .kernels import (
    JacobiPreconditioner,
    dot,
    dots,
    fused_pipecg_update,
    fused_pipecg_update_pc_dots,
    jacobi_apply,
    jacobi_setup,
    norm2,
    residual,
    spmv,
)
from .solvers import (
    DeviceOptions,
    PipecgSolver,
    PipecgState,
    SolveReport,
    SolverBreakdown,
    SolverConfig,
    pcg_solve,
    pipecg_init,
    pipecg_scalars,
    pipecg_solve,
    true_residual_norm,
)

from ._device import invalidate_device_cache

__version__ = "0.1.0"

__all__ = [
    "CapacityError",
    "CsrMatrix",
    "DeviceCsr",
    "as_device_csr",
    "csr_from_dense",
    "generate_poisson125",
    "generate_powerlaw",
    "MatrixMarketError",
    "load_matrix_market",
    "parse_matrix_market",
    "poisson125_shape",
    "stencil_device",
    "stencil_host",
    "stencil_shape",
    "JacobiPreconditioner",
    "dot",
    "dots",
    "fused_pipecg_update",
    "fused_pipecg_update_pc_dots",
    "jacobi_apply",
    "jacobi_setup",
    "norm2",
    "residual",
    "spmv",
    "DeviceOptions",
    "PipecgSolver",
    "PipecgState",
    "SolveReport",
    "SolverBreakdown",
    "SolverConfig",
    "pcg_solve",
    "pipecg_init",
    "pipecg_scalars",
    "pipecg_solve",
    "true_residual_norm",
    "invalidate_device_cache",
]
