"""paper_2504_03074_b200 — B200-native WaveHoltz explicit iteration.

Drop-in for the explicit hot path of the reference package ``waveholtz``
(arXiv 2504.03074): the same public names and signatures for the path
(wave_solve_filtered, fpi_solve, krylov_solve, waveholtz_operator, apply_A,
step_explicit and the host objects they take), with every grid-sized
operation executed by hand-written sm_100a CUDA kernels in libwhb200.so
(C ABI: include/whb200.h).  Reference objects are accepted by duck typing,
so ``waveholtz.driver.wave_solve_filtered = paper_2504_03074_b200.wave_solve_filtered``
reroutes the reference's own drivers onto the GPU.

Implicit (trapezoidal) mode runs on the device too: CG with a multigrid or
tridiagonal preconditioner (``implicit.py``).

Extensions beyond the reference: 3D grids, batched frequencies
(``batch.fpi_solve_batched``) and slab decomposition across GPUs
(``slab.SlabFPI``, ``slab.SlabKrylov``).
"""

from .device import DeviceProblem, release_device_cache
from .driver import (
    HelmholtzProblem,
    HostFPIStep,
    NearSingularError,
    WaveHoltzRun,
    apply_A,
    fpi_solve,
    gaussian_source,
    krylov_solve,
    measure_rate,
    multi_gaussian_source,
    resolve_time_discretization,
    waveholtz_operator,
)
from .filters import ExplicitStabilityError, FilterConfig, ResonanceError, TimeMode, alpha_d
from .grid import BC, CartesianGrid, DiscreteOperator, GridField, build_grid, stencil_coefficients
from .implicit import HostImplicitSolver, make_implicit_solver
from .linalg import SolveReport, device_gmres, gmres_solve
from .timestep import (
    TimeCorrection,
    WaveState,
    cfl_constant,
    correct_explicit,
    correct_implicit,
    step_explicit,
    step_implicit,
    time_schedule,
    wave_solve_filtered,
)

__version__ = "0.1.0"
