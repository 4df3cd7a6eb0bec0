"""B200-native SCS indirect-method hot path (arXiv 1312.3039).

Drop-in for the indirect (conjugate-gradient) path of the reference package
``conesplit`` 0.1.0: same ``solve`` / ``Workspace`` surface and the same
``Solution`` / ``Status`` / ``solution_to_dict`` results, with the whole
iteration loop running as hand-written sm_100a CUDA kernels behind the
C-ABI of ``include/scs_b200.h``.
"""

from .api import (  # noqa: F401
    ConeSpec,
    ProblemData,
    Residuals,
    ScalingData,
    SetupError,
    Settings,
    Solution,
    SolveInfo,
    SolverState,
    SparseMatrix,
    Status,
    Workspace,
    packed_length,
    solution_to_dict,
    solve,
    validate_problem,
)

from .problem_io import (  # noqa: F401
    FileFormatError,
    read_problem,
    write_problem,
)

from .native import pinned_empty, pinned_zeros  # noqa: F401,E402

__version__ = "0.1.0"
