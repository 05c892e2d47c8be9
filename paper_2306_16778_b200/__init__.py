"""B200-native partial-fraction exp(A)V engine (hot path of arXiv 2306.16778).

Drop-in for the reference package's hot path (`pfexpm.engine._run_tasks`,
/root/reference/pkg/src/pfexpm/engine.py:178-230): same public entry points,
options, results and errors; the n/2 complex-shifted solves and the residue
combine run in hand-written sm_100a kernels behind the C ABI in include/pfx.h.
"""
from .engine import (
    MODE_ACTION,
    MODE_FULL,
    ExpOptions,
    ExpResult,
    apriori_bound,
    matexp_action,
    matexp_action_batched,
    matexp_full,
    matexp_shifted,
)
from .errors import (
    BadSpec,
    ConditionViolated,
    ConvergenceFailure,
    InvariantViolation,
    IterationLimitExceeded,
    OrderOutOfRange,
    OrderTooSmall,
    OrderTooSmallWarning,
    Overflow,
    ParseError,
    PfexpmError,
    PoleHit,
    SingularSystem,
)
from .linalg import (
    BandedHermitian,
    HermitianMatrix,
    SpectralBounds,
    TridiagonalHermitian,
    gershgorin_bounds,
    shifted_inverse,
    shifted_solve,
    solve_residual_bound,
)
from .roots import PoleTable, check_order, default_table
from .scalar import approx_error, exp_trunc

__version__ = "0.1.0"
