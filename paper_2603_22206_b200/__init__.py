"""chimera-b200: the per-tick scheduling hot path of Chimera (arxiv 2603.22206)
as hand-written sm_100a CUDA kernels behind a C-ABI (include/chimera_b200.h).

Router encoder -> remaining-length predictor -> activity monitor (in-flight
load) -> confidence-gated slack selection -> STJF + aging queues, serial-exact
against the reference scheduler (hetsched, /root/reference/pkg/src/hetsched).
"""

from .config import (  # noqa: F401
    AGING_DISABLED,
    AgingConfig,
    BalancerConfig,
    Decision,
    ModelProfile,
    Pool,
)
from .errors import (  # noqa: F401
    AssignmentConflict,
    DuplicateRequest,
    EmptyTrainingSet,
    SimError,
    UnknownModel,
    UnknownRequest,
    UnknownStage,
    ValidationError,
)

__version__ = "0.1.0"


def load_library():
    """Load libchimera_sm100a.so (raises if it has not been built)."""
    from . import _lib

    return _lib.load()
