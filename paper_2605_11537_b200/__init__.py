"""B200-native (sm_100a) MoE-MPMC inference hot path, drop-in for the
``moesim`` predictor / replica-planner / MoE-forward API of arXiv 2605.11537.
"""

from .errors import (  # noqa: F401
    ConfigurationError,
    DeviceError,
    InfeasibleCapacityError,
    MoesimError,
    NumericError,
    PlacementError,
    TraceParseError,
    TrainingError,
    ValidationError,
)

__version__ = "0.1.0"
