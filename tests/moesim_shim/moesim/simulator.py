"""Test-only shim: ``moesim.simulator`` -> paper_2605_11537_b200.simulator."""
from paper_2605_11537_b200.simulator import *  # noqa: F401,F403
from paper_2605_11537_b200.simulator import (  # noqa: F401
    DISTINCT_ONLY,
    ORACLE_PREDICTOR,
    REPLICATED,
    RESIDENT_ALL,
    BatchOutcome,
    BatchRunner,
)
