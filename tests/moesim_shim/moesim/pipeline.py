"""Test-only shim: ``moesim.pipeline`` -> paper_2605_11537_b200.pipeline."""
from paper_2605_11537_b200.pipeline import *  # noqa: F401,F403
from paper_2605_11537_b200.pipeline import _concurrent_outcomes, _sequential_outcomes  # noqa: F401
