"""Test-only shim: ``moesim.placement`` -> paper_2605_11537_b200.placement."""
from paper_2605_11537_b200.placement import *  # noqa: F401,F403
from paper_2605_11537_b200.placement import LOAD, OFFLOAD, REPLICATE  # noqa: F401
