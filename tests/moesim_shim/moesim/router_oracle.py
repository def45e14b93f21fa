"""Test-only shim: ``moesim.router_oracle`` -> paper_2605_11537_b200.router_oracle."""
from paper_2605_11537_b200.router_oracle import *  # noqa: F401,F403
from paper_2605_11537_b200.router_oracle import (  # noqa: F401
    LayerPlacement,
    Placement,
    ToyMoeParams,
    load_params,
    random_params,
    save_params,
)
