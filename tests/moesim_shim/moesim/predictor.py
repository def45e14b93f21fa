"""Test-only shim: ``moesim.predictor`` -> paper_2605_11537_b200.predictor (+ GPU training)."""
from paper_2605_11537_b200.predictor import *  # noqa: F401,F403
from paper_2605_11537_b200.predictor import SruLayerParams, SruParams, load_sru_params, save_sru_params  # noqa: F401
from paper_2605_11537_b200.training import loss_and_grads  # noqa: F401
