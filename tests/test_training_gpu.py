"""GPU SRU predictor training against the reference's own
loss/gradients and training run (tests/golden/train.npz, made by make_golden.py),
plus the reference's training tests (pkg/tests/test_predictor.py TestTraining)."""

from pathlib import Path

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

from oracle import moesim_oracle as O  # noqa: E402
from paper_2605_11537_b200.errors import TrainingError  # noqa: E402
from paper_2605_11537_b200.predictor import evaluate_accuracy, init_params, predict_batch  # noqa: E402
from paper_2605_11537_b200.training import loss_and_grads, train_predictor  # noqa: E402
from paper_2605_11537_b200.workload import Batch, ModelShape, RoutingTrace  # noqa: E402

Z = np.load(Path(__file__).resolve().parent / "golden" / "train.npz")
NAMES = ("w", "w_f", "w_r", "b_f", "b_r")


def _rel(a, b):
    return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-300))


@pytest.mark.parametrize("k", [0, 1, 2])
def test_loss_and_grads_match_reference(k):
    S, T, d, L, E, nl, seed = (int(v) for v in Z[f"g{k}_meta"])
    p = init_params(L, E, d, num_sru_layers=nl, seed=seed)
    loss, g = loss_and_grads(p, Z[f"g{k}_x"], Z[f"g{k}_y"])
    assert abs(loss - float(Z[f"g{k}_loss"])) <= 1e-12 * abs(float(Z[f"g{k}_loss"]))
    assert _rel(g.heads, Z[f"g{k}_heads"]) <= 1e-10
    for i, lay in enumerate(g.layers):
        for n in NAMES:
            assert _rel(getattr(lay, n), Z[f"g{k}_{i}_{n}"]) <= 1e-10, (k, i, n)


def _golden_trace():
    shape = ModelShape(num_layers=2, experts_per_layer=4, d_model=16, batch_size=32)
    return RoutingTrace(shape, [Batch(b, Z["t_emb"][b], Z["t_lab"][b]) for b in range(Z["t_emb"].shape[0])])


def test_training_run_matches_reference():
    res = train_predictor(_golden_trace(), epochs=4, learning_rate=0.01, seed=3, num_sru_layers=2,
                          sequences_per_step=5)
    assert np.allclose(res.loss_curve, Z["t_curve"], rtol=1e-10, atol=0)
    assert _rel(res.params.heads, Z["t_heads"]) <= 1e-9
    for i, lay in enumerate(res.params.layers):
        for n in NAMES:
            assert _rel(getattr(lay, n), Z[f"t_{i}_{n}"]) <= 1e-9, (i, n)


def test_zero_epochs_returns_seeded_init():
    tr = _golden_trace()
    res = train_predictor(tr, epochs=0, seed=11, num_sru_layers=2)
    ref = init_params(2, 4, 16, num_sru_layers=2, seed=11)
    assert res.loss_curve == []
    assert np.array_equal(res.params.heads, ref.heads)
    assert np.array_equal(res.params.layers[1].w, ref.layers[1].w)


def test_divergence_raises_with_epoch():
    with pytest.raises(TrainingError) as info:
        train_predictor(_golden_trace(), epochs=20, learning_rate=1e200, seed=0, num_sru_layers=2)
    assert info.value.epoch is not None


def test_deterministic_and_loss_decreases():
    a = train_predictor(_golden_trace(), epochs=6, seed=5, num_sru_layers=2, learning_rate=0.01)
    b = train_predictor(_golden_trace(), epochs=6, seed=5, num_sru_layers=2, learning_rate=0.01)
    assert a.loss_curve == b.loss_curve
    assert np.array_equal(a.params.heads, b.params.heads)
    assert a.loss_curve[-1] < a.loss_curve[0]


def test_degenerate_skew_reaches_high_accuracy():
    """pkg/tests/test_predictor.py: skew 10, 32 training batches, 80 epochs -> >= 0.99 held-out."""
    shape = ModelShape(num_layers=2, experts_per_layer=4, d_model=16, batch_size=32)
    batches = O.generate_trace(2, 4, 16, 32, 40, 10.0, seed=2)
    bs = [Batch(i, emb, rt) for i, (emb, rt) in enumerate(batches)]
    res = train_predictor(RoutingTrace(shape, bs[:32]), epochs=80, learning_rate=0.001, seed=0, num_sru_layers=2)
    scores = [evaluate_accuracy(predict_batch(b, res.params), b.oracle_routing) for b in bs[32:]]
    assert float(np.mean(scores)) >= 0.99


@pytest.mark.parametrize("ta,tb", [(0, 0), (0, 1), (1, 0), (1, 1)])
def test_dgemm_matches_float64_reference(ta, tb):
    """mp_dgemm (the trainer's float64 products) vs a float64 matmul, ragged sizes, accumulate."""
    import torch

    from paper_2605_11537_b200.training import _mm

    g = torch.Generator().manual_seed(7 + 2 * ta + tb)
    for M, N, K in ((1, 1, 1), (70, 33, 129), (128, 64, 512), (5, 200, 3), (300, 17, 0)):
        a = torch.randn((K, M) if ta else (M, K), generator=g, dtype=torch.float64)
        b = torch.randn((N, K) if tb else (K, N), generator=g, dtype=torch.float64)
        ref = (a.T if ta else a) @ (b.T if tb else b)
        got = _mm(a.cuda(), b.cuda(), ta=bool(ta), tb=bool(tb)).cpu()
        assert torch.allclose(got, ref, rtol=1e-12, atol=1e-12 * max(1, K))
        c0 = torch.randn(M, N, generator=g, dtype=torch.float64)
        out = c0.cuda()
        _mm(a.cuda(), b.cuda(), ta=bool(ta), tb=bool(tb), out=out, accumulate=True)
        assert torch.allclose(out.cpu(), ref + c0, rtol=1e-12, atol=1e-12 * max(1, K))
