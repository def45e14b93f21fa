"""Trace / parameter file adapters against files written by the
reference's own writers (tests/golden/io/, made by tests/golden/make_golden.py --only-io):
exact arrays on read, byte-identical files on write, the reference's error cases."""

from pathlib import Path

import numpy as np
import pytest

from paper_2605_11537_b200.errors import TraceParseError, ValidationError
from paper_2605_11537_b200.predictor import load_sru_params, save_sru_params
from paper_2605_11537_b200.router_oracle import load_params, save_params
from paper_2605_11537_b200.workload import read_trace, write_trace

IO = Path(__file__).resolve().parent / "golden" / "io"
REF = np.load(IO / "io.npz")


def test_trace_round_trip(tmp_path):
    tr = read_trace(IO / "trace.txt")
    assert tr.shape.num_layers == 2 and tr.shape.experts_per_layer == 4 and tr.shape.d_model == 8
    assert tr.shape.batch_size == 5 and tr.num_batches == 2 and tr.skew == 1.2 and tr.seed == 3
    emb = np.stack([b.embeddings for b in tr.batches])
    rt = np.stack([b.oracle_routing for b in tr.batches])
    assert emb.dtype == np.float32 and emb.tobytes() == REF["emb"].tobytes()
    assert np.array_equal(rt, REF["routing"])
    write_trace(tr, tmp_path / "t.txt")
    assert (tmp_path / "t.txt").read_bytes() == (IO / "trace.txt").read_bytes()


def test_sru_params_round_trip(tmp_path):
    p = load_sru_params(IO / "sru_params.txt")
    assert p.num_sru_layers == 2 and p.num_moe_layers == 2 and p.num_experts == 4 and p.d_model == 8
    assert np.array_equal(p.heads, REF["heads"])
    for i, lay in enumerate(p.layers):
        for k in ("w", "w_f", "w_r", "b_f", "b_r"):
            assert np.array_equal(getattr(lay, k), REF[f"sru{i}_{k}"]), (i, k)
    save_sru_params(p, tmp_path / "s.txt")
    assert (tmp_path / "s.txt").read_bytes() == (IO / "sru_params.txt").read_bytes()


def test_moe_params_round_trip(tmp_path):
    p = load_params(IO / "moe_params.txt")
    for k, a in (("router", p.router_weights), ("u", p.expert_u), ("v", p.expert_v)):
        assert a.dtype == np.float32 and a.tobytes() == REF[k].tobytes(), k
    save_params(p, tmp_path / "m.txt")
    assert (tmp_path / "m.txt").read_bytes() == (IO / "moe_params.txt").read_bytes()


def _lines(path):
    return (IO / path).read_text().splitlines()


@pytest.mark.parametrize("mutate,exc,line", [
    (lambda ls: [], TraceParseError, 1),                                          # empty file
    (lambda ls: ["moesim-trace v2 layers=2"] + ls[1:], TraceParseError, 1),       # wrong version
    (lambda ls: [ls[0].replace(" seed=3", "")] + ls[1:], TraceParseError, 1),     # missing field
    (lambda ls: [ls[0], ls[2], ls[1]] + ls[3:], TraceParseError, 2),              # out of order
    (lambda ls: ls[:-1], TraceParseError, 11),                                    # truncated
    (lambda ls: ls[:2] + [""] + ls[2:], TraceParseError, 3),                      # blank token line
    (lambda ls: [ls[0], ls[1] + " 0.5"] + ls[2:], TraceParseError, 2),            # field count
    (lambda ls: ls + ["1 5 0 0 " + " ".join(["0"] * 8)], TraceParseError, 12),    # too many lines
    (lambda ls: [ls[0], " ".join(["0", "0", "9"] + ls[1].split()[3:])] + ls[2:], ValidationError, None),
])
def test_trace_errors(tmp_path, mutate, exc, line):
    p = tmp_path / "bad.txt"
    p.write_text("\n".join(mutate(_lines("trace.txt"))) + "\n" if mutate(_lines("trace.txt")) else "")
    with pytest.raises(exc) as info:
        read_trace(p)
    if line is not None:
        assert info.value.line == line


@pytest.mark.parametrize("name,loader", [("sru_params.txt", load_sru_params), ("moe_params.txt", load_params)])
def test_param_file_errors(tmp_path, name, loader):
    ls = _lines(name)
    cases = [
        (["not-a-header"] + ls[1:], 1),
        ([ls[0].split()[0] + " v1 layers=x"] + ls[1:], 1),
        (ls[:5], 6),                       # truncated
        (ls + ["extra 1 2 3"], len(ls) + 1),  # trailing data
        ([ls[0], "zz " + ls[1].split(" ", 1)[1]] + ls[2:], 2),  # wrong row tag
    ]
    for lines, line in cases:
        p = tmp_path / "bad.txt"
        p.write_text("\n".join(lines) + "\n")
        with pytest.raises(TraceParseError) as info:
            loader(p)
        assert info.value.line == line, (lines[:2], info.value)
