"""CPU-only checks: the C-ABI library loads and exports every symbol the
header declares; host-side logic (validation, snapshot format, model
records, candidate merge) behaves like the reference."""

from __future__ import annotations

import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_library_exports_header_symbols():
    from paper_2509_17360_b200 import _native as N
    header = open(os.path.join(ROOT, "include", "sine_b200.h")).read()
    declared = set(re.findall(r"\b(sine_[a-z_0-9]+)\s*\(", header))
    assert declared, "no declarations parsed"
    lib = N.load_library()
    for name in sorted(declared):
        assert hasattr(lib, name), name
    assert declared == set(N.EXPORTED)
    assert lib.sine_version() == 1


def test_status_mapping():
    from paper_2509_17360_b200 import _native as N
    from paper_2509_17360_b200.errors import ValidationError
    N.check(N.SINE_OK)
    for code in (N.SINE_EINVAL, N.SINE_ENOTFOUND, N.SINE_EDUP, N.SINE_ENORM):
        with pytest.raises(ValidationError):
            N.check(code)
    with pytest.raises(RuntimeError):
        N.check(N.SINE_ECUDA)
    with pytest.raises(MemoryError):
        N.check(N.SINE_ENOMEM)


def test_check_vector_mirrors_reference():
    from paper_2509_17360_b200.errors import ValidationError
    from paper_2509_17360_b200.index import check_matrix, check_vector
    v = np.array([3.0, 4.0]) / 5.0
    assert check_vector(v, 2).tolist() == v.tolist()
    with pytest.raises(ValidationError):
        check_vector([1.0, 1.0], 2)
    with pytest.raises(ValidationError):
        check_vector(v, 3)
    with pytest.raises(ValidationError):
        check_vector(np.ones((2, 2)) / 2, 2)
    # the reference lets NaN through (abs(nan - 1) > tol is False)
    check_vector([float("nan"), 0.0], 2)
    with pytest.raises(ValidationError):
        check_matrix(np.ones((3, 2)), 2)

    class E:
        components = (0.6, 0.8)
    assert check_vector(E(), 2).tolist() == [0.6, 0.8]


def test_snapshot_parser_matches_reference_format():
    from paper_2509_17360_b200.errors import ValidationError
    from paper_2509_17360_b200.index import parse_snapshot_lines
    lines = ["exact-cosine-index", "dimension: 2", "seed: 4", "count: 2",
             f"7 {0.6.hex()} {0.8.hex()}", f"3 {1.0.hex()} {0.0.hex()}"]
    d, s, e = parse_snapshot_lines(lines, "exact-cosine-index")
    assert (d, s) == (2, 4) and [i for i, _ in e] == [7, 3] and e[0][1].tolist() == [0.6, 0.8]
    with pytest.raises(ValidationError):
        parse_snapshot_lines(lines, "small-world-index")
    with pytest.raises(ValidationError):
        parse_snapshot_lines(lines[:5], "exact-cosine-index")
    with pytest.raises(ValidationError):
        parse_snapshot_lines(["exact-cosine-index", "dimension: x"], "exact-cosine-index")


def test_model_records_round_trip_and_validation():
    from paper_2509_17360_b200 import model as M
    from paper_2509_17360_b200.errors import ValidationError
    el = M.make_element(M.SemanticKey("q\ttext", "search"), "a b\nc", M.EmbeddingVector((0.6, 0.8)),
                        7, 400.0, 0.005, 1.5, 10.0, frequency=2)
    assert el.size_tokens == 3 and el.expiration_time == 11.5
    back = M.deserialize_element(M.serialize_element(el))
    assert back == el
    for bad in (dict(staticity=0), dict(staticity=11), dict(ttl_seconds=0.0), dict(frequency=-1)):
        kw = dict(staticity=5, ttl_seconds=1.0, frequency=0)
        kw.update(bad)
        with pytest.raises(ValidationError):
            M.make_element(M.SemanticKey("q", "t"), "v", M.EmbeddingVector((1.0,)), kw["staticity"], 1.0, 1.0,
                           0.0, kw["ttl_seconds"], frequency=kw["frequency"])
    with pytest.raises(ValidationError):
        M.CacheConfig(capacity_tokens=0)
    with pytest.raises(ValidationError):
        M.CacheConfig(capacity_tokens=1, eviction_policy="fifo")
    with pytest.raises(ValidationError):
        M.token_count("   ")


def test_cal_score_matches_oracle_bits(evict_golden):
    from paper_2509_17360_b200 import model as M
    from paper_2509_17360_b200.engine import cal_score
    for f, c, lat, s, size, want in evict_golden["cal_score_grid"]:
        el = M.SemanticElement(M.SemanticKey("a", "b"), "v", M.EmbeddingVector((1.0,)), s, f,
                               float.fromhex(lat), float.fromhex(c), size, 0.0, 100.0)
        assert cal_score(el, 5.0) == float.fromhex(want)
    assert float.fromhex(evict_golden["cal_score_frozen"]) == 0.05063404135640259


def test_merge_topk_orders_like_reference():
    import torch
    from paper_2509_17360_b200.sharded import merge_topk
    sims = torch.tensor([[[0.9, 0.5, 0.0]], [[0.9, 0.7, 0.1]]], dtype=torch.float64)
    ids = torch.tensor([[[8, 2, -1]], [[3, 4, 9]]])
    i, s, c = merge_topk(sims, ids, 4)
    assert i.tolist() == [[3, 8, 4, 2]] and c.tolist() == [4]
    i, s, c = merge_topk(sims[:, :, :1] * 0 - 1, ids[:, :, :1] * 0 - 1, 2)
    assert i.tolist() == [[-1, -1]] and c.tolist() == [0]
