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


def _special_values():
    import math
    import struct
    vals = [0.0, -0.0, 1.0, -1.0, 0.5, 5e-324, -5e-324, 2.2250738585072014e-308, 2.225073858507201e-308,
            1.7976931348623157e308, -1.7976931348623157e308, math.inf, -math.inf, math.nan, 1e-300, 123456.789,
            0.1, 1 / 3, 2.0 ** 1023, 2.0 ** -1022, 2.0 ** -1074]
    vals.append(struct.unpack("<d", struct.pack("<Q", 0x7ff8000000000001 | (1 << 63)))[0])  # -nan
    return vals


def test_native_hex_matches_python_float_hex():
    """sine_hex_format is byte-identical to " ".join(float(c).hex() ...)
    (reference index.py:343-346, model.py:237), including zeros, signed
    zero, subnormals, extremes, inf and nan; ids print like str(int)."""
    from paper_2509_17360_b200 import _native as N
    rng = np.random.default_rng(0)
    rows = np.concatenate([rng.standard_normal((50, 7)) * 10.0 ** rng.integers(-300, 300, (50, 7)),
                           np.array(_special_values()[:21]).reshape(3, 7)])
    ids = rng.integers(-2 ** 62, 2 ** 62, rows.shape[0])
    ids[0], ids[1] = 0, -1
    want = "".join(f"{i} " + " ".join(float(c).hex() for c in r) + "\n" for i, r in zip(ids.tolist(), rows))
    assert bytes(N.hex_format(rows, ids)).decode() == want
    want_noid = "".join(" ".join(float(c).hex() for c in r) + "\n" for r in rows)
    assert bytes(N.hex_format(rows)).decode() == want_noid
    assert bytes(N.hex_format(np.array([[_special_values()[-1]]]))).decode() == "nan\n"


def test_native_hex_parse_round_trip_and_errors():
    from paper_2509_17360_b200 import _native as N
    from paper_2509_17360_b200.errors import ValidationError
    rng = np.random.default_rng(1)
    rows = rng.standard_normal((600, 33))
    rows[0, :5] = [0.0, -0.0, 5e-324, np.inf, -np.inf]
    ids = rng.permutation(10 ** 6)[:600]
    gi, gr = N.hex_parse(bytes(N.hex_format(rows, ids)), 600, 33, True)
    assert gi.tolist() == ids.tolist()
    assert gr.tobytes() == rows.tobytes()  # bit-exact, signed zero included
    # non-canonical spellings float.fromhex accepts
    _, r = N.hex_parse(b"0x1p-3 0X1.8P+1 -0x0.0p+0 inf\n", 1, 4, False)
    assert r[0].tolist() == [float.fromhex("0x1p-3"), 3.0, -0.0, np.inf]
    assert np.signbit(r[0, 2])
    for bad in (b"1 0x1.0p+0 zz\n", b"1 0x1.0p+0\n", b"1 0x1.0p+0 0x1.0p+0 0x1.0p+0\n", b"x 0x1.0p+0 0x1.0p+0\n",
                b"1 0x1.0p+0  0x1.0p+0\n"):
        with pytest.raises(ValidationError):
            N.hex_parse(bad, 1, 2, True)
    with pytest.raises(ValidationError):  # fewer lines than the count
        N.hex_parse(b"1 0x1.0p+0 0x1.0p+0\n", 2, 2, True)


def test_snapshot_bytes_parse_matches_reference_reader():
    """parse_snapshot_bytes reads the reference's own snapshot text (built
    here with the reference format's float.hex lines) bit-exactly."""
    from paper_2509_17360_b200.index import parse_snapshot_bytes, parse_snapshot_lines
    rng = np.random.default_rng(2)
    rows = rng.standard_normal((40, 6))
    lines = ["exact-cosine-index", "dimension: 6", "seed: 3", "count: 40"]
    lines += [f"{i * 7} " + " ".join(float(c).hex() for c in r) for i, r in enumerate(rows)]
    text = "\n".join(lines) + "\n"
    d, s, ids, got = parse_snapshot_bytes(text.encode(), "exact-cosine-index")
    d2, s2, entries = parse_snapshot_lines(text.splitlines(), "exact-cosine-index")
    assert (d, s) == (d2, s2) == (6, 3)
    assert ids.tolist() == [e[0] for e in entries]
    assert got.tobytes() == np.stack([e[1] for e in entries]).tobytes()


def test_blake2b64_matches_hashlib_goldens():
    """The device BLAKE2b (RFC 7693, keyed, 8-byte digest) that buckets the
    embedder's tokens equals hashlib on the reference's golden digests and
    on fresh random messages."""
    import hashlib
    import json
    from paper_2509_17360_b200 import _native as N
    lib = N.load_library()
    gold = json.load(open(os.path.join(ROOT, "tests", "golden", "embed_golden.json"), encoding="utf-8"))
    for g in gold["blake2b"]:
        m = bytes.fromhex(g["msg"])
        assert lib.sine_blake2b64(m, len(m), g["key"]) == g["digest"]
    rng = np.random.default_rng(9)
    for n in list(range(0, 260, 7)) + [1000]:
        m = rng.integers(0, 256, n, dtype=np.uint8).tobytes()
        key = int(rng.integers(0, 2 ** 63))
        want = int.from_bytes(hashlib.blake2b(m, key=key.to_bytes(8, "little"), digest_size=8).digest(), "little")
        assert lib.sine_blake2b64(m, len(m), key) == want


def test_embedder_tokenize_matches_reference_rules():
    from paper_2509_17360_b200.embedder import tokenize
    assert tokenize("Hello, World! héllo  WORLD...x") == ["hello", "world", "héllo", "world", "x"]
    assert tokenize("...!!!") == []


def test_vectorised_placement_equals_the_sequential_greedy_rule():
    """sharded.place_least_full == one-row-at-a-time argmin placement
    (least-full rank, lowest rank on ties), for ragged starting counts."""
    from paper_2509_17360_b200.sharded import place_least_full

    def greedy(c, n):
        c, out = list(c), []
        for _ in range(n):
            r = int(np.argmin(c))
            out.append(r)
            c[r] += 1
        return out

    rng = np.random.default_rng(0)
    for _ in range(500):
        P = int(rng.integers(1, 9))
        c = rng.integers(0, 7, P)
        n = int(rng.integers(0, 50))
        assert place_least_full(c, n).tolist() == greedy(c, n)
    assert place_least_full(np.zeros(8, dtype=np.int64), 10_000_000).shape == (10_000_000,)
