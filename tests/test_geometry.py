"""Host geometry mirror (paper_2507_14668_b200.geometry) vs the reference's
known answers and golden vectors. CPU only."""
import math

import numpy as np
import pytest

from paper_2507_14668_b200 import geometry as G


def test_factorize_sweep_matches_reference(golden):
    s = golden("factorize")
    for d, rows, *m in s["rows"]:
        got, _ = G.factorize_dims(int(rows), 4, int(d))
        assert got == [int(v) for v in m[:d]]
    for d, c, *n in s["cols"]:
        if n[0] == -1:
            with pytest.raises(ValueError):
                G.factorize_dims(100, int(c), int(d))
        else:
            assert G.factorize_dims(100, int(c), int(d))[1] == [int(v) for v in n[:d]]


def test_factorize_errors():
    with pytest.raises(ValueError):
        G.factorize_dims(100, 10, 3)
    with pytest.raises(ValueError):
        G.factorize_dims(100, 16, 4)
    with pytest.raises(ValueError):
        G.factorize_dims(0, 16, 3)
    assert sorted(G.factorize_dims(100, 7, 3)[1]) == [1, 1, 7]


def test_shape_validation():
    with pytest.raises(ValueError):
        G.TtShape((2, 2, 2, 2), (1, 1, 1, 1), (1, 1, 1, 1, 1))
    with pytest.raises(ValueError):
        G.TtShape((2, 2), (2, 2), (2, 3, 1))
    with pytest.raises(ValueError):
        G.TtShape((2, 2), (2,), (1, 3, 1))
    s = G.TtShape((10, 10, 10), (2, 2, 4), (1, 8, 8, 1))
    assert s.rows == 1000 and s.cols == 16 and s.core_extent(1) == (8, 20, 8)


def test_digits_roundtrip_and_frozen():
    assert G.linear_index_to_tt_index(5, [2, 3, 2]) == [0, 2, 1]
    assert G.linear_index_to_tt_index(1, [2, 2, 2]) == [0, 0, 1]
    assert G.linear_index_to_tt_index(15, [4, 4]) == [3, 3]
    for m in ([2, 3, 2], [4, 4], [1, 5, 3]):
        for i in range(math.prod(m)):
            assert G.tt_index_to_linear(G.linear_index_to_tt_index(i, m), m) == i
    with pytest.raises(ValueError):
        G.linear_index_to_tt_index(12, [2, 3, 2])


def test_param_counts():
    # test_tt_core.py:223-237 / test_acceptance.py:243-253 known answers
    st = G.param_stats(G.TtShape((128, 128, 128), (4, 4, 4), (1, 32, 32, 1)), 128 ** 3, 64)
    assert st["tt_params"] == 557_056 and st["dense_params"] == 134_217_728
    assert abs(st["ratio"] - 4096 / 17) < 1e-9
    st = G.param_stats(G.TtShape((2, 2, 2), (2, 2, 2), (1, 1, 1, 1)), 8, 8)
    assert st["tt_params"] == 12 and st["dense_params"] == 64
    with pytest.raises(ValueError):
        G.param_stats(G.TtShape((2, 2, 2), (2, 2, 2), (1, 1, 1, 1)), 9, 8)


def test_init_bit_identical(golden):
    s = golden("init")
    for j in range(4):
        rows, dim, seed, d = (int(v) for v in s[f"c{j}.args"])
        shape = G.TtShape(tuple(s[f"c{j}.m"]), tuple(s[f"c{j}.n"]), tuple(s[f"c{j}.r"]))
        assert list(shape.m) == G.factorize_dims(rows, dim, d)[0]
        got = G.init_random_cores(shape, seed, dtype=np.float32)
        for k in range(d):
            assert np.array_equal(got[k], s[f"c{j}.core{k}"])


def test_blob_roundtrip():
    shape = G.TtShape((3, 4, 5), (2, 2, 2), (1, 3, 2, 1))
    cores = G.init_random_cores(shape, 1)
    buf = G.table_to_bytes(shape, cores)
    assert buf.startswith(b"TTEMB1\n")
    s2, c2 = G.bytes_to_table(buf)
    assert s2 == shape and all(np.array_equal(a, b) for a, b in zip(cores, c2))
    with pytest.raises(ValueError):
        G.bytes_to_table(buf + b"x")
    with pytest.raises(ValueError):
        G.bytes_to_table(b"BAD" + buf[3:])
