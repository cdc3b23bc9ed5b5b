"""Index reordering (reference reorder.py): the oracle and the host-side
helpers against the reference's frozen vectors and tests/golden/reorder.npz
(CPU), and the GPU passes (ttb_count_frequencies / ttb_rank_rows /
ttb_apply_bijection) against both (marked gpu)."""
import numpy as np
import pytest
import torch

from oracle import ttb_oracle as O


def golden_batches(s):
    idx, off = s["idx"], s["off"]
    return [idx[off[i]:off[i + 1]].tolist() for i in range(off.size - 1)]


def test_oracle_frozen_vectors():
    counts, ror, rank = O.count_frequencies([[0, 2, 2], [2, 1]], 4)
    assert counts.tolist() == [1, 1, 3, 0]
    assert ror.tolist() == [2, 0, 1, 3]
    assert rank.tolist() == [1, 2, 0, 3]
    with pytest.raises(ValueError):
        O.count_frequencies([[4]], 4)
    assert O.apply_bijection([2, 0, 1], [[0, 1], [2, 2, 0]]) == [[2, 0], [1, 1, 2]]
    with pytest.raises(ValueError):
        O.apply_bijection([2, 0, 1], [[3]])
    # reorder tests: frozen community layout
    c = np.array([10, 9, 1, 5, 2, 4, 1, 3])
    ror = np.array(sorted(range(8), key=lambda r: (-c[r], r)))
    rank = np.empty(8, dtype=np.int64)
    rank[ror] = np.arange(8)
    fwd = O.build_bijection(np.array([0, 1, 2, 1, 0, 2]), {0, 1}, c, rank, 8)
    assert fwd.tolist() == [0, 1, 3, 2, 5, 4, 7, 6]


def test_oracle_matches_reference_golden(golden):
    s = golden("reorder")
    n = int(s["table_len"][0])
    batches = golden_batches(s)
    counts, ror, rank = O.count_frequencies(batches, n)
    assert np.array_equal(counts, s["counts"]) and np.array_equal(ror, s["row_of_rank"])
    assert np.array_equal(rank, s["rank_of"])
    fwd = O.build_bijection(s["community_of"], set(s["hot"].tolist()), counts, rank, n)
    assert np.array_equal(fwd, s["forward"])
    rel = O.apply_bijection(fwd, batches)
    assert np.array_equal(np.concatenate([np.asarray(b) for b in rel]), s["relabeled"])


def _freq_cpu(counts):
    from paper_2507_14668_b200.reorder import FreqOrder
    counts = np.asarray(counts, dtype=np.int64)
    n = counts.size
    ror = np.lexsort((np.arange(n), -counts))
    rank = np.empty(n, dtype=np.int64)
    rank[ror] = np.arange(n)
    return FreqOrder(torch.from_numpy(counts), torch.from_numpy(rank), torch.from_numpy(ror))


def test_host_build_bijection_matches_reference(golden):
    from paper_2507_14668_b200 import reorder as R
    s = golden("reorder")
    n = int(s["table_len"][0])
    freq = _freq_cpu(s["counts"])
    hot = R.hot_row_set(freq, 0.02)
    assert hot == set(s["hot"].tolist())
    bij = R.build_bijection(s["community_of"], hot, freq, n)
    assert np.array_equal(bij.forward, s["forward"]) and np.array_equal(bij.inverse, s["inverse"])
    # the reference's frozen layouts
    f = _freq_cpu([10, 9, 1, 5, 2, 4, 1, 3])
    assert R.hot_row_set(f, 0.25) == {0, 1}
    assert R.build_bijection(np.array([0, 1, 2, 1, 0, 2]), {0, 1}, f, 8).forward.tolist() == \
        [0, 1, 3, 2, 5, 4, 7, 6]
    f = _freq_cpu([1, 9, 2, 10])
    assert R.build_bijection(np.array([0, 1]), R.hot_row_set(f, 0.5), f, 4).forward.tolist() == [2, 1, 0, 3]
    f = _freq_cpu([5, 4, 3, 2])
    assert R.build_bijection(np.array([], dtype=np.int64), R.hot_row_set(f, 1.0), f, 4).forward.tolist() == \
        [0, 1, 2, 3]
    with pytest.raises(ValueError):
        R.hot_row_set(f, 1.5)


def test_bijection_text_format(tmp_path):
    from paper_2507_14668_b200 import reorder as R
    bij = R.IndexBijection(np.array([2, 0, 1, 3]), np.array([1, 2, 0, 3]))
    path = tmp_path / "map.txt"
    R.save_bijection(bij, path)
    assert path.read_text() == "0 2\n1 0\n2 1\n3 3\n"
    back = R.load_bijection(path)
    assert (back.forward == bij.forward).all() and (back.inverse == bij.inverse).all()
    path.write_text("0 1\n1 1\n")
    with pytest.raises(ValueError):
        R.load_bijection(path)
    path.write_text("0 0\n2 1\n")
    with pytest.raises(ValueError):
        R.load_bijection(path)
    with pytest.raises(ValueError):
        R.IndexBijection(np.array([0, 0]), np.array([0, 1]))


# ----------------------------------------------------------------- GPU
@pytest.mark.gpu
def test_gpu_count_and_rank_golden(golden):
    from paper_2507_14668_b200 import reorder as R
    s = golden("reorder")
    n = int(s["table_len"][0])
    batches = golden_batches(s)
    for src in (batches, torch.from_numpy(s["idx"]).cuda()):
        freq = R.count_frequencies(src, n)
        assert np.array_equal(freq.counts.cpu().numpy(), s["counts"])
        assert np.array_equal(freq.row_of_rank.cpu().numpy(), s["row_of_rank"])
        assert np.array_equal(freq.rank_of.cpu().numpy(), s["rank_of"])
    freq = R.count_frequencies([[0, 2, 2], [2, 1]], 4)
    assert freq.row_of_rank.cpu().tolist() == [2, 0, 1, 3]
    assert freq.rank_of.cpu().tolist() == [1, 2, 0, 3]
    with pytest.raises(ValueError):
        R.count_frequencies([[4]], 4)
    with pytest.raises(ValueError):
        R.count_frequencies([[-1]], 4)
    hot = R.hot_row_set(freq, 0.5)
    assert hot == {2, 0}
    bij = R.build_bijection(s["community_of"], set(s["hot"].tolist()), R.count_frequencies(batches, n), n)
    assert np.array_equal(bij.forward, s["forward"])


@pytest.mark.gpu
def test_gpu_rank_large_skewed():
    """10M-row table, 4M Zipf-ish indices: counts and the (count desc, id asc)
    order bit-exact against numpy."""
    from paper_2507_14668_b200 import reorder as R
    n = 10_000_000
    rng = np.random.default_rng(7)
    idx = np.minimum((rng.pareto(1.1, size=4_000_000) * 50).astype(np.int64), n - 1)
    idx = np.concatenate([idx, rng.integers(0, n, size=1_000_000)])
    freq = R.count_frequencies(torch.from_numpy(idx).cuda(), n)
    counts = np.bincount(idx, minlength=n)
    assert np.array_equal(freq.counts.cpu().numpy(), counts)
    ror = np.lexsort((np.arange(n), -counts))
    assert np.array_equal(freq.row_of_rank.cpu().numpy(), ror)
    rank = freq.rank_of.cpu().numpy()
    assert np.array_equal(rank[ror], np.arange(n))


@pytest.mark.gpu
def test_gpu_apply_bijection(golden):
    from paper_2507_14668_b200 import reorder as R
    s = golden("reorder")
    bij = R.IndexBijection(s["forward"], s["inverse"])
    batches = golden_batches(s)
    out = R.apply_bijection(bij, batches)
    assert [len(b) for b in out] == [len(b) for b in batches]
    assert np.array_equal(np.concatenate([np.asarray(b) for b in out]), s["relabeled"])
    dev = R.DeviceBijection(bij)
    t = dev.relabel(torch.from_numpy(s["idx"]).cuda())
    assert np.array_equal(t.cpu().numpy(), s["relabeled"])
    # inverse relabel restores the trace
    inv = R.DeviceBijection(R.IndexBijection(s["inverse"], s["forward"]))
    assert np.array_equal(inv.relabel(t).cpu().numpy(), s["idx"])
    small = R.IndexBijection(np.array([2, 0, 1]), np.array([1, 2, 0]))
    assert R.apply_bijection(small, [[0, 1], [2, 2, 0]]) == [[2, 0], [1, 1, 2]]
    with pytest.raises(ValueError):
        R.apply_bijection(small, [[3]])
    assert R.mean_distinct_prefixes(batches, 8) == pytest.approx(float(s["mdp_before"][0]))
    assert R.mean_distinct_prefixes(out, 8) == pytest.approx(float(s["mdp_after"][0]))
