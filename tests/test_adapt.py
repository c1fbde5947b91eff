"""ADAPT C-API packer (SampleRecord -> dense) against a plain Python restatement (CPU)."""

import numpy as np
import pytest

from paper_1905_13746_b200 import _adapt
from paper_1905_13746_b200.model import Label, OpcodeHistogram, SampleRecord


def _samples(rng, n):
    ops = [f"op{i}" for i in range(30)]
    out = []
    for i in range(n):
        h = {ops[j]: int(rng.integers(1, 1000)) for j in rng.choice(30, int(rng.integers(0, 12)),
                                                                     replace=False)}
        lab = (Label.MALWARE, Label.BENIGN, Label.UNKNOWN)[i % 3]
        out.append(SampleRecord(f"s{i}", lab, int(rng.integers(-10, 60000)),
                                OpcodeHistogram.from_counts(h)))
    return out


def test_densify_and_meta():
    rng = np.random.default_rng(0)
    s = _samples(rng, 500)
    cols = {f"op{i}": i // 2 for i in range(0, 30, 2)}   # every other opcode, packed
    x = np.zeros((500, 15), np.int32)
    _adapt.densify_into(s, cols, x, 15)
    want = np.zeros_like(x)
    for i, r in enumerate(s):
        for op, n in r.histogram.entries.items():
            if op in cols:
                want[i, cols[op]] = n
    assert np.array_equal(x, want)
    size = np.empty(500, np.int32)
    lab = np.empty(500, np.int32)
    _adapt.meta_into(s, 50000, Label.MALWARE, Label.BENIGN, size, lab)
    assert size.tolist() == [r.size_bytes if 0 <= r.size_bytes < 50000 else -1 for r in s]
    assert lab.tolist() == [{Label.MALWARE: 1, Label.BENIGN: 0}.get(r.label, -1) for r in s]


def test_gather_routes_per_sample():
    rng = np.random.default_rng(1)
    s = _samples(rng, 300)
    route = np.array([0, 1, 1, 0, 1, 0], np.int32)          # 6 groups of 10000 bytes
    colmaps = [{"op1": 0, "op2": 1, "op3": 2}, {"op29": 0, "op1": 2}]
    x = np.zeros((300, 3), np.int32)
    size = np.empty(300, np.int32)
    _adapt.gather_into(s, route, colmaps, 3, 10000, 60000, x, size)
    for i, r in enumerate(s):
        if not 0 <= r.size_bytes < 60000:
            assert size[i] == -1 and not x[i].any()
            continue
        assert size[i] == r.size_bytes // 10000         # the size group id
        cm = colmaps[route[r.size_bytes // 10000]]
        want = np.zeros(3, np.int32)
        for op, n in r.histogram.entries.items():
            if op in cm:
                want[cm[op]] = n
        assert np.array_equal(x[i], want)


def test_counts_beyond_int32_rejected():
    s = [SampleRecord("a", Label.MALWARE, 1, OpcodeHistogram({"op": 2**31}))]
    with pytest.raises(OverflowError):
        _adapt.densify_into(s, {"op": 0}, np.zeros((1, 1), np.int32), 1)


def test_gather_walks_either_dict():
    """gather_into gives the same rows whether it walks the model's features
    (k < nnz) or the histogram entries (k >= nnz)."""
    rng = np.random.default_rng(3)
    s = _samples(rng, 400)
    route = np.array([0, 1], np.int32)
    small = [{"op1": 0, "op5": 1}, {"op2": 1, "op7": 0}]                 # k=2 < most nnz
    large = [{f"op{i}": (i * 7) % 30 for i in range(30)}, {f"op{i}": 29 - i for i in range(30)}]
    for maps, width in ((small, 2), (large, 30)):
        x = np.zeros((400, width), np.int32)
        sz = np.zeros(400, np.int32)
        _adapt.gather_into(s, route, maps, width, 30000, 60000, x, sz)
        for i, r in enumerate(s):
            if not 0 <= r.size_bytes < 60000:
                assert sz[i] == -1 and not x[i].any()
                continue
            want = np.zeros(width, np.int32)
            for op, j in maps[r.size_bytes // 30000].items():
                want[j] = r.histogram.entries.get(op, 0)
            assert sz[i] == r.size_bytes // 30000 and np.array_equal(x[i], want)


def test_predictions_match_python_construction():
    import gc
    from paper_1905_13746_b200.model import INDEX_CLASS, Prediction
    rng = np.random.default_rng(4)
    n = 1000
    lab = rng.integers(-2, 2, size=n).astype(np.int32)
    lp = rng.standard_normal((n, 2))
    eff = rng.integers(0, 100, size=n).astype(np.int32)
    got = _adapt.predictions(lab, lp, eff, Prediction, INDEX_CLASS, Label.MALWARE, Label.BENIGN)
    want = [None if lab[i] < 0 else Prediction(
        INDEX_CLASS[lab[i]], {Label.MALWARE: float(lp[i, 1]), Label.BENIGN: float(lp[i, 0])},
        int(eff[i])) for i in range(n)]
    assert got == want
    assert gc.isenabled()
    p = next(x for x in got if x is not None)
    with pytest.raises(Exception):
        p.label = Label.BENIGN        # still a frozen dataclass instance


@pytest.mark.parametrize("n_ops", [30, 700])   # 700 > the first 512-column guess: retry
def test_dense_vocab_matches_sorted_union(n_ops):
    from paper_1905_13746_b200.api import _dense_vocab
    rng = np.random.default_rng(n_ops)
    ops = [f"m{rng.integers(0, 10**6)}_{i}" for i in range(n_ops)]
    samples = []
    for i in range(300):
        pick = rng.choice(n_ops, int(rng.integers(0, min(40, n_ops))), replace=False)
        samples.append(SampleRecord(f"s{i}", Label.BENIGN, 10, OpcodeHistogram.from_counts(
            {ops[j]: int(rng.integers(1, 50)) for j in pick})))
    x, vocab = _dense_vocab(samples)
    want_vocab = sorted({op for s in samples for op in s.histogram.entries})
    assert vocab == want_vocab
    want = np.zeros((300, max(len(vocab), 1)), np.int32)
    col = {op: j for j, op in enumerate(vocab)}
    for i, s in enumerate(samples):
        for op, c in s.histogram.entries.items():
            want[i, col[op]] = c
    assert np.array_equal(x, want)


@pytest.mark.parametrize("case", ["plain", "nonstr_key", "big_count", "bad_route", "copied_keys"])
def test_parallel_gather_matches_serial(case):
    """gather_into (threaded dict walk for >= 8192 samples) == the serial walk,
    and every unusual input falls back to the serial path with its errors."""
    rng = np.random.default_rng(7)
    s = _samples(rng, 20_000)
    route = np.array([0, 1, 1, 0, 1, 0], np.int32)
    colmaps = [{"op1": 0, "op2": 1, "op3": 2, "op17": 3}, {"op29": 0, "op1": 2, "op5": 1}]
    if case == "copied_keys":      # equal but not identical str keys in the column maps
        colmaps = [{("op" + str(int(k[2:])))[:]: v for k, v in cm.items()} for cm in colmaps]
    if case == "nonstr_key":
        s[12345].histogram.entries[7] = 3
    if case == "big_count":
        s[15000] = SampleRecord("big", Label.MALWARE, 100,
                                OpcodeHistogram.from_counts({"op1": 2**40}))
    if case == "bad_route":
        route = np.array([0, 1, 5, 0, 1, 0], np.int32)
    outs = []
    for fn in (_adapt.gather_into, _adapt.gather_into_serial):
        x = np.zeros((len(s), 4), np.int32)
        size = np.empty(len(s), np.int32)
        try:
            fn(s, route, colmaps, 4, 10000, 60000, x, size)
            outs.append((x, size))
        except Exception as e:  # noqa: BLE001
            outs.append(type(e))
    if case in ("big_count", "bad_route"):
        assert outs[0] == outs[1] and isinstance(outs[0], type)
    else:
        assert np.array_equal(outs[0][0], outs[1][0]) and np.array_equal(outs[0][1], outs[1][1])
        assert outs[0][0].any()


@pytest.mark.parametrize("case", ["plain", "nonstr_key", "big_count", "unicode"])
def test_vocab_dense_matches_serial(case, monkeypatch):
    """The threaded vocabulary walk (vocab_dense) == the serial discover_into +
    permute path: same sorted opcodes, same matrix; unusual inputs -> None and
    the serial path (with its errors)."""
    from paper_1905_13746_b200 import api
    rng = np.random.default_rng(3)
    s = _samples(rng, 12_000)
    if case == "unicode":
        s[77] = SampleRecord("u", Label.MALWARE, 5, OpcodeHistogram.from_counts(
            {"mové": 4, "\U0001f600op": 2, "op1": 1}))
    if case == "nonstr_key":
        s[9000].histogram.entries[7] = 3
    if case == "big_count":
        s[11000] = SampleRecord("big", Label.MALWARE, 100,
                                OpcodeHistogram.from_counts({"op1": 2**40}))
    fast = _adapt.vocab_dense(s)
    if case in ("nonstr_key", "big_count"):
        assert fast is None
        return
    assert fast is not None
    x_fast, v_fast = api._dense_vocab(s)
    monkeypatch.setattr(api._adapt, "vocab_dense", lambda samples: None)
    x_ser, v_ser = api._dense_vocab(s)
    assert v_fast == v_ser == sorted(v_ser)
    assert np.array_equal(x_fast, x_ser)


@pytest.mark.parametrize("case", ["plain", "nonstr_key", "big_count", "empty_map"])
def test_parallel_densify_matches_serial(case):
    """densify_into (threaded for >= 8192 samples) == the serial walk; unusual
    inputs take the serial path and raise its errors."""
    rng = np.random.default_rng(11)
    s = _samples(rng, 10_000)
    cols = {} if case == "empty_map" else {f"op{i}": (i * 7) % 15 for i in range(0, 30, 2)}
    if case == "nonstr_key":
        s[5000].histogram.entries[3] = 9
    if case == "big_count":
        s[9000] = SampleRecord("big", Label.MALWARE, 100,
                               OpcodeHistogram.from_counts({"op2": 2**40}))
    outs = []
    for fn in (_adapt.densify_into, _adapt.densify_into_serial):
        x = np.zeros((len(s), 15), np.int32)
        try:
            fn(s, cols, x, 15)
            outs.append(x)
        except Exception as e:  # noqa: BLE001
            outs.append(type(e))
    if case == "big_count":
        assert outs[0] == outs[1] and isinstance(outs[0], type)
    else:
        assert np.array_equal(outs[0], outs[1])
        assert outs[0].any() == (case != "empty_map")
