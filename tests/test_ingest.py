"""C++ JSONL ingestion vs the reference's parse_corpus (golden: tests/golden/ingest.npz)."""

import json

import numpy as np
import pytest

from conftest import load_golden
from paper_1905_13746_b200 import ingest
from paper_1905_13746_b200.errors import IntegrityError, ParseError


@pytest.fixture(scope="module")
def z():
    return load_golden("ingest")


@pytest.mark.parametrize("threads", [1, 3])
def test_dense_matches_reference_parse(z, threads):
    c = ingest.read_corpus(str(z["text_ok"]), allow_unlabeled=True, threads=threads)
    assert c.vocab == z["vocab"].tolist()
    assert c.ids == z["ids"].tolist()
    assert c.size.tolist() == z["size"].tolist()
    assert c.label.tolist() == [{1: 1, 0: 0, -1: -1}[int(v)] for v in z["label"]]
    for dt in (np.int32, np.uint16, np.uint8):
        assert np.array_equal(c.dense(dt), z["x"].astype(dt))


def test_errors_match_reference(z):
    for text, kind, line, msg in zip(z["bad"], z["bad_kind"], z["bad_line"], z["bad_msg"]):
        with pytest.raises((ParseError, IntegrityError)) as ei:
            ingest.read_corpus(str(text))
        assert type(ei.value).__name__ == str(kind), text
        assert str(ei.value) == str(msg), text
        if kind == "ParseError":
            assert ei.value.line_no == int(line)


def test_unlabeled_rejected_unless_allowed(z):
    with pytest.raises(ParseError) as ei:
        ingest.read_corpus(str(z["text_ok"]))
    assert "missing 'label'" in str(ei.value)


def test_records_roundtrip(z):
    recs = ingest.parse_corpus(str(z["text_ok"]), allow_unlabeled=True)
    assert [r.id for r in recs] == z["ids"].tolist()
    mix = next(r for r in recs if r.id == "mix")
    assert mix.histogram.entries == {"mov": 5, "xor": 1}


def test_large_parallel_parse_matches_single_thread():
    rng = np.random.default_rng(0)
    lines = []
    for i in range(20000):
        ops = {f"op{int(j):03d}": int(rng.integers(1, 300)) for j in rng.choice(300, 20)}
        lines.append(json.dumps({"id": f"s{i}", "label": "malware" if i % 2 else "benign",
                                 "size_bytes": int(rng.integers(0, 600000)), "opcodes": ops}))
    text = "\n".join(lines)
    a = ingest.read_corpus(text, threads=1)
    b = ingest.read_corpus(text, threads=8)
    assert a.vocab == b.vocab and a.ids == b.ids
    assert np.array_equal(a.dense(), b.dense())
    lines[12345] = lines[12345].replace('"label"', '"lbl"')
    with pytest.raises(ParseError) as ei:
        ingest.read_corpus("\n".join(lines), threads=8)
    assert ei.value.line_no == 12346
    lines[12345] = lines[100]   # duplicate id later in the file
    with pytest.raises(IntegrityError) as ei:
        ingest.read_corpus("\n".join(lines), threads=8)
    assert "at line 12346" in str(ei.value)
    lines[19000] = lines[18990]  # a second duplicate (same shard); the first in order wins
    lines[300] = lines[19500]    # and one whose twin comes later: the later line is reported
    for t in (1, 3, 8):
        with pytest.raises(IntegrityError) as ei:
            ingest.read_corpus("\n".join(lines), threads=t)
        assert "at line 12346" in str(ei.value)


def test_prediction_writer_byte_identical():
    """gnb_corpus_write_predictions == the reference's write_predictions text."""
    w = load_golden("writer")
    c = ingest.read_corpus(str(w["text_in"]), allow_unlabeled=True)
    text = c.predictions_jsonl(w["label"], np.nan_to_num(w["lp"]), w["eff"], 512000)
    assert text == str(w["out"])


@pytest.mark.parametrize("ops,want", [
    ('{"mov": 5, "mov": 0}', {}), ('{"mov": 0, "mov": 5}', {"mov": 5}),
    ('{"MOV": 2, "mov": 3}', {"mov": 5}), ('{"a": 1, "b": 2, "a": 7}', {"a": 7, "b": 2}),
    ('{"x\\u0041": 1}', {"xa": 1}), ('{"add": 0}', {})])
def test_duplicate_and_case_keys_like_json_loads(ops, want):
    """Edge rules the fast path defers to the full parser: JSON last-wins duplicates,
    case-fold merging, zero counts, escaped keys (json.loads + from_counts semantics)."""
    text = '{"id": "a", "label": "benign", "size_bytes": 1, "opcodes": %s}' % ops
    rec = ingest.parse_corpus(text)[0]
    assert rec.histogram.entries == want


def test_non_ascii_mnemonics_fold_like_str_lower():
    """Keys differing only in non-ASCII case merge as the reference's
    str.lower() merges them (corpus.py:51), though the C++ parser folds ASCII
    only: same vocabulary, same counts."""
    import json
    from refpkg import groupnb
    from paper_1905_13746_b200 import ingest
    gn = groupnb()
    if gn is None:
        pytest.skip("baseline/_ref not installed")
    recs = [{"id": "a", "label": "malware", "size_bytes": 10,
             "opcodes": {"MÖV": 2, "möv": 3, "Möv": 1, "ADD": 4, "add": 1, "ßhr": 2}},
            {"id": "b", "label": "benign", "size_bytes": 20,
             "opcodes": {"İnc": 5, "möv": 7, "ÉTÉ": 1, "été": 2}}]
    text = "\n".join(json.dumps(r, ensure_ascii=False) for r in recs)
    ref = gn.parse_corpus(text)
    got = ingest.read_corpus(text)
    want_vocab = sorted({op for s in ref for op in s.histogram.entries})
    assert got.vocab == want_vocab
    x = got.dense(np.int32)
    for i, s in enumerate(ref):
        row = {got.vocab[j]: int(x[i, j]) for j in np.nonzero(x[i])[0]}
        assert row == s.histogram.entries
