"""Generate the golden parity fixtures by running the REFERENCE package.

Run here (the container that has /root/reference); the GPU box never does.
Each case runs the reference's own stock path -- synthetic corpus,
`split_train_test`, `train_bundle`, `classify_sequential` -- and stores its
inputs as dense arrays plus its outputs (the canonical bundle JSON and every
prediction's label / log-scores / effective group / error message) in
`tests/golden/<case>.npz`.

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py

Reference entry points exercised (file:line under /root/reference):
  pkg/src/groupnb/synth.py:83        generate_synthetic
  pkg/src/groupnb/corpus.py:235,255  partition_by_group, split_train_test
  pkg/src/groupnb/engine.py:157      train_bundle
  pkg/src/groupnb/engine.py:209      classify_sequential
  pkg/src/groupnb/engine.py:324      bundle_to_json
"""

from __future__ import annotations

import os
import sys

sys.dont_write_bytecode = True
REF = "/root/reference/pkg/src"
sys.path.insert(0, REF)

import numpy as np  # noqa: E402

from groupnb import (  # noqa: E402
    GroupingConfig,
    Label,
    OpcodeHistogram,
    SampleRecord,
    SyntheticSpec,
    Workload,
    bundle_to_json,
    classify_sequential,
    generate_synthetic,
    partition_by_group,
    split_train_test,
    train_bundle,
)

OUT = os.path.dirname(os.path.abspath(__file__))
_LABEL_CODE = {Label.BENIGN: 0, Label.MALWARE: 1, Label.UNKNOWN: -1}


def _dense(samples, vocab):
    index = {op: i for i, op in enumerate(vocab)}
    x = np.zeros((len(samples), len(vocab)), dtype=np.uint16)
    for r, s in enumerate(samples):
        for op, n in s.histogram.entries.items():
            assert n < 65536
            x[r, index[op]] = n
    size = np.array([s.size_bytes for s in samples], dtype=np.int64)
    label = np.array([_LABEL_CODE[s.label] for s in samples], dtype=np.int8)
    return x, size, label


def _save(name, *, train_samples, test_samples, config, k, alpha, extra_vocab=()):
    grouped, rejected = partition_by_group(train_samples, config)
    assert not rejected
    bundle = train_bundle(grouped, k=k, alpha=alpha, created_at="golden")
    run = classify_sequential(bundle, Workload(tuple(test_samples), lanes=1), warmup=False)

    vocab = sorted(
        {op for s in list(train_samples) + list(test_samples) for op in s.histogram.entries}
        | set(extra_vocab)
    )
    tx, tsz, tlab = _dense(train_samples, vocab)
    qx, qsz, _ = _dense(test_samples, vocab)
    m = len(test_samples)
    pred_label = np.full(m, -1, dtype=np.int8)
    pred_lp = np.full((m, 2), np.nan, dtype=np.float64)  # [benign, malware]
    pred_group = np.full(m, -1, dtype=np.int32)
    for i, p in enumerate(run.predictions):
        if p is None:
            continue
        pred_label[i] = _LABEL_CODE[p.label]
        pred_lp[i, 0] = p.log_posterior[Label.BENIGN]
        pred_lp[i, 1] = p.log_posterior[Label.MALWARE]
        pred_group[i] = p.effective_group
    err_index = np.array([i for i, _ in run.errors], dtype=np.int64)
    err_msg = np.array([msg for _, msg in run.errors], dtype=np.str_)
    np.savez_compressed(
        os.path.join(OUT, f"{name}.npz"),
        vocab=np.array(vocab, dtype=np.str_),
        train_x=tx, train_size=tsz, train_label=tlab,
        test_x=qx, test_size=qsz,
        group_size_bytes=config.group_size_bytes,
        max_size_bytes=config.max_size_bytes,
        min_per_class=config.min_per_class,
        k=k, alpha=float(alpha),
        bundle_json=np.array(bundle_to_json(bundle)),
        pred_label=pred_label, pred_lp=pred_lp, pred_group=pred_group,
        err_index=err_index, err_msg=err_msg,
    )
    print(f"{name}: train={len(train_samples)} test={m} V={len(vocab)} "
          f"groups={bundle.trained_ids} errors={len(run.errors)}")


def _sample(sid, label, size, ops):
    return SampleRecord(sid, label, size, OpcodeHistogram.from_counts(ops))


def case_paper():
    """cfg 1: ~4k samples, one size group, V=256, k=100, 2 classes."""
    corpus = generate_synthetic(SyntheticSpec(1, 2000, 256, 0.1, 0))
    grouped, _ = partition_by_group(corpus, GroupingConfig())
    split = split_train_test(grouped, (2, 1), seed=0)
    train = split.train.all_samples()
    test = split.test.all_samples() + train  # also re-score the training rows
    _save("paper", train_samples=train, test_samples=test,
          config=GroupingConfig(), k=100, alpha=1.0)


def case_groups():
    """Ragged multi-group corpus with untrained groups, routing and oversize rows."""
    config = GroupingConfig()
    corpus = generate_synthetic(SyntheticSpec(12, 10, 40, 0.3, 5))
    train = []
    for s in corpus:
        g = s.size_bytes // config.group_size_bytes
        idx = int(s.id.split("-")[1])
        if g in (3, 7, 11) and s.label is Label.MALWARE and idx >= 2:
            continue  # below min_per_class: no model for 3, 7, 11
        if g == 9:
            continue  # empty group
        train.append(s)
    rng = np.random.default_rng(11)
    test = [corpus[i] for i in rng.permutation(len(corpus))]
    # unlabeled rows in every group incl. empty / untrained / above-last-trained
    for g in range(0, 14):
        size = g * config.group_size_bytes + int(rng.integers(0, config.group_size_bytes))
        ops = {f"op{int(j):02d}": int(rng.integers(1, 30)) for j in rng.choice(40, 9, replace=False)}
        ops["notinvocab"] = 3
        test.append(_sample(f"u{g}", Label.UNKNOWN, size, ops))
    for pos, size in ((5, 512000), (17, 600000), (30, -1), (31, 511999), (44, 0)):
        test.insert(pos, _sample(f"edge{pos}", Label.UNKNOWN, size, {"op01": 2, "op39": 1}))
    test.append(_sample("empty", Label.UNKNOWN, 100, {}))
    _save("groups", train_samples=train, test_samples=test, config=config, k=15, alpha=1.0)


def case_small_vocab():
    """k larger than the scored vocabulary; alpha != 1; small groups."""
    config = GroupingConfig(group_size_bytes=1000, max_size_bytes=4000, min_per_class=2)
    corpus = generate_synthetic(SyntheticSpec(4, 5, 6, 0.5, 3), group_size_bytes=1000)
    _save("small_vocab", train_samples=corpus, test_samples=corpus,
          config=config, k=50, alpha=0.5)


def case_ties():
    """Equal scores break by mnemonic; case folding; off-vocabulary test opcodes."""
    config = GroupingConfig(min_per_class=1)
    train = [
        _sample("m0", Label.MALWARE, 10, {"mov": 2, "ADD": 2, "jmp": 1, "call": 1, "xor": 4}),
        _sample("m1", Label.MALWARE, 20, {"mov": 2, "add": 2, "jmp": 1, "call": 1}),
        _sample("b0", Label.BENIGN, 30, {"mov": 1, "add": 1, "jmp": 2, "call": 2, "nop": 4}),
        _sample("b1", Label.BENIGN, 40, {"mov": 1, "add": 1, "jmp": 2, "call": 2}),
    ]
    test = list(train) + [
        _sample("t0", Label.UNKNOWN, 50, {"mov": 3, "jmp": 3}),
        _sample("t1", Label.UNKNOWN, 60, {"nop": 7, "lea": 9}),
        _sample("t2", Label.UNKNOWN, 70, {}),
    ]
    _save("ties", train_samples=train, test_samples=test, config=config, k=4, alpha=1.0,
          extra_vocab=("lea",))


if __name__ == "__main__":
    case_paper()
    case_groups()
    case_small_vocab()
    case_ties()


def case_ingest():
    """parse_corpus (corpus.py:133-189) on valid JSONL and on malformed lines."""
    import json as _json
    from groupnb import GroupNBError, parse_corpus, serialize_sample
    corpus = generate_synthetic(SyntheticSpec(3, 7, 12, 0.4, 9))
    lines = [serialize_sample(s) for s in corpus]
    # extra valid variety: unknown keys, mixed-case + merged mnemonics, zeros, blank lines
    lines.insert(3, _json.dumps({"id": "mix", "label": "malware", "size_bytes": 77,
                                 "opcodes": {"MOV": 2, "mov": 3, "Add": 0, "xor": 1},
                                 "extra": [1, 2]}))
    lines.insert(5, "")
    lines.insert(6, "   ")
    lines.append(_json.dumps({"id": "u1", "size_bytes": 5, "opcodes": {}}))
    text_ok = "\n".join(lines) + "\n"
    recs = parse_corpus(text_ok, allow_unlabeled=True)
    vocab = sorted({op for r in recs for op in r.histogram.entries})
    x, size, label = _dense(recs, vocab)
    bad_lines = [
        '{"id": "a", "label": "malware", "size_bytes": 1, "opcodes": {}}\n{"id": "a", "label": "benign", "size_bytes": 2, "opcodes": {}}',
        '{"id": "a", "label": "malware", "size_bytes": 1, "opcodes": {}}\n{"id": "a", "label": "bogus", "size_bytes": 2, "opcodes": {}}',
        '{"id": "a", "label": "malware", "size_bytes": 1, "opcodes": {}}\n[1, 2]',
        '{"id": "", "label": "malware", "size_bytes": 1, "opcodes": {}}',
        '{"label": "malware", "size_bytes": 1, "opcodes": {}}',
        '{"id": "b", "label": "spam", "size_bytes": 1, "opcodes": {}}',
        '{"id": "b", "label": 7, "size_bytes": 1, "opcodes": {}}',
        '{"id": "b", "size_bytes": 1, "opcodes": {}}',
        '{"id": "b", "label": "benign", "size_bytes": -1, "opcodes": {}}',
        '{"id": "b", "label": "benign", "size_bytes": 1.5, "opcodes": {}}',
        '{"id": "b", "label": "benign", "size_bytes": true, "opcodes": {}}',
        '{"id": "b", "label": "benign", "size_bytes": 3, "opcodes": [1]}',
        '{"id": "b", "label": "benign", "size_bytes": 3, "opcodes": {"": 1}}',
        '{"id": "b", "label": "benign", "size_bytes": 3, "opcodes": {"mov": -2}}',
        '{"id": "b", "label": "benign", "size_bytes": 3, "opcodes": {"mov": 2.0}}',
        '{"id": "b", "label": "benign", "size_bytes": 3, "opcodes": {"mov": "2"}}',
        '{"id": "b", "label": "benign", "size_bytes": 3, "opcodes": {"mov": false}}',
        '{"id": "b", "label": "benign", "size_bytes": 3, "opcodes": {"mov": 1}} trailing',
        '{"id": "b" "label": "benign"}',
    ]
    kinds, lines_no, msgs = [], [], []
    for t in bad_lines:
        try:
            parse_corpus(t)
            raise AssertionError("expected an error: " + t)
        except GroupNBError as exc:
            kinds.append(type(exc).__name__)
            lines_no.append(getattr(exc, "line_no", -1))
            msgs.append(str(exc))
    np.savez_compressed(
        os.path.join(OUT, "ingest.npz"),
        text_ok=np.array(text_ok), vocab=np.array(vocab, dtype=np.str_), x=x, size=size,
        label=label, ids=np.array([r.id for r in recs], dtype=np.str_),
        bad=np.array(bad_lines, dtype=np.str_), bad_kind=np.array(kinds, dtype=np.str_),
        bad_line=np.array(lines_no), bad_msg=np.array(msgs, dtype=np.str_))
    print(f"ingest: rows={len(recs)} V={len(vocab)} error cases={len(bad_lines)}")


def case_writer():
    """write_predictions (engine.py:466-481) text, incl. error rows and non-ASCII ids."""
    import io
    from groupnb import parse_corpus, serialize_sample, write_predictions
    config = GroupingConfig()
    corpus = generate_synthetic(SyntheticSpec(3, 8, 16, 0.3, 21))
    train, _ = partition_by_group(corpus, config)
    bundle = train_bundle(train, k=10, alpha=1.0, created_at="golden")
    rng = np.random.default_rng(5)
    test = [corpus[i] for i in rng.permutation(len(corpus))[:30]]
    odd = ["caf\u00e9-\u00fc", 'q"uote\\back', "tab\tnl", "emoji-\U0001F600"]
    for j, sid in enumerate(odd):
        s = test[j]
        test[j] = SampleRecord(sid, Label.UNKNOWN, s.size_bytes, s.histogram)
    test.insert(7, _sample("big", Label.UNKNOWN, 600000, {"op01": 1}))
    text_in = "\n".join(serialize_sample(s) for s in test) + "\n"
    samples = parse_corpus(text_in, allow_unlabeled=True)
    run = classify_sequential(bundle, Workload(tuple(samples), lanes=1), warmup=False)
    sink = io.StringIO()
    write_predictions(run, samples, sink)
    m = len(samples)
    lab = np.full(m, -1, np.int8)
    lp = np.full((m, 2), np.nan)
    eff = np.full(m, -1, np.int32)
    for i, p in enumerate(run.predictions):
        if p is not None:
            lab[i] = _LABEL_CODE[p.label]
            lp[i] = [p.log_posterior[Label.BENIGN], p.log_posterior[Label.MALWARE]]
            eff[i] = p.effective_group
    train_text = "\n".join(serialize_sample(s) for s in train.all_samples()) + "\n"
    np.savez_compressed(os.path.join(OUT, "writer.npz"), text_in=np.array(text_in),
                        train_text=np.array(train_text), label=lab, lp=lp, eff=eff,
                        out=np.array(sink.getvalue()), k=10)
    print(f"writer: rows={m} bytes={len(sink.getvalue())}")


if __name__ == "__main__":
    case_ingest()
    case_writer()
