"""Drop-in behaviour that runs on the host (no GPU): the Tc path
(classify_sequential, one thread, C) and the per-sample log_posterior / predict
on the reference's OWN objects, bit-identical to the reference; namespace
resolution; backend install / uninstall rebinding."""

import math

import numpy as np
import pytest

from refpkg import groupnb

gn = groupnb()
pytestmark = pytest.mark.skipif(gn is None, reason="baseline/_ref not installed")

from paper_1905_13746_b200 import _ns, api  # noqa: E402


def _corpus(seed=3, groups=4, per=30, vocab=64, div=0.5):
    spec = gn.SyntheticSpec(group_count=groups, samples_per_group_per_class=per,
                            vocabulary_size=vocab, divergence=div, seed=seed)
    corpus = gn.generate_synthetic(spec)
    train, _ = gn.partition_by_group(corpus, gn.GroupingConfig())
    return corpus, train


def test_namespace_resolution():
    corpus, train = _corpus()
    ns = _ns.of(train)
    assert ns.name == "groupnb" and ns.Label is gn.Label and ns.TimedRun is gn.TimedRun
    assert ns.errors.IntegrityError is gn.errors.IntegrityError
    import paper_1905_13746_b200 as own
    assert _ns.of(own.GroupingConfig()) is _ns.OWN
    assert _ns.of(object()) is _ns.OWN


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_sequential_is_reference_tc(seed):
    corpus, train = _corpus(seed=seed)
    bundle = gn.train_bundle(train, k=int(10 + 7 * seed), created_at="t")
    rng = np.random.default_rng(seed)
    samples = [corpus[i] for i in rng.integers(0, len(corpus), size=500)]
    samples[17] = gn.SampleRecord("big", gn.Label.UNKNOWN, 512000 + seed,
                                  gn.OpcodeHistogram.from_counts({"op01": 1}))
    samples[33] = gn.SampleRecord("neg", gn.Label.UNKNOWN, -5,
                                  gn.OpcodeHistogram.from_counts({"op01": 1}))
    work = gn.Workload(tuple(samples), lanes=3)
    ref = gn.classify_sequential(bundle, work)
    got = api.classify_sequential(bundle, work)
    assert type(got) is gn.TimedRun
    assert got.predictions == ref.predictions and got.errors == ref.errors
    assert all(type(p) is gn.Prediction for p in got.predictions if p is not None)
    assert got.elapsed_ns > 0


def test_sequential_empty_bundle_raises_reference_type():
    meta = gn.BundleMeta(k=3, alpha=1.0, seed=0, created_at="t")
    empty = gn.build_bundle([], gn.GroupingConfig(), meta)
    with pytest.raises(gn.errors.EmptyBundleError):
        api.classify_sequential(empty, gn.Workload((), lanes=1))


def test_log_posterior_exact_incl_unusual_inputs():
    corpus, train = _corpus()
    bundle = gn.train_bundle(train, k=25, created_at="t")
    m = bundle.models[bundle.trained_ids[0]]
    for s in corpus[:200]:
        assert api.log_posterior(m, s.histogram) == gn.log_posterior(m, s.histogram)
        assert api.predict(m, s.histogram) == gn.predict(m, s.histogram)
    ops = m.features.opcodes
    odd = [gn.OpcodeHistogram({ops[0]: 2**70}),              # int beyond 2^53: float(n)
           gn.OpcodeHistogram({ops[0]: 3, ops[1]: 2.5}),      # float count: generic protocol
           gn.OpcodeHistogram({ops[2]: True}),
           gn.OpcodeHistogram({}),
           gn.OpcodeHistogram({"not-a-feature": 9})]
    for h in odd:
        assert api.log_posterior(m, h) == gn.log_posterior(m, h)
    with pytest.raises(OverflowError):
        gn.log_posterior(m, gn.OpcodeHistogram({ops[0]: 10**400}))
    with pytest.raises(OverflowError):
        api.log_posterior(m, gn.OpcodeHistogram({ops[0]: 10**400}))


def test_duplicate_features_scored_twice_like_reference():
    corpus, train = _corpus()
    g = sorted(train.groups)[0]
    base = gn.train_bundle(train, k=5, created_at="t").models[g].features.opcodes
    feats = gn.FeatureSet((base[0], base[0], base[1]), 3)
    model = gn.train_group(train.groups[g], feats, 1.0, group=g)
    for s in corpus[:50]:
        assert api.log_posterior(model, s.histogram) == gn.log_posterior(model, s.histogram)


def test_own_objects_match_reference_tc():
    """Our own object model through Tc == the reference's Tc on the same data."""
    import paper_1905_13746_b200 as own
    corpus, train = _corpus(seed=5)
    rbundle = gn.train_bundle(train, k=12, created_at="t")
    conv = {gn.Label.MALWARE: own.Label.MALWARE, gn.Label.BENIGN: own.Label.BENIGN,
            gn.Label.UNKNOWN: own.Label.UNKNOWN}
    models = []
    for g, m in rbundle.models.items():
        models.append(own.GroupModel(
            group=g, features=own.FeatureSet(m.features.opcodes, m.features.k),
            log_prior={conv[c]: v for c, v in m.log_prior.items()},
            log_likelihood={conv[c]: dict(d) for c, d in m.log_likelihood.items()},
            alpha=m.alpha, train_counts={conv[c]: v for c, v in m.train_counts.items()}))
    obundle = own.build_bundle(models, own.GroupingConfig(),
                               own.BundleMeta(12, 1.0, 0, "t"))
    osamples = tuple(own.SampleRecord(s.id, conv[s.label], s.size_bytes,
                                      own.OpcodeHistogram.from_counts(s.histogram.entries))
                     for s in corpus)
    ref = gn.classify_sequential(rbundle, gn.Workload(tuple(corpus), lanes=1))
    got = own.classify_sequential(obundle, own.Workload(osamples, lanes=1))
    assert [(p.label.value, p.log_posterior[own.Label.MALWARE], p.log_posterior[own.Label.BENIGN],
             p.effective_group) for p in got.predictions] == \
        [(p.label.value, p.log_posterior[gn.Label.MALWARE], p.log_posterior[gn.Label.BENIGN],
          p.effective_group) for p in ref.predictions]


def test_backend_install_rebinds_and_restores():
    from paper_1905_13746_b200 import backend
    import groupnb.bench
    import groupnb.classifier
    import groupnb.engine
    orig = (gn.engine.classify_parallel, gn.engine.train_bundle, gn.classifier.train_group,
            gn.bench.train_bundles, gn.classify_parallel, gn.train_bundle, gn.train_group,
            gn.engine.train_group, gn.bench.train_group)
    seq = gn.engine.classify_sequential
    try:
        calls = backend.install(gn)
        assert backend.installed() and calls == {}
        now = (gn.engine.classify_parallel, gn.engine.train_bundle, gn.classifier.train_group,
               gn.bench.train_bundles, gn.classify_parallel, gn.train_bundle, gn.train_group,
               gn.engine.train_group, gn.bench.train_group)
        assert all(a is not b for a, b in zip(orig, now))
        assert gn.classify_parallel is gn.engine.classify_parallel
        assert gn.engine.classify_sequential is seq            # Tc stays the reference's
        assert gn.classifier.log_posterior.__module__ == "groupnb.classifier"
        assert backend.install(gn) is calls                    # idempotent
    finally:
        backend.uninstall()
    assert not backend.installed()
    back = (gn.engine.classify_parallel, gn.engine.train_bundle, gn.classifier.train_group,
            gn.bench.train_bundles, gn.classify_parallel, gn.train_bundle, gn.train_group,
            gn.engine.train_group, gn.bench.train_group)
    assert all(a is b for a, b in zip(orig, back))
