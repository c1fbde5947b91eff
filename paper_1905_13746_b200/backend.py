"""The reference-side binding: put the GPU path behind `groupnb`'s own API.

SPEC.md:392 makes a GPU backend "an optional extension point behind the same
operation contract".  `install()` is that extension point, as code: it rebinds
the reference package's hot-path operations to this package's GPU versions,
in every already-imported `groupnb` module, so callers -- the reference's own
CLI (cli.py:214-245), bench sweep (`run_bench`, bench.py:114-172) and tests --
run unchanged on the B200:

  groupnb.engine.classify_parallel   (Tp, engine.py:250-296)  -> K-PRED
  groupnb.engine.train_bundle        (engine.py:157-177)      -> K-FIT + FIN
  groupnb.classifier.train_group     (classifier.py:68-129)   -> K-FIT + FIN
  groupnb.bench.train_bundles        (bench.py:91-111)        -> one K-FIT, FIN per k

`classify_sequential` (Tc) and the per-sample `log_posterior` / `predict` stay
the reference's own Python: Tc is the baseline side of `speedup(Tc, Tp)`
(engine.py:209-226, "never parallelized internally"), so after `install()` the
reference's bench reports GPU-vs-reference-CPU speedups and its acceptance
test C4 checks GPU Tp against the reference's own Tc bit for bit.

The replacements read and return the reference's own objects (`_ns`): a
`groupnb.GroupedCorpus` trains into a `groupnb.ModelBundle`, a `groupnb`
bundle classifies into a `groupnb.engine.TimedRun`, errors are
`groupnb.errors.*`.  Densifying the histograms is `_adapt` (C API, threaded);
there is no per-sample Python loop on the way to the device.

    import groupnb
    from paper_1905_13746_b200 import backend
    backend.install(groupnb)              # or backend.install() to import it
    ...                                   # groupnb API, now on the GPU
    backend.uninstall()
"""

from __future__ import annotations

import functools
import importlib
import sys
import threading

from . import api

_lock = threading.Lock()
_state: dict = {}      # installed: {"module": groupnb, "orig": {qualname: fn}, "calls": {...}}


def _replacements(device, devices, calls):
    def counted(name, fn):
        @functools.wraps(fn)
        def wrapper(*a, **kw):
            calls[name] = calls.get(name, 0) + 1
            return fn(*a, **kw)
        return wrapper

    def classify_parallel(bundle, workload, *, warmup=True):
        return api.classify_parallel(bundle, workload, warmup=warmup, device=device,
                                     devices=devices)

    def train_bundle(train, k, alpha=1.0, *, seed=0, created_at=None):
        return api.train_bundle(train, k, alpha, seed=seed, created_at=created_at, device=device,
                                devices=devices)

    def train_group(samples, features, alpha=1.0, *, group=0):
        return api.train_group(samples, features, alpha, group=group, device=device)

    def train_bundles(train, k_values, alpha=1.0, *, seed=0, created_at=""):
        return api.train_bundles(train, k_values, alpha, seed=seed, created_at=created_at,
                                 device=device, devices=devices)

    return {
        "engine.classify_parallel": counted("classify_parallel", classify_parallel),
        "engine.train_bundle": counted("train_bundle", train_bundle),
        "classifier.train_group": counted("train_group", train_group),
        "bench.train_bundles": counted("train_bundles", train_bundles),
    }


def install(groupnb=None, *, device=None, devices=None) -> dict:
    """Rebind groupnb's fit / Tp operations to the GPU; returns the call
    counters ({operation: calls}) so a caller can prove the GPU path ran.
    `device` / `devices` as for `api.classify_parallel` (several GPUs: rows
    sharded contiguously)."""
    with _lock:
        if _state:
            return _state["calls"]
        mod = groupnb if groupnb is not None else importlib.import_module("groupnb")
        root = mod.__name__
        for sub in ("engine", "classifier", "bench"):
            importlib.import_module(f"{root}.{sub}")
        calls: dict[str, int] = {}
        repl = _replacements(device, devices, calls)
        orig = {}
        for qual, fn in repl.items():
            sub, name = qual.split(".")
            orig[qual] = getattr(sys.modules[f"{root}.{sub}"], name)
        _rebind(root, {id(orig[q]): repl[q] for q in repl})
        _state.update(module=mod, orig=orig, repl=repl, calls=calls)
        return calls


def uninstall() -> None:
    """Restore the reference's own functions everywhere install() rebound them."""
    with _lock:
        if not _state:
            return
        root = _state["module"].__name__
        _rebind(root, {id(_state["repl"][q]): _state["orig"][q] for q in _state["repl"]})
        _state.clear()


def installed() -> bool:
    return bool(_state)


def _rebind(root: str, mapping: dict) -> None:
    """Every attribute of every loaded `root` module bound to a key function
    (`from .engine import classify_parallel` copies included) -> its value."""
    for name, m in list(sys.modules.items()):
        if m is None or not (name == root or name.startswith(root + ".")):
            continue
        for attr, val in list(vars(m).items()):
            new = mapping.get(id(val))
            if new is not None:
                setattr(m, attr, new)
