"""pytest plugin: run a test session with the GPU backend installed in the
reference package (`python -m pytest -p paper_1905_13746_b200.pytest_backend
<groupnb tests>`).  Installs before any test module is imported, so the
reference's `from groupnb.engine import classify_parallel` lines bind the GPU
versions; the session summary reports how often each rebound operation ran."""

from __future__ import annotations

_calls: dict = {}


def pytest_configure(config):
    from . import backend
    _calls.update(backend.install())          # returns the live counters
    _calls["__live__"] = backend._state["calls"]


def pytest_terminal_summary(terminalreporter):
    live = _calls.get("__live__", {})
    terminalreporter.write_line(
        "[gnb-backend] " + " ".join(f"{k}={v}" for k, v in sorted(live.items())))
