"""pytest plugin: run the reference's OWN test files against the GPU path.

Loaded by tests/test_reference_suite_gpu.py as `-p refsuite_plugin` in a
child pytest whose rootdir is oracle/_ref (the reference package and its
tests, staged by oracle/make_ref.sh).  Before the reference's test modules
are collected it rebinds, inside the reference package itself,

* SINE_REF_INJECT=index  -- `semcache.index.ExactCosineIndex` and
  `semcache.engine.ExactCosineIndex` to `GpuCosineIndex`: every index the
  tests build, and every index the reference `CacheEngine` builds by
  default (engine.py:103-109), is the device index;
* SINE_REF_INJECT=engine -- additionally `semcache.CacheEngine` and
  `semcache.engine.CacheEngine` to `paper_2509_17360_b200.CacheEngine`
  (a subclass of the reference engine with the device eviction pass), so
  the engine tests, the bench replay and the proxy run on it.

The reference test files themselves are not modified.
"""

from __future__ import annotations

import os

MODE = os.environ.get("SINE_REF_INJECT", "index")
_injected = {}
_created = [0]  # GpuCosineIndex handles the reference tests created


def pytest_configure(config):
    import semcache
    import semcache.engine
    import semcache.index

    from paper_2509_17360_b200 import CacheEngine, GpuCosineIndex

    init = GpuCosineIndex.__init__

    def counted_init(self, *a, **kw):
        init(self, *a, **kw)
        _created[0] += 1

    GpuCosineIndex.__init__ = counted_init

    class ExactCosineIndex(GpuCosineIndex):
        """GpuCosineIndex under the reference's class name and constructor."""

        def __init__(self, dimension: int, seed: int = 1):
            super().__init__(dimension, seed=seed)

    semcache.index.ExactCosineIndex = ExactCosineIndex
    semcache.engine.ExactCosineIndex = ExactCosineIndex
    _injected["index"] = ExactCosineIndex
    if MODE == "engine":
        semcache.engine.CacheEngine = CacheEngine
        semcache.CacheEngine = CacheEngine
        _injected["engine"] = CacheEngine


def pytest_terminal_summary(terminalreporter):
    names = {k: f"{v.__module__}.{v.__qualname__}" for k, v in _injected.items()}
    terminalreporter.write_line(f"sine refsuite: injected {names} ({MODE}); "
                                f"device indexes created: {_created[0]}")
