"""The reference's own test suite, unchanged, against the GPU path
(SURVEY §7.3 step 3's acceptance gate).

oracle/make_ref.sh stages pkg/src/semcache and pkg/tests into oracle/_ref
(git-ignored; built by `__graft_entry__.build()` wherever /root/reference
exists, and shipped to the GPU box with the snapshot).  A child pytest runs
the reference's test files with tests/refsuite_plugin.py rebinding, inside
the reference package, `ExactCosineIndex` to `GpuCosineIndex` ("index"
mode: ref engine.py:103-109 builds the device index, every
`index.query` call site -- engine.py:177-178, :252-253, :284-285 -- runs on
the GPU) and, in "engine" mode, `CacheEngine` to the GPU engine subclass
(device TTL purge and victim selection, engine.py:300-383).

The files covered: test_index.py (exactness vs the linear-scan oracle,
ties, removal, snapshots), test_engine.py (cal_score known answers, judge
loop, eviction-order oracles, save/load), test_acceptance.py (the paper's
acceptance criteria incl. the eviction oracle :200-229 and index recall
:272-320), and in engine mode also the trace, bench-replay and proxy
suites that drive the engine end to end.
"""

from __future__ import annotations

import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
TESTS = os.path.join(ROOT, "tests")
REF = os.path.join(ROOT, "oracle", "_ref")

SUITES = {
    "index": ["tests/test_index.py", "tests/test_engine.py", "tests/test_acceptance.py"],
    "engine": ["tests/test_engine.py", "tests/test_acceptance.py", "tests/test_traces.py",
               "tests/test_bench.py", "tests/test_proxy.py", "tests/test_prefetch.py"],
}


@pytest.mark.parametrize("mode", sorted(SUITES))
def test_reference_suite_on_gpu(mode):
    if not os.path.isdir(os.path.join(REF, "tests")) or not os.path.isdir(os.path.join(REF, "semcache")):
        pytest.skip("oracle/_ref not staged (run oracle/make_ref.sh where /root/reference exists)")
    from paper_2509_17360_b200 import _native as N
    if N.device_count() < 1:
        pytest.skip("no CUDA device")
    env = dict(os.environ)
    env["PYTHONPATH"] = os.pathsep.join([REF, ROOT, TESTS] + ([env["PYTHONPATH"]] if env.get("PYTHONPATH") else []))
    env["SINE_REF_INJECT"] = mode
    cmd = [sys.executable, "-m", "pytest", "-q", "-rs", "-p", "refsuite_plugin", "-p", "no:cacheprovider",
           "--rootdir", REF, "-c", os.devnull, *SUITES[mode]]
    r = subprocess.run(cmd, cwd=REF, env=env, stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True,
                       timeout=1800)
    out = r.stdout
    log_dir = os.path.join(ROOT, "gpurun_out")
    if os.path.isdir(log_dir):
        with open(os.path.join(log_dir, f"refsuite_{mode}.log"), "w") as fh:
            fh.write(out)
    print(out[-3000:])
    assert f"sine refsuite: injected" in out and f"({mode})" in out, "plugin did not load"
    import re
    created = int(re.search(r"device indexes created: (\d+)", out).group(1))
    assert created > 10, "the reference tests did not run on the device index"
    assert r.returncode == 0, out[-6000:]
