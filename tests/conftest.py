"""Shared pytest setup: the `gpu` marker, import paths, golden loaders."""

from __future__ import annotations

import json
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden")
for p in (ROOT, GOLDEN):
    if p not in sys.path:
        sys.path.insert(0, p)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built libsine_b200.so")


def load_golden(name: str):
    with open(os.path.join(GOLDEN, name)) as fh:
        return json.load(fh)


@pytest.fixture(scope="session")
def index_golden():
    return load_golden("index_golden.json")


@pytest.fixture(scope="session")
def evict_golden():
    return load_golden("evict_golden.json")


@pytest.fixture(scope="session")
def trace_golden():
    return load_golden("engine_trace_golden.json")
