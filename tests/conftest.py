"""Shared fixtures.  ``-m gpu`` tests need a B200 (they run on the GPU box);
everything else runs on the CPU container."""

import os
import sys

import numpy as np
import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if REPO not in sys.path:
    sys.path.insert(0, REPO)
GOLDEN = os.path.join(REPO, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")


def _load(name):
    return dict(np.load(os.path.join(GOLDEN, name), allow_pickle=False))


@pytest.fixture(scope="session")
def golden_corpus():
    return _load("corpus.npz")


@pytest.fixture(scope="session")
def golden_c1():
    return _load("c1.npz")


@pytest.fixture(scope="session")
def golden_synth42():
    return _load("synth42.npz")


def corpus_graph(gold, i):
    """(n, src, dst) of corpus graph i as stored by make_golden.py."""
    return int(gold[f"g{i}_n"]), gold[f"g{i}_src"], gold[f"g{i}_dst"]
