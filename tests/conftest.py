"""Shared test setup: markers, paths, golden fixtures, reference availability."""

from __future__ import annotations

import json
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
GOLDEN = ROOT / "tests" / "golden"
REF_SRC = Path("/root/reference/pkg/src")
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built extension")
    config.addinivalue_line("markers", "ref: needs the reference package at /root/reference (build container)")


def have_ref() -> bool:
    return (REF_SRC / "offplan" / "__init__.py").exists()


@pytest.fixture(scope="session")
def offplan():
    if not have_ref():
        pytest.skip("reference package not present (GPU box): golden fixtures cover this")
    if str(REF_SRC) not in sys.path:
        sys.path.insert(0, str(REF_SRC))
    import offplan as ref

    return ref


@pytest.fixture(scope="session")
def golden_layouts():
    return json.loads((GOLDEN / "layouts.json").read_text())


@pytest.fixture(scope="session")
def adamw_golden():
    import numpy as np

    return dict(np.load(GOLDEN / "adamw_golden.npz"))


@pytest.fixture(scope="session")
def cuda():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2212_05339_b200 import _lib

    _lib.load()  # fail loudly if the extension is missing on a GPU box
    return torch.device("cuda:0")
