"""Shared pytest configuration.

Markers: ``gpu`` — needs a B200 (run on the GPU box with ``-m gpu``); everything
else runs on CPU.
"""
from __future__ import annotations

import json
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent
GOLDEN = Path(__file__).resolve().parent / "golden"
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))
# the reference package (the caller of the drop-in runtime): pip-installed into
# baseline/_ref by __graft_entry__.build(); travels to the GPU box
REF_PKG = ROOT / "baseline" / "_ref"
if REF_PKG.exists() and str(REF_PKG) not in sys.path:
    sys.path.append(str(REF_PKG))
RUN_GOLDEN = GOLDEN / "run"


def run_cases() -> list[str]:
    """<program>.<seed> ids of tests/golden/run (make_run_golden.py)."""
    return sorted(p.name[:-4] for p in RUN_GOLDEN.glob("*.npz"))


def load_run_case(case: str) -> dict:
    import json as _json
    name, _ = case.rsplit(".", 1)
    with np.load(RUN_GOLDEN / f"{case}.npz") as z:
        d = {k: z[k] for k in z.files}
    import re as _re

    def seq(prefix):
        n = sum(1 for k in d if _re.fullmatch(prefix + r"\d+", k))
        return [d[f"{prefix}{i}"] for i in range(n)]
    return {
        "name": name,
        "entry": str(d["entry"]),
        "inputs": seq("in"),
        "outputs": seq("out"),
        "orig_outputs": seq("orig"),
        "trace": str(d["trace"]), "eager_trace": str(d["eager_trace"]),
        "orig_trace": str(d["orig_trace"]),
        "counters": _json.loads(str(d["counters"])),
        "orig_counters": _json.loads(str(d["orig_counters"])),
        "lowered": (RUN_GOLDEN / f"{name}.lowered.mlir").read_text(),
        "orig": (RUN_GOLDEN / f"{name}.orig.mlir").read_text(),
    }


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 device (sm_100a)")


def load_golden(name: str) -> dict:
    """A reference-generated fixture: inputs list, outputs list, trace, hints."""
    with np.load(GOLDEN / f"{name}.npz") as z:
        d = {k: z[k] for k in z.files}
    ins = [d[f"in{i}"] for i in range(sum(1 for k in d if k.startswith("in")))]
    outs = [d[f"out{i}"] for i in range(sum(1 for k in d if k.startswith("out")))]
    orig = [d[f"orig{i}"] for i in range(sum(1 for k in d if k.startswith("orig")))]
    return {"inputs": ins, "outputs": outs, "orig": orig,
            "trace": json.loads(str(d["trace"])), "hints": json.loads(str(d["hints"]))}


def golden_names(prefix: str = "") -> list[str]:
    return sorted(p.stem for p in GOLDEN.glob(f"{prefix}*.npz"))


def bits_equal(a, b) -> bool:
    """Bitwise equality (floats compared through their integer views)."""
    a, b = np.asarray(a), np.asarray(b)
    if a.shape != b.shape or a.dtype != b.dtype:
        return False
    if a.dtype.kind == "f":
        iv = {2: np.uint16, 4: np.uint32, 8: np.uint64}[a.dtype.itemsize]
        return np.array_equal(a.view(iv), b.view(iv))
    return np.array_equal(a, b)


@pytest.fixture(scope="session")
def cuda_device():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch.device("cuda:0")
