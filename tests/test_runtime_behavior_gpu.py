"""Error, stale-access, configuration and scalar-semantics parity of the B200
executor against the reference interpreter (golden files:
tests/golden/make_behavior_golden.py).  Errors must match the reference's
exception class and message (op path included); successful runs must match
outputs, trace and counters."""
import json
from pathlib import Path

import numpy as np
import pytest

from conftest import GOLDEN, bits_equal

pytestmark = pytest.mark.gpu

lapis_parser = pytest.importorskip("lapis.parser")
from lapis.interp import ExecConfig, diff_outputs, format_trace  # noqa: E402

BEHAVIOR = GOLDEN / "behavior"
CASES = sorted(p.stem for p in BEHAVIOR.glob("*.npz"))


def _load(name):
    with np.load(BEHAVIOR / f"{name}.npz") as z:
        d = {k: z[k] for k in z.files}
    import re
    seq = lambda p: [d[f"{p}{i}"] for i in range(sum(1 for k in d if re.fullmatch(p + r"\d+", k)))]
    return d, seq("in"), seq("out")


@pytest.mark.parametrize("library", [True, False], ids=["library", "generated"])
@pytest.mark.parametrize("name", CASES)
def test_behavior(name, library, cuda_device):
    from paper_2509_25605_b200 import runtime
    d, inputs, outputs = _load(name)
    program = lapis_parser.parse((BEHAVIOR / f"{name}.mlir").read_text())
    config = ExecConfig(**json.loads(str(d["config"])))
    want_err = str(d["error"])
    try:
        r = runtime.run(program, str(d["entry"]), [np.array(a, copy=True) for a in inputs], config,
                        library=library)
    except Exception as e:  # noqa: BLE001 - the reference's error is the golden
        assert want_err, f"unexpected {type(e).__name__}: {e}"
        assert f"{type(e).__name__}: {e}" == want_err
        return
    assert not want_err, f"expected {want_err}"
    if library:
        rep = diff_outputs(r.outputs, outputs, rel_tol=1e-12)
        assert rep.match, str(rep)
    else:
        for got, want in zip(r.outputs, outputs):
            assert bits_equal(np.asarray(got), np.asarray(want)), (got, want)
    assert format_trace(r.trace) == str(d["trace"])
    assert {k: dict(v) for k, v in r.counters.items()} == json.loads(str(d["counters"]))
