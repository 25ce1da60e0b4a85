"""Runs the reference package's own tests (staged by make_suite.py) against the drop-in.

``l1pcp`` and its submodules are aliased to ``paper_1108_5359_b200``; the reference's
``l1pcp.bench`` harness maps to ``paper_1108_5359_b200.suites``.  Every test here needs the GPU
(the drop-in has no CPU path), so all are marked ``gpu``.  Reference tests that cannot hold for a
documented reason are listed in KNOWN_BREAKS (INTEGRATION.md §4 carries the same list); they run
as strict xfails, so a fix shows up as an XPASS failure and the list must shrink with it.
"""

import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

import paper_1108_5359_b200 as _pkg  # noqa: E402
from paper_1108_5359_b200 import (cli, l1filter, l1reg, matcore, matio, pcp_adm,  # noqa: E402
                                  suites, synth)

sys.modules["l1pcp"] = _pkg
for _name, _mod in (("cli", cli), ("l1filter", l1filter), ("l1reg", l1reg), ("matcore", matcore),
                    ("matio", matio), ("pcp_adm", pcp_adm), ("synth", synth), ("bench", suites)):
    sys.modules["l1pcp." + _name] = _mod
    setattr(_pkg, _name, _mod)

# nodeid suffix -> reason
KNOWN_BREAKS = {
    # The drop-in's synth.generate draws from Philox, not PCG64 (not bit-compatible by design,
    # SURVEY 8(a) a12), so "seed 3" is a different 500x500 instance.  On it the reference's own
    # estimate_rank_and_solve reaches RelErr 8.42e-4 as well (the drop-in's L differs from the
    # reference's by 2e-10 relative on all five instances): tests/test_gpu_reference_instances.py.
    "test_ref_acceptance.py::test_exact_recovery_m500":
        "instance-dependent: Philox seed-3 instance is hard for the reference algorithm itself",
    # Wall-clock complexity exponents of a CPU implementation: on the GPU the full ADM at
    # n <= 2000 is latency-bound (exponent ~1.4, not >= 1.7) and the l1-filter/ADM ratio at 2000 is
    # set by kernel launches, not flops.
    "test_ref_acceptance.py::test_scaling_law":
        "CPU timing-shape assertion (ADM exponent >= 1.7); GPU ADM is latency-bound at n <= 2000",
}

HERE = os.path.dirname(os.path.abspath(__file__))


def pytest_collection_modifyitems(config, items):
    for item in items:
        if not str(item.fspath).startswith(HERE):
            continue
        item.add_marker(pytest.mark.gpu)
        for suffix, reason in KNOWN_BREAKS.items():
            if item.nodeid.endswith(suffix):
                item.add_marker(pytest.mark.xfail(reason=reason, strict=True))
