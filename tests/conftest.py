import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


import time

_SESSION_T0 = time.monotonic()

# The four full-size C4 / C5 GPU tests spend 1-10 minutes each in the host H-LU (stage B, 16 threads); the
# whole `-m gpu` suite is 30 min with them (profiles/round2_pytest_gpu.log: 138 passed).  They run LAST, in
# the order below, and one is skipped (never failed) when starting it would take the session past
# HM_GPU_TEST_BUDGET_S (default 1600 s; 0 = no budget, run everything), so a caller with a fixed time limit
# still gets every other result.  Costs are the durations measured on the B200 box (round 2).
_HEAVY_COST_S = [
    ("test_config4_apply_and_solve_sampled", 140.0),
    ("test_sphere_exact_solve_sherman_morrison[7]", 75.0),
    ("test_config5_sphere_exact_rank_one_and_closed_form", 40.0),
    ("test_config5_flat_apply_solve_sampled", 580.0),
    ("test_sphere_exact_solve_sherman_morrison[8]", 360.0),
]


def _heavy_index(item):
    for i, (name, _) in enumerate(_HEAVY_COST_S):
        if item.name == name:
            return i
    return -1


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs the CUDA path through the C ABI)")
    config.addinivalue_line("markers", "slow: larger oracle cases")


def pytest_collection_modifyitems(config, items):
    light = [it for it in items if _heavy_index(it) < 0]
    heavy = sorted((it for it in items if _heavy_index(it) >= 0), key=_heavy_index)
    items[:] = light + heavy


def pytest_runtest_setup(item):
    i = _heavy_index(item)
    if i < 0:
        return
    budget = float(os.environ.get("HM_GPU_TEST_BUDGET_S", "1600"))
    if budget <= 0:
        return
    elapsed = time.monotonic() - _SESSION_T0
    cost = _HEAVY_COST_S[i][1]
    if elapsed + cost > budget:
        pytest.skip(f"session time budget: {elapsed:.0f} s elapsed + ~{cost:.0f} s for this test > "
                    f"HM_GPU_TEST_BUDGET_S={budget:.0f} (0 runs everything; full run: "
                    f"profiles/round2_pytest_gpu.log)")


@pytest.fixture(scope="session")
def cfg1():
    import synth
    return synth.make_config(1)
