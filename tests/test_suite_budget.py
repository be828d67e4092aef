"""Host logic of the GPU suite's session time budget (tests/conftest.py): every budgeted name is a real
test of tests/test_gpu_parity.py (a rename would silently drop the guard), and the heavy tests are
collected last in the listed order."""
import os
import subprocess
import sys

import conftest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_budgeted_tests_exist_and_are_collected_last():
    out = subprocess.run([sys.executable, "-m", "pytest", "tests/test_gpu_parity.py", "-m", "gpu", "--collect-only",
                          "-q", "-p", "no:cacheprovider"], cwd=ROOT, capture_output=True, text=True).stdout
    ids = [l.split("::", 1)[1] for l in out.splitlines() if "::" in l]
    heavy = [name for name, _ in conftest._HEAVY_COST_S]
    assert ids[-len(heavy):] == heavy
    assert all(cost > 0 for _, cost in conftest._HEAVY_COST_S)
