"""The HM_DEVICE_CHECKS build (VERDICT r1 "What's weak" 9: compute-sanitizer is closed on the GPU pool,
so the engines check every chunk descriptor and gathered index on the device and trap on a violation).

The checked library is linked to its own path (libhm_checked.so) and loaded through HM_LIB in child
processes, so the product library of this session is untouched.  (1) The checked build runs the
single-vector, multi-RHS and sharded (virtual-rank) parity tests unchanged: every descriptor of those
programs is inside its bounds.  (2) With HM_CHECK_SELFTEST=1 one chunk is moved past the end of its
arena at program finalisation; the checked engine must trap on it (the call fails, the device printf
names the check) -- proof that the checks are compiled in and reached.
"""
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def checked_lib():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a B200")
    sys.path.insert(0, ROOT)
    from paper_2305_06891_b200 import build
    return build.build(defines=("HM_DEVICE_CHECKS=1",), lib=os.path.join(ROOT, "paper_2305_06891_b200", "libhm_checked.so"))


def _env(lib, **extra):
    env = dict(os.environ)
    env["HM_LIB"] = lib
    env.update(extra)
    return env


def test_checked_build_runs_the_parity_tests(checked_lib):
    cmd = [sys.executable, "-m", "pytest", "-x", "-q", "-p", "no:cacheprovider",
           os.path.join(ROOT, "tests", "test_gpu_parity.py") + "::test_solve_and_flux_match_dense_oracle",
           os.path.join(ROOT, "tests", "test_gpu_parity.py") + "::test_multi_rhs_dmma_matches_single_columns_and_oracle",
           os.path.join(ROOT, "tests", "test_gpu_shard.py") + "::test_virtual_shards_match_single_rank_and_oracle",
           os.path.join(ROOT, "tests", "test_gpu_shard.py") + "::test_virtual_shards_multi_rhs",
           os.path.join(ROOT, "tests", "test_gpu_shard.py") + "::test_virtual_shards_forced_colsrc_path"]
    r = subprocess.run(cmd, cwd=ROOT, env=_env(checked_lib), capture_output=True, text=True, timeout=1500)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert "hm device check" not in r.stdout


_SELFTEST = r"""
import numpy as np, torch, paper_2305_06891_b200 as hm, synth
assert hm.load_library()._name.endswith("libhm_checked.so")
cfg = synth.make_config(1); f = cfg.facets
ctx = hm.hm_init(0)
g = hm.hm_build_geometry(ctx, f.centroid, f.normal, f.area, f.aabb, n_min=cfg.n_min, eta=cfg.eta)
F = hm.hm_assemble_aca(ctx, g, eps_aca=cfg.eps_aca)
x = torch.ones(f.n, dtype=torch.float64, device="cuda"); y = torch.empty_like(x)
try:
    hm.hm_apply_F(ctx, F, x, y)
    torch.cuda.synchronize()
except Exception as e:
    print("CALL FAILED:", type(e).__name__, e, flush=True)
    raise SystemExit(3)
print("CALL RETURNED", flush=True)
"""


def test_checked_build_traps_on_a_chunk_outside_its_arena(checked_lib):
    r = subprocess.run([sys.executable, "-c", _SELFTEST], cwd=ROOT, env=_env(checked_lib, HM_CHECK_SELFTEST="1"),
                       capture_output=True, text=True, timeout=600)
    out = r.stdout + r.stderr
    assert "CALL RETURNED" not in out, out[-3000:]
    assert "hm device check failed" in out, out[-3000:]
