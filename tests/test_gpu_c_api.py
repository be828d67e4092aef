"""The C ABI without Python (include/hm.h): examples/c_api_demo.c compiled with gcc against the in-tree
libhm.so and run on the GPU -- a closed cube of square facets, F x against direct one-point sums, the
black-body solve (C = I) and the uniform-temperature flux (q = 0)."""
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_c_api_demo(tmp_path):
    import paper_2305_06891_b200.build as b
    lib = b.build()
    exe = str(tmp_path / "c_api_demo")
    libdir = os.path.dirname(lib)
    r = subprocess.run(["gcc", "-O2", "-Wall", "-I", os.path.join(ROOT, "include"),
                        os.path.join(ROOT, "examples", "c_api_demo.c"), "-L", libdir, "-lhm",
                        f"-Wl,-rpath,{libdir}", "-lm", "-o", exe], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    r = subprocess.run([exe, "12"], capture_output=True, text=True, timeout=300)
    print(r.stdout, r.stderr)
    assert r.returncode == 0 and r.stdout.strip().endswith("OK"), r.stdout + r.stderr
