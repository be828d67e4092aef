"""Stress the virtual-shard level-form tests in one process (flakiness hunt)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import test_gpu_shard as T  # noqa: E402

for it in range(4):
    for (w, c) in [(2, 99), (4, 99), (4, 1), (8, 2), (4, 0)]:
        try:
            T.test_virtual_shards_level_form(w, c)
            print(it, w, c, "ok", flush=True)
        except AssertionError as e:
            print(it, w, c, "FAIL", str(e)[:400], flush=True)
