"""Repeat the loopback sharded-C5 parity run under several settings (diagnostic)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from tests.test_gpu_loopback import _run  # noqa: E402

for p, contract, graph in [(4, "3xtf32", 1), (4, "3xtf32", 0), (2, "f64", 0), (4, "f64", 1), (8, "3xtf32", 1)]:
    for rep in range(3):
        try:
            w = _run(p, contract, 2, graph=graph)
            print(f"p={p} {contract} graph={graph} rep {rep}: ok worst {w:.2e}", flush=True)
        except AssertionError as e:
            print(f"p={p} {contract} graph={graph} rep {rep}: FAIL {str(e)[:160]}", flush=True)
