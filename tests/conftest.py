"""Shared pytest setup.

* ``gpu`` marks tests that need a B200 (run with ``-m gpu`` on the box);
  everything else must pass on a CPU-only host.
* The repo root goes on ``sys.path`` so ``oracle`` (test infrastructure) and
  the package import without installation.
"""

import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: long-running CPU test")
