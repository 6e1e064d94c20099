"""pytest configuration: the `gpu` marker and shared paths.

`-m "not gpu"` runs the oracle-vs-golden checks, host-side logic and ABI
loading on CPU; `-m gpu` runs the parity tests proper through libqsb.so on a
B200 (they fail loudly, never skip silently, when the GPU path is missing).
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
TESTS = os.path.dirname(os.path.abspath(__file__))
if TESTS not in sys.path:
    sys.path.insert(0, TESTS)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")
