"""Puts tests/ on sys.path so tools can reuse the test helpers (initial conditions)."""
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
