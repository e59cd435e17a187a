"""Shim: qcur.linalg -> paper_2402_19147_b200.linalg (test infrastructure)."""
from paper_2402_19147_b200.linalg import *  # noqa: F401,F403
