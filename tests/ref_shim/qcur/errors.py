"""Shim: qcur.errors -> paper_2402_19147_b200.errors (test infrastructure)."""
from paper_2402_19147_b200.errors import *  # noqa: F401,F403
