"""Shim: qcur.cur -> paper_2402_19147_b200.cur (test infrastructure)."""
from paper_2402_19147_b200.cur import *  # noqa: F401,F403
