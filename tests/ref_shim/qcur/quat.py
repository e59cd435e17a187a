"""Shim: qcur.quat -> paper_2402_19147_b200.quat (test infrastructure)."""
from paper_2402_19147_b200.quat import *  # noqa: F401,F403
