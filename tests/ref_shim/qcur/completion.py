"""Shim: qcur.completion -> paper_2402_19147_b200.completion (test infrastructure)."""
from paper_2402_19147_b200.completion import *  # noqa: F401,F403
