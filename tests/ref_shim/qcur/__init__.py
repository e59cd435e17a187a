"""Test shim: the reference package's import names (`qcur`, `qcur.cur`, ...) bound to this
repository's GPU implementation, so the reference's own test modules run unmodified against
it (tests/test_gpu_reference_suite.py).  Test infrastructure only; never on the product path."""
from paper_2402_19147_b200 import *  # noqa: F401,F403
from paper_2402_19147_b200 import __all__  # noqa: F401
