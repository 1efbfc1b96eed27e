"""B200-native batched Schur-complement (FETI dual operator) assembly — arXiv 2509.21037 hot path.

C ABI: include/sc_b200.h, implemented by libsc_b200.so (sm_100a) built from csrc/.
Python binding (marshalling only): paper_2509_21037_b200.sc.SCPlan.
"""
from .sc import SCPlan, ScError, SKIP_NONE, SKIP_ENVELOPE, SKIP_EXACT, STRIP_AUTO, STRIP_SHARED, STRIP_GLOBAL, lib  # noqa: F401
