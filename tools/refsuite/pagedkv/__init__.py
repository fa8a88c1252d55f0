"""Import-swap shim: the reference test suite's `pagedkv` imports resolved to
the B200 package (test scaffolding for tools/run_reference_suite.py; not part
of the product).  Modules the hot path does not cover (workload, cli) are
absent on purpose, so their tests fail at import."""
from paper_2410_00161_b200 import *  # noqa: F401,F403
from paper_2410_00161_b200 import errors  # noqa: F401
