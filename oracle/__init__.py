"""fp64 CPU oracle -- TEST INFRASTRUCTURE ONLY (tests/, smoke(), bench.py cpu_baseline/reference).

The product package never imports this; see asot_oracle.py's header.
"""
from . import asot_oracle  # noqa: F401
