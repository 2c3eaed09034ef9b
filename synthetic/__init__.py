"""Seeded synthetic inputs shared by the oracle side and the CUDA side.

Holds NONE of the method's arithmetic: it only draws token ids, tables and
output gradients.  Imported by tests/, bench.py and
__graft_entry__.smoke(); never by oracle/ or the product package.
"""

from .workloads import CONFIGS, Workload, get_config, make_workload  # noqa: F401
