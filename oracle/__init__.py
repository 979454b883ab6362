"""fp64 CPU oracle (TEST INFRASTRUCTURE ONLY; see attention_oracle.py header).

Importable only from tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference legs.  The product package never imports it.
"""
from .attention_oracle import NEG_INF, attention, attention_group, merge, partial  # noqa: F401
