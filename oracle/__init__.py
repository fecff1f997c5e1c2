"""CPU oracle -- TEST INFRASTRUCTURE ONLY.

Restatements of the reference's semiring-MM / Strassen arithmetic used as the
checker by tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg.
The product package (paper_2011_01441_b200/) never imports this directory.
"""
