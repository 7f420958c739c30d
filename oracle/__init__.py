"""CPU oracle of the M2Cache sparse mixed-precision FFN decode step.

TEST INFRASTRUCTURE ONLY (see m2c_oracle.c header): importable by tests/,
__graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs only.
"""
