"""ORACLE -- test infrastructure only (see deft_oracle.py / subset_sum.c headers).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
reference legs may import this package, and only as the checker.
"""
