"""CPU oracle of ASSE's hot path — TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
reference legs may import this package. See oracle/asse_oracle.c.
"""
