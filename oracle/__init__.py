"""CPU oracle for parity tests and the CPU baseline -- test infrastructure only.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline/reference legs
may import this package.  See port.py for what it restates and how it is pinned.
"""
