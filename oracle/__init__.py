"""CPU oracle for the MI hot path -- TEST INFRASTRUCTURE ONLY.

Imported by tests/, __graft_entry__.smoke() and bench.py's CPU-baseline /
--impl reference leg, never by the product package.  See oracle/oracle.py.
"""
