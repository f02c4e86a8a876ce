"""CPU oracle for the fork-attention path — TEST INFRASTRUCTURE ONLY.

Imported by tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
--impl reference legs, as the checker or the timed CPU baseline; never by
the product package.
"""
