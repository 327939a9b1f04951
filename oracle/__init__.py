"""ORACLE -- test infrastructure only.

CPU restatement of the reference `rasterbound` join path, used as
the parity checker by tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference legs.  The product package never imports it.
"""
