"""Test-infrastructure oracle package (see particula_oracle.py header).

Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline legs may
import this package.  It is never part of the product path.
"""
