"""ORACLE -- TEST INFRASTRUCTURE ONLY (see pf_oracle.py).

Only tests/, __graft_entry__.smoke() and bench.py's CPU baseline legs import this.
"""
