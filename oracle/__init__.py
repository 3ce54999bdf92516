"""Test-infrastructure oracle (CPU restatement of the reference hot path).

Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline legs may
import this package.  See lf_oracle.py for the header and citations.
"""
