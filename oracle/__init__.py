"""Parity oracle package -- TEST INFRASTRUCTURE ONLY (see oracle/rf_oracle.c header).

Importable from tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference
legs; never from paper_2603_12646_b200/.
"""
from .oracle import *  # noqa: F401,F403
