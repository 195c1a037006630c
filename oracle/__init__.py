"""Parity oracle (TEST INFRASTRUCTURE ONLY; see oracle.py)."""
