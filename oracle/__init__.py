"""Oracles — TEST INFRASTRUCTURE ONLY (see oracle/o1.h, o2_exact.py)."""
