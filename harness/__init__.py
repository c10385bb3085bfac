"""Measurement harness shared by tests and bench.py (no BILU arithmetic here)."""
