"""Checkers for the Certaindex hot path (TEST INFRASTRUCTURE ONLY; see oracle.py)."""
