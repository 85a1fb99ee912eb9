"""CPU oracles (test infrastructure only; see numerics.py header)."""
