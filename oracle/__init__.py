"""CPU oracle for the LPA hot path -- test infrastructure only (see oracle.py)."""
