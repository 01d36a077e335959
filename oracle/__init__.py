"""CPU oracle for the SSH hot path (test infrastructure only; see oracle.py)."""
