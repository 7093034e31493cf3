"""CPU oracle (test infrastructure only; see sparse_oracle.py header)."""
