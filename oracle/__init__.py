"""CPU oracle (test infrastructure only -- see ctkv_oracle.py header)."""
