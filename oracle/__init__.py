"""CPU oracle (test infrastructure only; see ensmhd_oracle.py header)."""
