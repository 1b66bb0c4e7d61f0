"""CPU oracle package — test infrastructure only (see pppm_oracle.py header)."""
