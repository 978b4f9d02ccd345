"""CPU oracle (test infrastructure only; see oracle/wbf_oracle.py header)."""
