"""CPU oracle (test infrastructure only; see lfmm_oracle.py header)."""
