"""CPU oracle for the CODA hot path — test infrastructure only (see coda_oracle.py)."""
