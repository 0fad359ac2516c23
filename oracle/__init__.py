"""CPU oracle for the hot path — TEST INFRASTRUCTURE ONLY (see nnmg_oracle.py)."""
