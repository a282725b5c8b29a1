"""CPU oracle -- TEST INFRASTRUCTURE ONLY (see ring_oracle.py header)."""
