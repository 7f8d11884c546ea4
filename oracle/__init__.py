"""CPU oracle package -- TEST INFRASTRUCTURE ONLY (see kriging_oracle.py)."""
