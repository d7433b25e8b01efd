"""CPU RNS-CKKS oracle — TEST INFRASTRUCTURE ONLY (see ckks_oracle.c header)."""
