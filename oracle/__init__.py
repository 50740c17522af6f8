"""TEST INFRASTRUCTURE ONLY: CPU oracles for the parity tests (see oracle/faith_oracle.h)."""
