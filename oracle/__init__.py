"""TEST INFRASTRUCTURE ONLY: CPU oracles for the SAD hot path (see oracle/sad_oracle.h)."""
