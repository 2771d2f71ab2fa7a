"""CPU oracle (TEST INFRASTRUCTURE ONLY): see oracle/drs_oracle.h."""
